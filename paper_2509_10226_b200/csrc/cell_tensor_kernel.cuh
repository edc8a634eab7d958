// Cell-term kernel, reference-tensor form (affine cells), on FP64 tensor cores.
//
// The reference sums over quadrature points (operator.py:255-278,
// numpy_backend.py:48-88):
//     y_e = E^T W (D_e (E u_e)),   D_e = J^-1 jxw J^-T  (constant per affine cell)
// Because D_e does not depend on the point for affine geometry (the reference's
// "affine" GeometryData mode, geometry.py:145-151), the point sum can be taken
// once per plan on the host:
//     y_e = sum_{k<=l} G_kl,e S^kl u_e  (+ m_e M u_e)
//     S^kk = sum_q w_q d_k phi_i d_k phi_j,   S^kl = sum_q w_q (d_k phi_i d_l phi_j + d_l phi_i d_k phi_j)
//     M    = sum_q w_q phi_i phi_j
// with G = stiff * kappa_e * det J * J^-1 J^-T packed (00,01,02,11,12,22) and
// m_e = mass * det J (cell_geometry_kernel).  Per 8-cell tile that is ONE GEMM
//     W^T[8 cells, (i, kl)] = U^T[8, N] . S[N, (i, kl)]
// of KK x (NP KK) DMMAs (KK = ceil(N/4), NP = 3 column pairs, 4 with mass) and a
// 6 (7)-term contraction per output DoF in registers: 3 / 27 / 75 / 243 DMMAs
// per tile at P1-P4 against 9 / 42 / 151 / 513 for the quadrature-point form
// (cell_kernel.cuh), i.e. 12 N^2 instead of 12 n_q N multiply-adds per cell.
//
// Column order: n-tile (ib, p) holds, in column n, DoF i = 4 ib + (n >> 1) and
// packed coefficient kl = 2 p + (n & 1), so the C fragment gives lane
// (cs = lane>>2, q4 = lane&3) the coefficient pair (2p, 2p+1) of DoF 4 ib + q4
// of cell cs: the contraction needs no shuffles, and the lane's output DoF is
// the DoF whose index it gathered for GEMM k-step ib (the scatter reuses it).
//
// The quadrature-point engine (cell_kernel.cuh) stays the general path (per
// point geometry/coefficients); this engine needs per-cell constant D_e, which
// is what every operator of this library has.
#pragma once
#include "cell_kernel.cuh"

namespace tmf {

template <int N, bool MASS>
struct TensorShape {
  static constexpr int KK = (N + 3) / 4;    // k-steps (gathered DoFs j) = i-blocks (output DoFs)
  static constexpr int NP = MASS ? 4 : 3;   // coefficient pairs per i-block
  static constexpr int NFRAG = KK * NP * KK;
  static constexpr int SMEM = NFRAG * 32 * 8;
  static constexpr int DMMA_PER_TILE = NFRAG;
};

// MT: 8-cell tiles per warp iteration (they share every B-fragment load)
template <int N, bool MASS, bool DG, int BLOCK, int MT, int MINB, bool PEER = false>
__global__ void __launch_bounds__(BLOCK, MINB) cell_tensor_kernel(CellArgs a) {
  using S = TensorShape<N, MASS>;
  constexpr int KK = S::KK, NP = S::NP;
  extern __shared__ __align__(16) double smem[];
  {
    const double2* src = reinterpret_cast<const double2*>(a.frags);
    double2* dst = reinterpret_cast<double2*>(smem);
    for (int i = threadIdx.x; i < S::NFRAG * 16; i += BLOCK) dst[i] = __ldg(src + i);
  }
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int cs = lane >> 2;
  const int q4 = lane & 3;
  const int64_t ctiles = (a.n_cells + 7) / 8;
  const int64_t cst = (ctiles + MT - 1) / MT;   // super-tiles per component
  const int64_t nst = cst * a.nc;
  const int64_t nwarps = (int64_t)gridDim.x * (BLOCK / 32);
  const int64_t step = nwarps;
  int64_t st = (int64_t)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5);

  // DoF indices of the warp's next super-tile are loaded while this one computes
  int nidx[MT][KK];
  auto load_indices = [&](int64_t t) {
    const int cmp = a.nc == 1 ? 0 : (int)(t / cst);
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int64_t c = ((t - (int64_t)cmp * cst) * MT + m) * 8 + cs;
      const bool ok = t < nst && c < a.n_cells;
#pragma unroll
      for (int kk = 0; kk < KK; ++kk) {
        const int j = 4 * kk + q4;
        nidx[m][kk] = -1;
        if (ok && j < N) nidx[m][kk] = DG ? (int)(c * N + j) : __ldg(a.dofs + c * N + j);
      }
    }
  };
  load_indices(st);

  // gathered u, indices (kept for the scatter) and geometry of super-tile t
  auto load_data = [&](int64_t t, int (&ix)[MT][KK], double (&av)[MT][KK], double (&G)[MT][6],
                       double (&mdet)[MT]) {
    const int cmp = a.nc == 1 ? 0 : (int)(t / cst);
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int64_t c = ((t - (int64_t)cmp * cst) * MT + m) * 8 + cs;
      const bool ok = t < nst && c < a.n_cells;
#pragma unroll
      for (int kk = 0; kk < KK; ++kk) {
        const int g = ix[m][kk] = nidx[m][kk];
        TMF_CHECK(a, g < 0 || (int64_t)g * a.nc + cmp < a.dbg_n_dofs, TMF_DBG_DOF);
        TMF_CHECK(a, !ok || c < a.dbg_n_cells, TMF_DBG_CELL);
        if (PEER)
          av[m][kk] = (g >= 0) ? __ldg(peer_src(a.peer, a.u, g, a.nc, cmp)) : 0.0;
        else
          av[m][kk] = (g >= 0) ? __ldg(a.u + (int64_t)g * a.nc + cmp) : 0.0;
      }
      const double2* gp = reinterpret_cast<const double2*>(a.cgeo + 8 * (ok ? c : 0));
      const double2 g01 = __ldg(gp), g23 = __ldg(gp + 1), g45 = __ldg(gp + 2);
      G[m][0] = g01.x; G[m][1] = g01.y; G[m][2] = g23.x;
      G[m][3] = g23.y; G[m][4] = g45.x; G[m][5] = g45.y;
      mdet[m] = MASS ? __ldg(a.cgeo + 8 * (ok ? c : 0) + 6) : 0.0;
    }
  };
  double en = 0.0;   // sum of u_i y_i over the lane's outputs (element energies, CG)

  if (!DG) pdl_wait_prior_grid();   // y cleared (common.cuh); nothing above touches y
  for (; st < nst; st += step) {
    const int comp = a.nc == 1 ? 0 : (int)(st / cst);
    int64_t cell[MT];
    int idx[MT][KK];
    double av[MT][KK], G[MT][6], mdet[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) cell[m] = ((st - (int64_t)comp * cst) * MT + m) * 8 + cs;
    load_data(st, idx, av, G, mdet);
    load_indices(st + step);

    // one i-block at a time: GEMM columns (ib, kl), contraction, then its scatter/store
    // (the lane owns DoF 4 ib + q4 of cell cs, whose index it gathered for k-step ib)
#pragma unroll
    for (int ib = 0; ib < KK; ++ib) {
      double yv[MT];
#pragma unroll
      for (int m = 0; m < MT; ++m) yv[m] = 0.0;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        double w[MT][2];
#pragma unroll
        for (int m = 0; m < MT; ++m) w[m][0] = w[m][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KK; ++kk) {
          const double b = smem[((ib * NP + p) * KK + kk) * 32 + lane];
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma(w[m], av[m][kk], b);
        }
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          if (p < 3) {
            yv[m] = fma(G[m][2 * p], w[m][0], yv[m]);
            yv[m] = fma(G[m][2 * p + 1], w[m][1], yv[m]);
          } else {
            yv[m] = fma(mdet[m], w[m][0], yv[m]);
          }
        }
      }
      const int j = 4 * ib + q4;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (j >= N || cell[m] >= a.n_cells) continue;
        if (DG) {
          TMF_CHECK(a, (cell[m] * N + j) * a.nc + comp < a.dbg_n_dofs, TMF_DBG_DOF);
          a.y[(cell[m] * N + j) * a.nc + comp] = yv[m];
        } else {
          const int g = idx[m][ib];
          en = fma(av[m][ib], yv[m], en);   // av = u at this DoF (0 when masked)
          if (g >= 0) {
            if (PEER)
              peer_red_add(peer_dst(a.peer, a.y, g, a.nc, comp), yv[m]);
            else
              atomicAdd(a.y + (int64_t)g * a.nc + comp, yv[m]);
          }
        }
      }
    }
  }
  if (!DG && a.energy != nullptr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) en += __shfl_xor_sync(0xffffffffu, en, o);
    if (lane == 0) atomicAdd(a.energy, en);
  }
  if (PEER && a.peer.y != nullptr) __threadfence_system();
}

}  // namespace tmf
