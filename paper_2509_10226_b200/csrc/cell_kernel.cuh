// Cell-term kernel of the matrix-free apply on FP64 tensor cores (sm_100a).
//
// Restates the reference cell loop (operator.py:255-278):
//     U = gather(u)                      numpy_backend.py:23-35
//     V = E_grad @ U                     numpy_backend.py:48-55
//     D = J^-1 (jxw * J^-T V)            numpy_backend.py:68-76
//     R = E_grad^T @ D  (+ E_val^T (mass_scale jxw E_val U))  :58-65, :86-88
//     y += scatter(R)                    numpy_backend.py:38-40
// as two chained DMMA GEMMs per warp over a tile of 8 cells (M = cells):
//
//   GEMM1  V^T[8 cells, (t,c,pt)] = U^T[8, N] . E^T[N, (t,c,pt)]
//          component-major point tiles: tile (t, c) holds component c of the
//          8 quadrature points 8t..8t+7, so each lane ends up owning ALL
//          components of points 8t + 2(lane&3) + {0,1} for its cell;
//   D      in registers: d = w_q (G g)  (w_q folded into the GEMM2 table)
//   GEMM2  Y^T[8, N] += D^T[8, (t,c,i,lane&3)] . Ew[(t,c,i,k), N]
//          the C fragment of GEMM1 *is* the A fragment of GEMM2 once the K
//          index of GEMM2 is ordered (t, c, i, lane&3): no shuffles, no smem.
//
// Both B operands are constant tables, pre-swizzled on the host into
// lane-major fragments (frag[f][lane]) and staged once per CTA in shared
// memory (one conflict-free LDS.64 per DMMA).  Geometry (J, det, adjugate)
// is recomputed from the 4 vertex coordinates, so the only per-cell traffic
// is the vertex ids, DoF indices and the gathered/scattered vector entries.
//
// CG: masked (Dirichlet) DoFs are encoded as ~idx (< 0): gathered as 0 and
// never scattered (operator.py:327-328 fixes y on them afterwards).  The
// scatter uses fp64 RED (red.global.add.f64); DG cells own their DoFs, so
// the DG variant stores y directly and the face kernel adds onto it.
#pragma once
#include "common.cuh"

namespace tmf {

struct CellArgs {
  const double* __restrict__ u;
  double* __restrict__ y;
  const int* __restrict__ dofs;    // CG: (n_cells, N) encoded; DG: nullptr (contiguous)
  const int* __restrict__ cells;   // (n_cells, 4)
  const double* __restrict__ verts;
  const double* __restrict__ kappa;  // per-cell Laplace coefficient or nullptr
  const double* __restrict__ frags;  // B1 then B2 fragments (global; staged to smem)
  int64_t n_cells;
  int nc;                          // interleaved components
  double mass_scale;
  double stiff_scale;
};

template <int N, int Q, bool MASS>
struct CellShape {
  static constexpr int KK = (N + 3) / 4;     // GEMM1 k-steps (DoFs)
  static constexpr int T = (Q + 7) / 8;      // point tiles
  static constexpr int NJ = (N + 7) / 8;     // GEMM2 n-tiles (DoFs)
  static constexpr int NC = MASS ? 4 : 3;    // value (mass) + 3 reference gradients
  static constexpr int NB1 = T * NC * KK;
  static constexpr int NB2 = T * NC * 2 * NJ;
  static constexpr int NFRAG = NB1 + NB2;
  static constexpr int SMEM = NFRAG * 32 * 8;
  static constexpr int DMMA_PER_TILE = NB1 + NB2;
};

template <int N, int Q, bool MASS, bool DG, int BLOCK>
__global__ void __launch_bounds__(BLOCK) cell_apply_kernel(CellArgs a) {
  using S = CellShape<N, Q, MASS>;
  extern __shared__ __align__(16) double smem[];
  {
    const double2* src = reinterpret_cast<const double2*>(a.frags);
    double2* dst = reinterpret_cast<double2*>(smem);
    for (int i = threadIdx.x; i < S::NFRAG * 16; i += BLOCK) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const double* sB1 = smem;
  const double* sB2 = smem + S::NB1 * 32;

  const int lane = threadIdx.x & 31;
  const int cs = lane >> 2;  // cell slot in the tile
  const int q4 = lane & 3;
  const int64_t ctiles = (a.n_cells + 7) / 8;
  const int64_t ntiles = ctiles * a.nc;
  const int64_t nwarps = (int64_t)gridDim.x * (BLOCK / 32);

  // Index prefetch: the DoF indices and vertex ids of the warp's next tile are
  // loaded while the current tile computes, so each tile start pays one memory
  // round trip (u, coordinates) instead of two (indices, then data).
  int64_t tile = (int64_t)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5);
  int nidx[S::KK];
  int nvid[4];
  auto load_indices = [&](int64_t t) {
    const int cmp = (int)(t / ctiles);
    const int64_t c = (t - (int64_t)cmp * ctiles) * 8 + cs;
    const bool ok = t < ntiles && c < a.n_cells;
#pragma unroll
    for (int kk = 0; kk < S::KK; ++kk) {
      const int j = 4 * kk + q4;
      nidx[kk] = -1;
      if (ok && j < N) nidx[kk] = DG ? (int)(c * N + j) : __ldg(a.dofs + c * N + j);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) nvid[i] = ok ? __ldg(a.cells + 4 * c + i) : 0;
  };
  load_indices(tile);

  for (; tile < ntiles; tile += nwarps) {
    const int comp = (int)(tile / ctiles);
    const int64_t cell = (tile - (int64_t)comp * ctiles) * 8 + cs;
    const bool valid = cell < a.n_cells;
    int vid[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) vid[i] = nvid[i];

    // ---- gather: A fragments of GEMM1 (lane owns DoFs 4kk + q4 of its cell)
    double av[S::KK];
#pragma unroll
    for (int kk = 0; kk < S::KK; ++kk) {
      const int g = nidx[kk];
      av[kk] = (g >= 0) ? __ldg(a.u + (int64_t)g * a.nc + comp) : 0.0;
    }
    // DG indices are (cell*N + j) and may exceed int range only beyond 2^31 DoFs
    // (rejected at plan creation).

    // ---- geometry: G = scale * adj adj^T / det, mass factor det
    double G[6];
    double mdet = 0.0;
    {
      const int64_t c = valid ? cell : 0;
      Affine g;
      affine_from_vertices(load_vertex(a.verts, vid[0]), load_vertex(a.verts, vid[1]),
                           load_vertex(a.verts, vid[2]), load_vertex(a.verts, vid[3]), g);
      double sc = a.stiff_scale;
      if (a.kappa) sc *= __ldg(a.kappa + c);
      stiffness_metric(g, sc, G);
      if (MASS) mdet = a.mass_scale * g.det;
    }
    load_indices(tile + nwarps);

    double yacc[S::NJ][2];
#pragma unroll
    for (int nj = 0; nj < S::NJ; ++nj) yacc[nj][0] = yacc[nj][1] = 0.0;

#pragma unroll
    for (int t = 0; t < S::T; ++t) {
      double v[S::NC][2];
#pragma unroll
      for (int c = 0; c < S::NC; ++c) v[c][0] = v[c][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk) {
#pragma unroll
        for (int c = 0; c < S::NC; ++c)
          dmma(v[c], av[kk], sB1[((t * S::NC + c) * S::KK + kk) * 32 + lane]);
      }
      // D action at the lane's two points (w_q lives in the GEMM2 table)
      double d[S::NC][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        constexpr int o = MASS ? 1 : 0;
        const double g0 = v[o][i], g1 = v[o + 1][i], g2 = v[o + 2][i];
        d[o][i] = G[0] * g0 + G[1] * g1 + G[2] * g2;
        d[o + 1][i] = G[1] * g0 + G[3] * g1 + G[4] * g2;
        d[o + 2][i] = G[2] * g0 + G[4] * g1 + G[5] * g2;
        if (MASS) d[0][i] = mdet * v[0][i];
      }
#pragma unroll
      for (int c = 0; c < S::NC; ++c)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int nj = 0; nj < S::NJ; ++nj)
            dmma(yacc[nj], d[c][i], sB2[(((t * S::NC + c) * 2 + i) * S::NJ + nj) * 32 + lane]);
    }

    // ---- scatter / store: lane owns DoFs 8nj + 2q4 + {0,1}
    if (valid) {
#pragma unroll
      for (int nj = 0; nj < S::NJ; ++nj)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int j = 8 * nj + 2 * q4 + i;
          if (j < N) {
            if (DG) {
              a.y[(cell * N + j) * a.nc + comp] = yacc[nj][i];
            } else {
              const int64_t g = __ldg(a.dofs + cell * N + j);
              if (g >= 0) atomicAdd(a.y + g * a.nc + comp, yacc[nj][i]);
            }
          }
        }
    }
  }
}

// y[c] = u[c] on strongly constrained DoFs (identity rows, operator.py:327-328)
static __global__ void dirichlet_fixup_kernel(const double* __restrict__ u, double* __restrict__ y,
                                       const int* __restrict__ list, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = list[i];
    y[g] = u[g];
  }
}

}  // namespace tmf
