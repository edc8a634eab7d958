// Cell-term kernel on the FP64 vector pipe (DFMA), for low degrees.
//
// Same algorithm as cell_kernel.cuh (operator.py:255-278: gather -> E_grad U
// -> D action -> E_grad^T D -> scatter-add), but one thread owns MC cells and
// runs the point loop itself:
//
//   for q:  g_c   = sum_j E_c(q, j) u_j              (c = value? + 3 gradients)
//           d     = G g  (+ mass: m g_0)               D action, G = det J^-1 J^-T
//           y_j  += sum_c w_q E_c(q, j) d_c
//
// At P1/P2 the DMMA tile shapes waste most of the tensor work on padding (P1:
// 8-point tiles for 5 points and 8-wide DoF tiles for 4 DoFs, 42 % useful;
// P2: 67 %), while DFMA and DMMA share one FP64 datapath on B200 at the same
// FMA rate (profiles/r01_fp64_peak.json, r01/fp64_mix_microbench.json).  Here
// every issued FMA is useful.  Both tables are point-major rows [q][c][j]
// (j padded to even) in shared memory and are read as warp-uniform LDS.128
// broadcasts, each feeding 2*MC DFMAs.
//
// Masked (Dirichlet) CG DoFs are ~idx < 0 exactly as in the DMMA kernel.
#pragma once
#include "cell_kernel.cuh"

namespace tmf {

template <int N, int Q, bool MASS>
struct DfmaShape {
  static constexpr int NP = (N + 1) & ~1;        // padded row length
  static constexpr int NC = MASS ? 4 : 3;
  static constexpr int TAB = Q * NC * NP;        // doubles per table
  static constexpr int SMEM = 2 * TAB * 8;
};

// The point loop of one thread's MC cells: uu (gathered u, padded to NP) ->
// yy (cell residual), G / md the per-cell metric and mass factor, T1 / T2 the
// point-major rows E and w_q E in shared memory.
template <int N, int Q, bool MASS, int MC>
__device__ __forceinline__ void dfma_cell_points(const double2* __restrict__ T1, const double2* __restrict__ T2,
                                                 const double (&uu)[MC][DfmaShape<N, Q, MASS>::NP],
                                                 const double (&G)[MC][6], const double (&md)[MC],
                                                 double (&yy)[MC][DfmaShape<N, Q, MASS>::NP]) {
  using S = DfmaShape<N, Q, MASS>;
  constexpr int NP = S::NP, NC = S::NC;
#pragma unroll
  for (int m = 0; m < MC; ++m)
#pragma unroll
    for (int j = 0; j < NP; ++j) yy[m][j] = 0.0;
#pragma unroll (Q <= 5 ? Q : 1)
  for (int q = 0; q < Q; ++q) {
    const double2* t1 = T1 + q * (NC * NP / 2);
    const double2* t2 = T2 + q * (NC * NP / 2);
    double g[MC][NC];
#pragma unroll
    for (int m = 0; m < MC; ++m)
#pragma unroll
      for (int c = 0; c < NC; ++c) g[m][c] = 0.0;
#pragma unroll
    for (int j = 0; j < NP; j += 2)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double2 e = t1[(c * NP + j) / 2];
#pragma unroll
        for (int m = 0; m < MC; ++m) {
          g[m][c] = fma(e.x, uu[m][j], g[m][c]);
          if (j + 1 < N) g[m][c] = fma(e.y, uu[m][j + 1], g[m][c]);
        }
      }
    double d[MC][NC];
#pragma unroll
    for (int m = 0; m < MC; ++m) {
      constexpr int o = MASS ? 1 : 0;
      const double g0 = g[m][o], g1 = g[m][o + 1], g2 = g[m][o + 2];
      d[m][o] = G[m][0] * g0 + G[m][1] * g1 + G[m][2] * g2;
      d[m][o + 1] = G[m][1] * g0 + G[m][3] * g1 + G[m][4] * g2;
      d[m][o + 2] = G[m][2] * g0 + G[m][4] * g1 + G[m][5] * g2;
      if (MASS) d[m][0] = md[m] * g[m][0];
    }
#pragma unroll
    for (int j = 0; j < NP; j += 2)
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const double2 e = t2[(c * NP + j) / 2];
#pragma unroll
        for (int m = 0; m < MC; ++m) {
          yy[m][j] = fma(e.x, d[m][c], yy[m][j]);
          if (j + 1 < N) yy[m][j + 1] = fma(e.y, d[m][c], yy[m][j + 1]);
        }
      }
  }
}

template <int N, int Q, bool MASS, bool DG, int BLOCK, int MC, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) cell_dfma_kernel(CellArgs a) {
  using S = DfmaShape<N, Q, MASS>;
  constexpr int NP = S::NP;
  constexpr int CH = BLOCK * MC;                     // cells per CTA iteration
  extern __shared__ __align__(16) double smem[];
  {
    const double2* src = reinterpret_cast<const double2*>(a.frags);
    double2* dst = reinterpret_cast<double2*>(smem);
    for (int i = threadIdx.x; i < S::TAB; i += BLOCK) dst[i] = __ldg(src + i);   // 2*TAB doubles
  }
  __syncthreads();
  const double2* T1 = reinterpret_cast<const double2*>(smem);
  const double2* T2 = reinterpret_cast<const double2*>(smem + S::TAB);

  const int64_t cpc = (a.n_cells + CH - 1) / CH;     // chunks per component
  const int64_t nch = cpc * a.nc;
  for (int64_t ch = blockIdx.x; ch < nch; ch += gridDim.x) {
    const int comp = a.nc == 1 ? 0 : (int)(ch / cpc);
    const int64_t base = (ch - (int64_t)comp * cpc) * CH + threadIdx.x;
    double uu[MC][NP], yy[MC][NP], G[MC][6], md[MC];
#pragma unroll
    for (int m = 0; m < MC; ++m) {
      const int64_t c = base + (int64_t)m * BLOCK;
      const bool ok = c < a.n_cells;
      const int64_t cc = ok ? c : 0;
      if (DG) {
#pragma unroll
        for (int j = 0; j < N; ++j) uu[m][j] = ok ? __ldg(a.u + (cc * N + j) * a.nc + comp) : 0.0;
      } else {
        int id[NP];
        const int* dp = a.dofs + cc * N;
        if (N % 4 == 0) {
#pragma unroll
          for (int j = 0; j < N; j += 4) {
            const int4 v = __ldg(reinterpret_cast<const int4*>(dp + j));
            id[j] = v.x; id[j + 1] = v.y; id[j + 2] = v.z; id[j + 3] = v.w;
          }
        } else if (N % 2 == 0) {
#pragma unroll
          for (int j = 0; j < N; j += 2) {
            const int2 v = __ldg(reinterpret_cast<const int2*>(dp + j));
            id[j] = v.x; id[j + 1] = v.y;
          }
        } else {
#pragma unroll
          for (int j = 0; j < N; ++j) id[j] = __ldg(dp + j);
        }
#pragma unroll
        for (int j = 0; j < N; ++j) uu[m][j] = (ok && id[j] >= 0) ? __ldg(a.u + (int64_t)id[j] * a.nc + comp) : 0.0;
      }
      if (NP > N) uu[m][N] = 0.0;
      const double2* gp = reinterpret_cast<const double2*>(a.cgeo + 8 * cc);
      const double2 g01 = __ldg(gp), g23 = __ldg(gp + 1), g45 = __ldg(gp + 2);
      G[m][0] = g01.x; G[m][1] = g01.y; G[m][2] = g23.x;
      G[m][3] = g23.y; G[m][4] = g45.x; G[m][5] = g45.y;
      md[m] = MASS ? __ldg(a.cgeo + 8 * cc + 6) : 0.0;
    }
    dfma_cell_points<N, Q, MASS, MC>(T1, T2, uu, G, md, yy);
#pragma unroll
    for (int m = 0; m < MC; ++m) {
      const int64_t c = base + (int64_t)m * BLOCK;
      if (c >= a.n_cells) continue;
      if (DG) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double* dst = a.y + (c * N + j) * a.nc + comp;
          if (a.accumulate)
            atomicAdd(dst, yy[m][j]);
          else
            *dst = yy[m][j];
        }
      } else {
        const int* dp = a.dofs + c * N;
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const int gid = __ldg(dp + j);
          if (gid >= 0) atomicAdd(a.y + (int64_t)gid * a.nc + comp, yy[m][j]);
        }
      }
    }
  }
}

}  // namespace tmf
