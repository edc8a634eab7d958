// Single-precision CG Laplace cell kernel for the multigrid V-cycle (mixed precision: the
// paper runs its V-cycle in fp32 while the outer CG stays fp64).
//
// The modal form of the cell term: y_e = sum_m E'_m^T G_e E'_m u_e with the
// M = dim P_{p-1} unit-weight modes E'(k, m, i) of the plan's gradient tables, so per cell
// 2 * 3 M N FFMAs + 15 M for the G action.  One thread per cell: gathered u and the
// cell's residual live in registers, the mode rows E'[m][k][0..NP) (NP = N rounded up to
// 4) sit in shared memory and are read as warp-uniform float4 broadcasts, each feeding 4
// FFMAs.  Geometry: G (6 floats, padded to 8) per cell, converted once from the fp64
// plan geometry.  Scatter: fp32 RED.  Dirichlet DoFs are ~idx < 0 as in the fp64 kernels.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace tmf {

template <int N>
struct F32Shape {
  static constexpr int NP = (N + 3) & ~3;
};

template <int N, int M, int BLOCK>
__global__ void __launch_bounds__(BLOCK) cell_f32_kernel(const float* __restrict__ u, float* __restrict__ y,
                                                         const int* __restrict__ dofs,
                                                         const float4* __restrict__ g32,
                                                         const float4* __restrict__ rows, int64_t n_cells) {
  constexpr int NP = F32Shape<N>::NP;
  constexpr int R4 = M * 3 * NP / 4;   // float4 rows in shared memory
  __shared__ float4 sr[R4];
  for (int i = threadIdx.x; i < R4; i += BLOCK) sr[i] = rows[i];
  __syncthreads();
  for (int64_t c = (int64_t)blockIdx.x * BLOCK + threadIdx.x; c < n_cells; c += (int64_t)gridDim.x * BLOCK) {
    float uu[NP], yy[NP];
    const int* dp = dofs + c * N;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      uu[j] = 0.0f;
      yy[j] = 0.0f;
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const int g = __ldg(dp + j);
      uu[j] = g >= 0 ? __ldg(u + g) : 0.0f;
    }
    const float4 ga = __ldg(g32 + 2 * c), gb = __ldg(g32 + 2 * c + 1);
    const float G0 = ga.x, G1 = ga.y, G2 = ga.z, G3 = ga.w, G4 = gb.x, G5 = gb.y;
#pragma unroll (M <= 4 ? M : 2)
    for (int m = 0; m < M; ++m) {
      const float4* r = sr + m * 3 * (NP / 4);
      float g[3] = {0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int j4 = 0; j4 < NP / 4; ++j4) {
          const float4 e = r[k * (NP / 4) + j4];
          g[k] = fmaf(e.x, uu[4 * j4], g[k]);
          g[k] = fmaf(e.y, uu[4 * j4 + 1], g[k]);
          g[k] = fmaf(e.z, uu[4 * j4 + 2], g[k]);
          g[k] = fmaf(e.w, uu[4 * j4 + 3], g[k]);
        }
      const float d0 = G0 * g[0] + G1 * g[1] + G2 * g[2];
      const float d1 = G1 * g[0] + G3 * g[1] + G4 * g[2];
      const float d2 = G2 * g[0] + G4 * g[1] + G5 * g[2];
      const float d[3] = {d0, d1, d2};
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int j4 = 0; j4 < NP / 4; ++j4) {
          const float4 e = r[k * (NP / 4) + j4];
          yy[4 * j4] = fmaf(e.x, d[k], yy[4 * j4]);
          yy[4 * j4 + 1] = fmaf(e.y, d[k], yy[4 * j4 + 1]);
          yy[4 * j4 + 2] = fmaf(e.z, d[k], yy[4 * j4 + 2]);
          yy[4 * j4 + 3] = fmaf(e.w, d[k], yy[4 * j4 + 3]);
        }
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const int g = __ldg(dp + j);
      if (g >= 0) atomicAdd(y + g, yy[j]);
    }
  }
}

// fp64 plan geometry (8 doubles: G[6], mass, pad) -> fp32 G (8 floats)
static __global__ void geo_to_f32_kernel(const double* __restrict__ g64, float* __restrict__ g32, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i >> 3;
    const int k = (int)(i & 7);
    g32[i] = k < 6 ? (float)g64[8 * e + k] : 0.0f;
  }
}

// identity rows on Dirichlet DoFs (fp32 mirror of dirichlet_fixup_kernel)
static __global__ void fixup_f32_kernel(const float* __restrict__ u, float* __restrict__ y,
                                        const int* __restrict__ list, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int g = list[i];
    y[g] = u[g];
  }
}

}  // namespace tmf
