// Matrix-free diagonal and the fused vector kernels of point-Jacobi PCG.
//
// Diagonal (replaces sparse.assemble(...).diagonal(), sparse.py:237-243, which
// the reference only offers on an assembled CSR matrix):
//   diag_i += sum_kl G_kl S_kl[j],  S_kl[j] = sum_q w_q dphi_j/dxi_k dphi_j/dxi_l
// with S precomputed on the host (6 x n_dpc), G = det J^-1 J^-T per cell.
//
// PCG (SPEC.md:509-517 restated; x0 = 0, fixed iteration count): every scalar
// lives on the device in per-iteration slots (rz[k], pq[k], rr[k]), so an
// iteration is apply -> dot(p,q) -> fused {x,r,z update + r.z + r.r} ->
// p = z + beta p, with no host round trip.
#pragma once
#include "common.cuh"

namespace tmf {

struct DiagArgs {
  double* __restrict__ diag;
  const int* __restrict__ dofs;    // encoded (masked < 0)
  const int* __restrict__ cells;
  const double* __restrict__ verts;
  const double* __restrict__ S;    // (6, n_dpc): 00,01,02,11,12,22
  int64_t n_cells;
  int n_dpc;
  int nc;
  const double* __restrict__ cgeo = nullptr;  // plan geometry (G scaled by any per-cell kappa)
};

__global__ void diag_kernel(DiagArgs a) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.n_cells;
       e += (int64_t)gridDim.x * blockDim.x) {
    double G[6];
    if (a.cgeo) {   // the apply's own metric (includes the stiffness scale and per-cell kappa)
#pragma unroll
      for (int i = 0; i < 6; ++i) G[i] = __ldg(a.cgeo + 8 * e + i);
    } else {
      int vid[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) vid[i] = __ldg(a.cells + 4 * e + i);
      Affine g;
      affine_from_vertices(load_vertex(a.verts, vid[0]), load_vertex(a.verts, vid[1]),
                           load_vertex(a.verts, vid[2]), load_vertex(a.verts, vid[3]), g);
      stiffness_metric(g, 1.0, G);
    }
    const int n = a.n_dpc;
    for (int j = 0; j < n; ++j) {
      const int dof = __ldg(a.dofs + e * n + j);
      if (dof < 0) continue;
      const double v = G[0] * __ldg(a.S + j) + 2.0 * G[1] * __ldg(a.S + n + j) +
                       2.0 * G[2] * __ldg(a.S + 2 * n + j) + G[3] * __ldg(a.S + 3 * n + j) +
                       2.0 * G[4] * __ldg(a.S + 4 * n + j) + G[5] * __ldg(a.S + 5 * n + j);
      for (int c = 0; c < a.nc; ++c) atomicAdd(a.diag + (int64_t)dof * a.nc + c, v);
    }
  }
}

__global__ void set_list_kernel(double* __restrict__ v, const int* __restrict__ list, int64_t n, double val) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v[list[i]] = val;
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sh[w] = v;
  __syncthreads();
  v = 0.0;
  if (threadIdx.x < (blockDim.x >> 5)) v = sh[threadIdx.x];
  if (w == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;  // valid in thread 0
}

// r = b, z = r / d, p = z, x = 0; rz0 += r.z, rr0 += r.r
__global__ void pcg_init_kernel(const double* __restrict__ b, const double* __restrict__ d,
                                double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                                double* __restrict__ p, int64_t n, double* rz, double* rr) {
  __shared__ double sh[32];
  double s1 = 0.0, s2 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = b[i], zi = ri / d[i];
    x[i] = 0.0;
    r[i] = ri;
    z[i] = zi;
    p[i] = zi;
    s1 += ri * zi;
    s2 += ri * ri;
  }
  s1 = block_sum(s1, sh);
  __syncthreads();
  s2 = block_sum(s2, sh);
  if (threadIdx.x == 0) {
    atomicAdd(rz, s1);
    atomicAdd(rr, s2);
  }
}

__global__ void dot_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s += a[i] * b[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) atomicAdd(out, s);
}

// alpha = rz[k] / pq[k]; x += alpha p; r -= alpha q; z = r / d; rz[k+1] += r.z; rr[k+1] += r.r
__global__ void pcg_update_kernel(const double* __restrict__ p, const double* __restrict__ q,
                                  const double* __restrict__ d, double* __restrict__ x, double* __restrict__ r,
                                  double* __restrict__ z, int64_t n, const double* rz_k, const double* pq_k,
                                  double* rz_next, double* rr_next) {
  __shared__ double sh[32];
  const double alpha = *pq_k != 0.0 ? *rz_k / *pq_k : 0.0;   // 0 at exact breakdown
  double s1 = 0.0, s2 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    const double zi = ri / d[i];
    r[i] = ri;
    z[i] = zi;
    s1 += ri * zi;
    s2 += ri * ri;
  }
  s1 = block_sum(s1, sh);
  __syncthreads();
  s2 = block_sum(s2, sh);
  if (threadIdx.x == 0) {
    atomicAdd(rz_next, s1);
    atomicAdd(rr_next, s2);
  }
}

// p = z + (rz[k+1] / rz[k]) p
__global__ void pcg_direction_kernel(const double* __restrict__ z, double* __restrict__ p, int64_t n,
                                     const double* rz_k, const double* rz_next) {
  const double beta = *rz_k != 0.0 ? *rz_next / *rz_k : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

// ---- fused iteration (single GPU, tensor cell engine): p.Ap comes out of the cell kernel as
// the sum of element energies (CellArgs::energy) and the x update and the zeroing of the
// next A p ride along with the search-direction update -- 11 vector passes per iteration
// instead of 14 (memset, dot, update, direction).

// r = b, z = r / d, p = z, x = 0, q = 0; rz0 += r.z, rr0 += r.r
__global__ void pcg_init_fused_kernel(const double* __restrict__ b, const double* __restrict__ d,
                                      double* __restrict__ x, double* __restrict__ r, double* __restrict__ z,
                                      double* __restrict__ p, double* __restrict__ q, int64_t n, double* rz,
                                      double* rr) {
  __shared__ double sh[32];
  double s1 = 0.0, s2 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = b[i], zi = ri / d[i];
    x[i] = 0.0;
    q[i] = 0.0;
    r[i] = ri;
    z[i] = zi;
    p[i] = zi;
    s1 += ri * zi;
    s2 += ri * ri;
  }
  s1 = block_sum(s1, sh);
  __syncthreads();
  s2 = block_sum(s2, sh);
  if (threadIdx.x == 0) {
    atomicAdd(rz, s1);
    atomicAdd(rr, s2);
  }
}

// alpha = rz[k] / pq[k]; r -= alpha q; z = r / d; rz[k+1] += r.z; rr[k+1] += r.r
__global__ void pcg_residual_kernel(const double* __restrict__ q, const double* __restrict__ d,
                                    double* __restrict__ r, double* __restrict__ z, int64_t n, const double* rz_k,
                                    const double* pq_k, double* rz_next, double* rr_next) {
  __shared__ double sh[32];
  const double alpha = *pq_k != 0.0 ? *rz_k / *pq_k : 0.0;   // 0 at exact breakdown
  double s1 = 0.0, s2 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double ri = r[i] - alpha * q[i];
    const double zi = ri / d[i];
    r[i] = ri;
    z[i] = zi;
    s1 += ri * zi;
    s2 += ri * ri;
  }
  s1 = block_sum(s1, sh);
  __syncthreads();
  s2 = block_sum(s2, sh);
  if (threadIdx.x == 0) {
    atomicAdd(rz_next, s1);
    atomicAdd(rr_next, s2);
  }
}

// x += alpha p (the old p), p = z + beta p, q = 0 (the next apply scatters into it)
__global__ void pcg_step_kernel(const double* __restrict__ z, double* __restrict__ p, double* __restrict__ x,
                                double* __restrict__ q, int64_t n, const double* rz_k, const double* pq_k,
                                const double* rz_next) {
  const double alpha = *pq_k != 0.0 ? *rz_k / *pq_k : 0.0, beta = *rz_k != 0.0 ? *rz_next / *rz_k : 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double pi = p[i];
    x[i] += alpha * pi;
    p[i] = z[i] + beta * pi;
    q[i] = 0.0;
  }
}

}  // namespace tmf
