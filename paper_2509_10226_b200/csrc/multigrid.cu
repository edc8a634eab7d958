// p- and c-multigrid building blocks (the paper's solver layer PAPER.md:423-436,
// SPEC.md:494-565; the reference ships none of it): degree-transfer operators between
// two CG spaces (or a DG and a CG space) on the same mesh and the fused Chebyshev-Jacobi
// smoother update.
//
// Prolongation P: the coarse (degree pc) function interpolated at the fine (degree pf)
// nodes, cell by cell: x_f[i] = sum_j P_loc[i, j] x_c[cdofs[j]], P_loc[i, j] =
// phi^c_j(node^f_i).  A fine DoF shared by several cells is written by exactly ONE of
// them (its owner = the first cell in cell order that contains it), so prolongation
// needs no atomics, is deterministic, and restriction R = P^T (the exact transpose of
// the global interpolation matrix) sums every fine row once:
//   r_c[cdofs[j]] += sum_{i owned by e} P_loc[i, j] r_f[fdofs[i]]     (fp64 RED)
// c-transfer (DG fine space over the CG space of the same degree, P_loc = I): every DG
// DoF belongs to one cell, prolongation copies the CG value of a node into each cell's
// DG DoF and restriction sums the DG values of a node into its CG DoF.
// Dirichlet DoFs: fine ones are written as 0 (overwrite) / left alone (add) and never
// restricted; coarse ones are gathered as 0 and never scattered (their rows are
// identity rows of the coarse operator and stay zero in the correction).
// All kernels are memory-bound thread-per-cell loops (a few % of one apply).
#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/tetmf_b200.h"

extern "C" int tmf_internal_set_error(int code, const char* msg);

namespace {

constexpr int kNotOwned = INT_MIN;

int mg_fail(int code, const std::string& m) { return tmf_internal_set_error(code, m.c_str()); }

#define MG_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return mg_fail(TMF_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));    \
  } while (0)

// fdofs: fine DoF id (owned, free), ~id (owned, Dirichlet) or kNotOwned
// cdofs: coarse DoF id, or ~id for a coarse Dirichlet DoF
template <int NC, typename T>
__global__ void prolongate_kernel(const int* __restrict__ fdofs, const int* __restrict__ cdofs,
                                  const T* __restrict__ Pg, int nf, int64_t n_cells,
                                  const T* __restrict__ xc, T* __restrict__ xf, int add) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sP = reinterpret_cast<T*>(smraw);
  for (int i = threadIdx.x; i < nf * NC; i += blockDim.x) sP[i] = Pg[i];
  __syncthreads();
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_cells;
       c += (int64_t)gridDim.x * blockDim.x) {
    T v[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int g = __ldg(cdofs + c * NC + j);
      v[j] = g >= 0 ? __ldg(xc + g) : T(0);
    }
    for (int i = 0; i < nf; ++i) {
      const int f = __ldg(fdofs + c * nf + i);
      if (f == kNotOwned) continue;
      if (f < 0) {
        if (!add) xf[~f] = T(0);
        continue;
      }
      T s = T(0);
#pragma unroll
      for (int j = 0; j < NC; ++j) s = fma(sP[i * NC + j], v[j], s);
      xf[f] = add ? xf[f] + s : s;
    }
  }
}

template <int NC, typename T>
__global__ void restrict_kernel(const int* __restrict__ fdofs, const int* __restrict__ cdofs,
                                const T* __restrict__ Pg, int nf, int64_t n_cells,
                                const T* __restrict__ rf, T* __restrict__ rc) {
  extern __shared__ __align__(16) unsigned char smraw[];
  T* sP = reinterpret_cast<T*>(smraw);
  for (int i = threadIdx.x; i < nf * NC; i += blockDim.x) sP[i] = Pg[i];
  __syncthreads();
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_cells;
       c += (int64_t)gridDim.x * blockDim.x) {
    T acc[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) acc[j] = T(0);
    for (int i = 0; i < nf; ++i) {
      const int f = __ldg(fdofs + c * nf + i);
      if (f < 0) continue;   // not owned, or Dirichlet
      const T r = __ldg(rf + f);
#pragma unroll
      for (int j = 0; j < NC; ++j) acc[j] = fma(sP[i * NC + j], r, acc[j]);
    }
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int g = __ldg(cdofs + c * NC + j);
      if (g >= 0 && acc[j] != T(0)) atomicAdd(rc + g, acc[j]);
    }
  }
}

// first == 1 (x = 0 on entry, ax unused):  d = c2 D^-1 b;  x = d
// otherwise:                               d = c1 d + c2 D^-1 (b - ax);  x += d
template <typename T>
__global__ void chebyshev_kernel(int64_t n, const T* __restrict__ ax, const T* __restrict__ b,
                                 const T* __restrict__ dinv, T* __restrict__ x,
                                 T* __restrict__ d, T c1, T c2, int first) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (first) {
      const T di = c2 * dinv[i] * b[i];
      d[i] = di;
      x[i] = di;
    } else {
      const T di = c1 * d[i] + c2 * dinv[i] * (b[i] - ax[i]);
      d[i] = di;
      x[i] += di;
    }
  }
}

template <typename T>
__global__ void axpby_kernel(int64_t n, T alpha, const T* __restrict__ x, T beta,
                             const T* __restrict__ y, T* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = alpha * x[i] + beta * y[i];
}

// Point transfers (h-coarsening onto a non-nested coarse mesh): fine row i has K coarse
// entries (idx[i*K + k], w[i*K + k]); fine rows ~i < 0 are Dirichlet (0 / untouched),
// coarse entries ~c < 0 are Dirichlet columns (skipped).
template <int K, typename T>
__global__ void point_prolongate_kernel(const int* __restrict__ rows, const int* __restrict__ idx,
                                        const T* __restrict__ w, int64_t n, const T* __restrict__ xc,
                                        T* __restrict__ xf, int add) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int f = rows[i];
    if (f < 0) {
      if (!add) xf[~f] = T(0);
      continue;
    }
    T s = T(0);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = __ldg(idx + i * K + k);
      if (c >= 0) s = fma(__ldg(w + i * K + k), __ldg(xc + c), s);
    }
    xf[f] = add ? xf[f] + s : s;
  }
}

template <int K, typename T>
__global__ void point_restrict_kernel(const int* __restrict__ rows, const int* __restrict__ idx,
                                      const T* __restrict__ w, int64_t n, const T* __restrict__ rf,
                                      T* __restrict__ rc) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int f = rows[i];
    if (f < 0) continue;
    const T r = __ldg(rf + f);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int c = __ldg(idx + i * K + k);
      const T v = __ldg(w + i * K + k) * r;
      if (c >= 0 && v != T(0)) atomicAdd(rc + c, v);
    }
  }
}

int sm_count(int dev) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

}  // namespace

struct tmf_transfer {
  int device = 0;
  int sms = 148;
  int64_t n_cells = 0;
  int nf = 0, nc = 0;
  int64_t n_fine = 0, n_coarse = 0;
  int* fdofs = nullptr;
  int* cdofs = nullptr;
  double* P = nullptr;
  float* P32 = nullptr;
  // point mode (tmf_transfer_create_points): n_cells = fine rows, nc = entries per row
  bool points = false;
  double* W = nullptr;
  float* W32 = nullptr;
};

extern "C" {

int tmf_transfer_create(const tmf_transfer_desc* d, tmf_transfer** out) {
  if (!d || !out) return mg_fail(TMF_EINVAL, "null descriptor/output");
  *out = nullptr;
  if (d->n_cells <= 0) return mg_fail(TMF_EINVAL, "empty mesh");
  if (!d->fine_cell_dofs || !d->coarse_cell_dofs || !d->interp)
    return mg_fail(TMF_EINVAL, "missing dof maps / interpolation matrix");
  if (d->n_coarse_dpc != 4 && d->n_coarse_dpc != 10 && d->n_coarse_dpc != 20 && d->n_coarse_dpc != 35)
    return mg_fail(TMF_EINVAL, "coarse space must be P1-P4 (4/10/20/35 DoFs per cell)");
  if (d->n_fine_dpc < d->n_coarse_dpc || d->n_fine_dpc > 35)
    return mg_fail(TMF_EINVAL, "fine space needs at least as many DoFs per cell as the coarse one (<= 35)");
  if (d->n_fine_dofs <= 0 || d->n_coarse_dofs <= 0 || d->n_fine_dofs >= INT_MAX)
    return mg_fail(TMF_EINVAL, "bad DoF counts");
  const int64_t n = d->n_cells;
  const int nf = d->n_fine_dpc, nc = d->n_coarse_dpc;
  // owners: first cell (in cell order) that contains the fine DoF
  std::vector<int> f(n * nf), c(n * nc);
  std::vector<char> seen(d->n_fine_dofs, 0);
  for (int64_t e = 0; e < n; ++e)
    for (int i = 0; i < nf; ++i) {
      const int g = d->fine_cell_dofs[e * nf + i];
      if (g < 0 || g >= d->n_fine_dofs) return mg_fail(TMF_EINVAL, "fine DoF index out of range");
      if (seen[g]) {
        f[e * nf + i] = kNotOwned;
        continue;
      }
      seen[g] = 1;
      f[e * nf + i] = (d->fine_dirichlet && d->fine_dirichlet[g]) ? ~g : g;
    }
  for (int64_t e = 0; e < n; ++e)
    for (int j = 0; j < nc; ++j) {
      const int g = d->coarse_cell_dofs[e * nc + j];
      if (g < 0 || g >= d->n_coarse_dofs) return mg_fail(TMF_EINVAL, "coarse DoF index out of range");
      c[e * nc + j] = (d->coarse_dirichlet && d->coarse_dirichlet[g]) ? ~g : g;
    }
  for (int64_t g = 0; g < d->n_fine_dofs; ++g)
    if (!seen[g]) return mg_fail(TMF_EINVAL, "a fine DoF belongs to no cell");
  MG_CUDA(cudaSetDevice(d->device));
  auto* t = new tmf_transfer();
  t->device = d->device;
  t->sms = sm_count(d->device);
  t->n_cells = n;
  t->nf = nf;
  t->nc = nc;
  t->n_fine = d->n_fine_dofs;
  t->n_coarse = d->n_coarse_dofs;
  cudaError_t e = cudaMalloc(&t->fdofs, f.size() * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&t->cdofs, c.size() * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&t->P, (size_t)nf * nc * sizeof(double));
  if (e == cudaSuccess) e = cudaMemcpy(t->fdofs, f.data(), f.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(t->cdofs, c.data(), c.size() * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(t->P, d->interp, (size_t)nf * nc * sizeof(double), cudaMemcpyHostToDevice);
  std::vector<float> p32(d->interp, d->interp + (size_t)nf * nc);
  if (e == cudaSuccess) e = cudaMalloc(&t->P32, p32.size() * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(t->P32, p32.data(), p32.size() * sizeof(float), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    tmf_transfer_destroy(t);
    return mg_fail(TMF_ECUDA, std::string("transfer upload: ") + cudaGetErrorString(e));
  }
  *out = t;
  return TMF_OK;
}

int tmf_transfer_destroy(tmf_transfer* t) {
  if (!t) return TMF_OK;
  cudaSetDevice(t->device);
  cudaFree(t->fdofs);
  cudaFree(t->cdofs);
  cudaFree(t->P);
  cudaFree(t->P32);
  cudaFree(t->W);
  cudaFree(t->W32);
  delete t;
  return TMF_OK;
}

}  // extern "C"

namespace {

template <typename T>
int prolongate_t(tmf_transfer* t, const T* Pd, const T* xc, T* xf, int add, void* stream) {
  if (!t || !xc || !xf) return mg_fail(TMF_EINVAL, "null argument");
  MG_CUDA(cudaSetDevice(t->device));
  const cudaStream_t st = (cudaStream_t)stream;
  const int block = 256;
  int64_t grid = (t->n_cells + block - 1) / block;
  if (grid > (int64_t)t->sms * 16) grid = (int64_t)t->sms * 16;
  if (t->points) {
    point_prolongate_kernel<4, T><<<(unsigned)grid, block, 0, st>>>(t->fdofs, t->cdofs, Pd, t->n_cells, xc, xf, add);
    MG_CUDA(cudaGetLastError());
    return TMF_OK;
  }
  const size_t smem = (size_t)t->nf * t->nc * sizeof(T);
  const unsigned g = (unsigned)grid;
  switch (t->nc) {
    case 4: prolongate_kernel<4, T><<<g, block, smem, st>>>(t->fdofs, t->cdofs, Pd, t->nf, t->n_cells, xc, xf, add); break;
    case 10: prolongate_kernel<10, T><<<g, block, smem, st>>>(t->fdofs, t->cdofs, Pd, t->nf, t->n_cells, xc, xf, add); break;
    case 20: prolongate_kernel<20, T><<<g, block, smem, st>>>(t->fdofs, t->cdofs, Pd, t->nf, t->n_cells, xc, xf, add); break;
    default: prolongate_kernel<35, T><<<g, block, smem, st>>>(t->fdofs, t->cdofs, Pd, t->nf, t->n_cells, xc, xf, add);
  }
  MG_CUDA(cudaGetLastError());
  return TMF_OK;
}

template <typename T>
int restrict_t(tmf_transfer* t, const T* Pd, const T* rf, T* rc, void* stream) {
  if (!t || !rf || !rc) return mg_fail(TMF_EINVAL, "null argument");
  MG_CUDA(cudaSetDevice(t->device));
  const cudaStream_t st = (cudaStream_t)stream;
  MG_CUDA(cudaMemsetAsync(rc, 0, t->n_coarse * sizeof(T), st));
  const int block = 256;
  int64_t grid = (t->n_cells + block - 1) / block;
  if (grid > (int64_t)t->sms * 16) grid = (int64_t)t->sms * 16;
  if (t->points) {
    point_restrict_kernel<4, T><<<(unsigned)grid, block, 0, st>>>(t->fdofs, t->cdofs, Pd, t->n_cells, rf, rc);
    MG_CUDA(cudaGetLastError());
    return TMF_OK;
  }
  const size_t smem = (size_t)t->nf * t->nc * sizeof(T);
  const unsigned g = (unsigned)grid;
  switch (t->nc) {
    case 4: restrict_kernel<4, T><<<g, block, smem, st>>>(t->fdofs, t->cdofs, Pd, t->nf, t->n_cells, rf, rc); break;
    case 10: restrict_kernel<10, T><<<g, block, smem, st>>>(t->fdofs, t->cdofs, Pd, t->nf, t->n_cells, rf, rc); break;
    case 20: restrict_kernel<20, T><<<g, block, smem, st>>>(t->fdofs, t->cdofs, Pd, t->nf, t->n_cells, rf, rc); break;
    default: restrict_kernel<35, T><<<g, block, smem, st>>>(t->fdofs, t->cdofs, Pd, t->nf, t->n_cells, rf, rc);
  }
  MG_CUDA(cudaGetLastError());
  return TMF_OK;
}

template <typename T>
int chebyshev_t(int64_t n, const T* ax, const T* b, const T* dinv, T* x, T* d, T c1, T c2, void* stream) {
  if (n < 0 || !b || !dinv || !x || !d) return mg_fail(TMF_EINVAL, "bad argument");
  int dev = 0;
  MG_CUDA(cudaGetDevice(&dev));
  chebyshev_kernel<T><<<sm_count(dev) * 4, 512, 0, (cudaStream_t)stream>>>(n, ax, b, dinv, x, d, c1, c2,
                                                                            ax == nullptr ? 1 : 0);
  MG_CUDA(cudaGetLastError());
  return TMF_OK;
}

template <typename T>
int axpby_t(int64_t n, T alpha, const T* x, T beta, const T* y, T* out, void* stream) {
  if (n < 0 || !x || !y || !out) return mg_fail(TMF_EINVAL, "bad argument");
  int dev = 0;
  MG_CUDA(cudaGetDevice(&dev));
  axpby_kernel<T><<<sm_count(dev) * 4, 512, 0, (cudaStream_t)stream>>>(n, alpha, x, beta, y, out);
  MG_CUDA(cudaGetLastError());
  return TMF_OK;
}

}  // namespace

extern "C" {

int tmf_prolongate(tmf_transfer* t, const double* xc, double* xf, int add, void* stream) {
  return prolongate_t<double>(t, t ? (t->points ? t->W : t->P) : nullptr, xc, xf, add, stream);
}
int tmf_restrict(tmf_transfer* t, const double* rf, double* rc, void* stream) {
  return restrict_t<double>(t, t ? (t->points ? t->W : t->P) : nullptr, rf, rc, stream);
}
int tmf_prolongate_f32(tmf_transfer* t, const float* xc, float* xf, int add, void* stream) {
  return prolongate_t<float>(t, t ? (t->points ? t->W32 : t->P32) : nullptr, xc, xf, add, stream);
}
int tmf_restrict_f32(tmf_transfer* t, const float* rf, float* rc, void* stream) {
  return restrict_t<float>(t, t ? (t->points ? t->W32 : t->P32) : nullptr, rf, rc, stream);
}

int tmf_transfer_create_points(const tmf_point_transfer_desc* d, tmf_transfer** out) {
  if (!d || !out) return mg_fail(TMF_EINVAL, "null descriptor/output");
  *out = nullptr;
  if (d->n_fine_dofs <= 0 || d->n_coarse_dofs <= 0 || d->n_fine_dofs >= INT_MAX || d->n_coarse_dofs >= INT_MAX)
    return mg_fail(TMF_EINVAL, "bad DoF counts");
  if (d->entries_per_row != 4) return mg_fail(TMF_EINVAL, "point transfers take 4 coarse entries per fine row");
  if (!d->coarse_index || !d->weights) return mg_fail(TMF_EINVAL, "missing coarse indices / weights");
  const int64_t n = d->n_fine_dofs;
  std::vector<int> rows(n), idx(n * 4);
  std::vector<float> w32(n * 4);
  for (int64_t i = 0; i < n; ++i) {
    rows[i] = (d->fine_dirichlet && d->fine_dirichlet[i]) ? ~(int)i : (int)i;
    for (int k = 0; k < 4; ++k) {
      const int c = d->coarse_index[i * 4 + k];
      if (c < 0 || c >= d->n_coarse_dofs) return mg_fail(TMF_EINVAL, "coarse index out of range");
      idx[i * 4 + k] = (d->coarse_dirichlet && d->coarse_dirichlet[c]) ? ~c : c;
      w32[i * 4 + k] = (float)d->weights[i * 4 + k];
    }
  }
  MG_CUDA(cudaSetDevice(d->device));
  auto* t = new tmf_transfer();
  t->points = true;
  t->device = d->device;
  t->sms = sm_count(d->device);
  t->n_cells = n;
  t->nf = 1;
  t->nc = 4;
  t->n_fine = n;
  t->n_coarse = d->n_coarse_dofs;
  cudaError_t e = cudaMalloc(&t->fdofs, n * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&t->cdofs, n * 4 * sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&t->W, n * 4 * sizeof(double));
  if (e == cudaSuccess) e = cudaMalloc(&t->W32, n * 4 * sizeof(float));
  if (e == cudaSuccess) e = cudaMemcpy(t->fdofs, rows.data(), n * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(t->cdofs, idx.data(), n * 4 * sizeof(int), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(t->W, d->weights, n * 4 * sizeof(double), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(t->W32, w32.data(), n * 4 * sizeof(float), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    tmf_transfer_destroy(t);
    return mg_fail(TMF_ECUDA, std::string("point transfer upload: ") + cudaGetErrorString(e));
  }
  *out = t;
  return TMF_OK;
}
int tmf_chebyshev_step(int64_t n, const double* ax, const double* b, const double* dinv, double* x,
                       double* d, double c1, double c2, void* stream) {
  return chebyshev_t<double>(n, ax, b, dinv, x, d, c1, c2, stream);
}
int tmf_chebyshev_step_f32(int64_t n, const float* ax, const float* b, const float* dinv, float* x,
                           float* d, float c1, float c2, void* stream) {
  return chebyshev_t<float>(n, ax, b, dinv, x, d, c1, c2, stream);
}
int tmf_vec_axpby(int64_t n, double alpha, const double* x, double beta, const double* y, double* out,
                  void* stream) {
  return axpby_t<double>(n, alpha, x, beta, y, out, stream);
}
int tmf_vec_axpby_f32(int64_t n, float alpha, const float* x, float beta, const float* y, float* out,
                      void* stream) {
  return axpby_t<float>(n, alpha, x, beta, y, out, stream);
}

}  // extern "C"
