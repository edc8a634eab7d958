// Cell-kernel dispatch, geometry and fix-up launchers (sm_100a).  The kernel
// instantiations live in cell_p{1,2,3,4}.cu and face_launch.cu.
#include <cuda_runtime.h>

#include "cell_kernel.cuh"
#include "launch.h"

namespace tmf {

cudaError_t cell_dispatch_4_4(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                              CellLaunchInfo* info, int engine);
cudaError_t cell_dispatch_4_5(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                              CellLaunchInfo* info, int engine);
cudaError_t cell_dispatch_10_14(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                              CellLaunchInfo* info, int engine);
cudaError_t cell_dispatch_10_15(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                              CellLaunchInfo* info, int engine);
cudaError_t cell_dispatch_20_35(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                              CellLaunchInfo* info, int engine);
cudaError_t cell_dispatch_4_1(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                              CellLaunchInfo* info, int engine);
cudaError_t cell_dispatch_10_4(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                              CellLaunchInfo* info, int engine);
cudaError_t cell_dispatch_20_10(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                              CellLaunchInfo* info, int engine);
cudaError_t cell_dispatch_35_20(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                              CellLaunchInfo* info, int engine);
cudaError_t cell_dispatch_35_70(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                              CellLaunchInfo* info, int engine);

cudaError_t launch_cell(int n_dpc, int n_q, bool mass, bool dg, const CellArgs& a, int n_sm,
                        cudaStream_t st, CellLaunchInfo* info, bool* supported, int engine) {
  *supported = true;
#define TMF_CELL(NN, QQ)   \
  if (n_dpc == NN && n_q == QQ) \
    return cell_dispatch_##NN##_##QQ(mass, dg, a, n_sm, st, info, engine);
  TMF_CELL(4, 4)
  TMF_CELL(4, 5)
  TMF_CELL(10, 14)
  TMF_CELL(10, 15)
  TMF_CELL(20, 35)
  TMF_CELL(35, 70)
  TMF_CELL(4, 1)
  TMF_CELL(10, 4)
  TMF_CELL(20, 10)
  TMF_CELL(35, 20)
#undef TMF_CELL
  *supported = false;
  return cudaSuccess;
}

cudaError_t launch_cell_geometry(const CellGeoArgs& a, int n_sm, cudaStream_t st) {
  cell_geometry_kernel<<<n_sm * 8, 256, 0, st>>>(a);
  return cudaGetLastError();
}

thread_local bool tl_pdl = false;

// y = 0 with 16-byte stores; the dependents (the cell kernel's prologue) start at once
__global__ void __launch_bounds__(256) zero_y_kernel(double* __restrict__ y, int64_t n) {
  pdl_release_dependents();
  const int64_t tid = (int64_t)blockIdx.x * 256 + threadIdx.x, nt = (int64_t)gridDim.x * 256;
  const int64_t head = (reinterpret_cast<uintptr_t>(y) & 8) ? 1 : 0;   // y is 8-byte aligned
  if (tid == 0 && head && n > 0) y[0] = 0.0;
  if (n <= head) return;
  double2* y2 = reinterpret_cast<double2*>(y + head);
  const int64_t n2 = (n - head) / 2;
  for (int64_t i = tid; i < n2; i += nt) y2[i] = make_double2(0.0, 0.0);
  if (tid == 0 && ((n - head) & 1)) y[n - 1] = 0.0;
}

cudaError_t launch_zero(double* y, int64_t n, int n_sm, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n / 2 + 1023) / 1024;   // >= 4 stores per thread on large vectors
  if (blocks > 8 * (int64_t)n_sm) blocks = 8 * (int64_t)n_sm;
  if (blocks < 1) blocks = 1;
  zero_y_kernel<<<(unsigned)blocks, 256, 0, st>>>(y, n);
  return cudaGetLastError();
}

cudaError_t launch_fixup(const double* u, double* y, const int* list, int64_t n, int n_sm,
                         cudaStream_t st, double* energy) {
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4 * n_sm) blocks = 4 * n_sm;
  dirichlet_fixup_kernel<<<(unsigned)blocks, 256, 0, st>>>(u, y, list, n, energy);
  return cudaGetLastError();
}

}  // namespace tmf
