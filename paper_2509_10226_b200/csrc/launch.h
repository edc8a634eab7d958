// Internal launcher interface between the C-ABI (capi.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace tmf {

struct CellArgs;
struct FaceArgs;
struct FaceGeoArgs;
struct CellGeoArgs;
struct BlockArgs;

struct CellLaunchInfo {
  int dmma_per_tile = 0;
  int64_t tiles = 0;
  int block = 0;
  int grid = 0;
  int smem = 0;
  int frag_doubles = 0;
  int table = 0;             // 0 = DMMA lane fragments (cell_kernel.cuh),
                             // 2 = reference-tensor fragments (cell_tensor_kernel.cuh)
  double flops_issued = 0;   // FP64 FMA*2 issued per launch (padding included)
};

struct FaceLaunchInfo {
  int nfrag = 0;            // fragments per (lf, code) combo
  int chunk = 0;            // batches per CTA chunk
  int dmma_per_batch = 0;
  int grid = 0;
};

// info != nullptr: only fill the launch description (no launch).
cudaError_t launch_cell(int n_dpc, int n_q, bool mass, bool dg, const CellArgs& a, int n_sm,
                        cudaStream_t st, CellLaunchInfo* info, bool* supported, int engine);
cudaError_t launch_face(int n_dpc, int n_qf, bool boundary, const FaceArgs& a, int n_sm,
                        cudaStream_t st, FaceLaunchInfo* info, bool* supported);
cudaError_t launch_face_geometry(bool boundary, const FaceGeoArgs& a, int n_sm, cudaStream_t st);
cudaError_t launch_cell_geometry(const CellGeoArgs& a, int n_sm, cudaStream_t st);
// CG block assembly (cell_block_kernel.cuh): cells per block for n_dpc (0 = no kernel),
// and the launch (host_tab: the M x 3 x n_dpc modal table, passed as a kernel parameter)
int block_cells_for(int n_dpc);
cudaError_t launch_cell_block(int n_dpc, const BlockArgs& a, const double* host_tab, cudaStream_t st);
// Clear y ahead of a CG cell kernel (zero_y_kernel: releases its dependents at once).  While
// tl_pdl is set on the calling thread the cell launchers launch with programmatic stream
// serialization, so the kernel's prologue overlaps the clear (common.cuh pdl_wait_prior_grid).
extern thread_local bool tl_pdl;
cudaError_t launch_zero(double* y, int64_t n, int n_sm, cudaStream_t st);
cudaError_t launch_fixup(const double* u, double* y, const int* list, int64_t n, int n_sm,
                         cudaStream_t st, double* energy = nullptr);

}  // namespace tmf
