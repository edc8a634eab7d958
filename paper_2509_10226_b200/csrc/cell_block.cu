// Block-assembly cell kernel launchers (cell_block_kernel.cuh), P1-P3 CG Laplace.
#include <cuda_runtime.h>

#include <cstring>

#include "cell_block_kernel.cuh"
#include "launch.h"
#include "launch_common.cuh"

namespace tmf {

// Cells per block and CTA shape per degree: B = BLOCK * CPT cells, one thread per cell
// (CPT cells per thread at P1, whose per-cell work is small).
template <int N>
struct BlockConfig;
template <>
struct BlockConfig<4> {
  static constexpr int M = 1, BLOCK = 256, CPT = 2, MINB = 4;
};
template <>
struct BlockConfig<10> {
  static constexpr int M = 4, BLOCK = 256, CPT = 1, MINB = 4;
};


int block_cells_for(int n_dpc) {
  switch (n_dpc) {
    case 4: return BlockConfig<4>::BLOCK * BlockConfig<4>::CPT;
    case 10: return BlockConfig<10>::BLOCK * BlockConfig<10>::CPT;
    // P3 (M = 10, N = 20): the thread-per-cell DFMA form needs ~220 registers (measured
    // 2.4x slower than the DMMA modal tile kernel at 48^3); not used
    default: return 0;
  }
}

template <int N>
static cudaError_t launch_block_n(const BlockArgs& a, const double* tab, cudaStream_t st) {
  using C = BlockConfig<N>;
  constexpr int B = C::BLOCK * C::CPT;
  BlockTab<N, C::M> T;
  std::memcpy(T.e, tab, sizeof(T.e));
  auto kern = cell_block_kernel<N, C::M, C::BLOCK, C::CPT, C::MINB>;
  const size_t smem = block_smem_bytes(N, B, a.numax, a.nvmax);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  // the whole unified L1 / shared array as shared memory (several CTAs per SM)
  if (cudaError_t e = opt_in_smem(kern, 227 * 1024, true); e != cudaSuccess) return e;
  if (a.n_blocks == 0) return cudaSuccess;
  return launch_kernel(kern, (unsigned)a.n_blocks, C::BLOCK, smem, st, a, T);
}

cudaError_t launch_cell_block(int n_dpc, const BlockArgs& a, const double* host_tab, cudaStream_t st) {
  switch (n_dpc) {
    case 4: return launch_block_n<4>(a, host_tab, st);
    case 10: return launch_block_n<10>(a, host_tab, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tmf
