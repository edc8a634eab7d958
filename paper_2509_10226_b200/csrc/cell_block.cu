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
  if (cudaError_t e = opt_in_smem(kern, 227 * 1024); e != cudaSuccess) return e;
  {
    static bool carve = false;   // the whole unified L1/shared array as shared memory
    if (!carve) {
      if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
          e != cudaSuccess)
        return e;
      carve = true;
    }
  }
  if (a.n_blocks == 0) return cudaSuccess;
  kern<<<(unsigned)a.n_blocks, C::BLOCK, smem, st>>>(a, T);
  return cudaGetLastError();
}

// Pipelined block-DMMA kernel: cells per block and CTA size per degree
template <int N>
struct PipeConfig;
template <>
struct PipeConfig<4> {
  static constexpr int M = 1, BLOCK = 256, B = 512;
};
template <>
struct PipeConfig<10> {
  static constexpr int M = 4, BLOCK = 256, B = 256;
};
template <>
struct PipeConfig<20> {
  static constexpr int M = 10, BLOCK = 256, B = 128;
};

int pipe_cells_for(int n_dpc) {
  switch (n_dpc) {
    case 4: return PipeConfig<4>::B;
    case 10: return PipeConfig<10>::B;
    case 20: return PipeConfig<20>::B;
    default: return 0;
  }
}

size_t pipe_smem_bytes(int n_dpc, int numax, int nvmax) {
  int M = 0;
  switch (n_dpc) {
    case 4: M = PipeConfig<4>::M; break;
    case 10: M = PipeConfig<10>::M; break;
    case 20: M = PipeConfig<20>::M; break;
    default: return 0;
  }
  int nfrag = 0;
  if (n_dpc == 4) nfrag = CellShape<4, 1, false>::NFRAG;
  if (n_dpc == 10) nfrag = CellShape<10, 4, false>::NFRAG;
  if (n_dpc == 20) nfrag = CellShape<20, 10, false>::NFRAG;
  (void)M;
  const BpipeLayout L{numax, nvmax, pipe_cells_for(n_dpc), n_dpc, (n_dpc + 3) & ~3, nfrag};
  return (size_t)L.total();
}

template <int N>
static cudaError_t launch_pipe_n(const BpipeArgs& a, int n_sm, cudaStream_t st) {
  using C = PipeConfig<N>;
  auto kern = cell_bpipe_kernel<N, C::M, C::BLOCK, C::B>;
  const size_t smem = pipe_smem_bytes(N, a.numax, a.nvmax);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if (cudaError_t e = opt_in_smem(kern, 227 * 1024); e != cudaSuccess) return e;
  {
    static bool carve = false;
    if (!carve) {
      if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
          e != cudaSuccess)
        return e;
      carve = true;
    }
  }
  if (a.n_blocks == 0) return cudaSuccess;
  int per_sm = 0;
  if (cudaError_t e = blocks_per_sm(kern, C::BLOCK, smem, &per_sm); e != cudaSuccess) return e;
  int64_t grid = (int64_t)n_sm * (per_sm < 1 ? 1 : per_sm);
  if (grid > a.n_blocks) grid = a.n_blocks;
  kern<<<(unsigned)grid, C::BLOCK, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_cell_bpipe(int n_dpc, const BpipeArgs& a, int n_sm, cudaStream_t st) {
  switch (n_dpc) {
    case 4: return launch_pipe_n<4>(a, n_sm, st);
    case 10: return launch_pipe_n<10>(a, n_sm, st);
    case 20: return launch_pipe_n<20>(a, n_sm, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_cell_block(int n_dpc, const BlockArgs& a, const double* host_tab, cudaStream_t st) {
  switch (n_dpc) {
    case 4: return launch_block_n<4>(a, host_tab, st);
    case 10: return launch_block_n<10>(a, host_tab, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace tmf
