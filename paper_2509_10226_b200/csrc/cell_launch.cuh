// Cell-kernel launchers: tuning variants and per-degree defaults of the DMMA
// (cell_kernel.cuh) and DFMA (cell_dfma_kernel.cuh) engines.  Each degree is
// instantiated in its own translation unit (cell_p*.cu) through TMF_CELL_TU so
// the kernels compile in parallel; kernels.cu dispatches on (n_dpc, n_q).
#pragma once
#include <cuda_runtime.h>

#include "cell_dfma_kernel.cuh"
#include "cell_kernel.cuh"
#include "cell_patch_kernel.cuh"
#include "cell_tensor_kernel.cuh"
#include "launch.h"
#include "launch_common.cuh"

namespace tmf {

template <int N, int Q, bool MASS, bool DG, int BLOCK, int MT, int MINB, bool PF = false, bool BLK = false,
          bool SKEW = false, bool PEER = false, int AS = 0>
static cudaError_t launch_cell_v(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info) {
  using S = CellShape<N, Q, MASS>;
  constexpr int MTE = MT ? MT : S::MT;
  // tables + the per-warp async rings
  constexpr int SMEM = S::SMEM + (AS > 0 ? AS * MTE * (S::KK * 32 + 64) * 8 * (BLOCK / 32) : 0);
  static_assert(SMEM <= 227 * 1024, "shared memory");
  auto kern = cell_apply_kernel<N, Q, MASS, DG, BLOCK, MT, MINB, PF, BLK, SKEW, PEER, AS>;
  if (cudaError_t e = opt_in_smem(kern, SMEM); e != cudaSuccess) return e;
  int per_sm = 0;
  cudaError_t e = blocks_per_sm(kern, BLOCK, SMEM, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t supertiles = ((a.n_cells + 8 * MTE - 1) / (8 * MTE)) * a.nc;
  int64_t blocks = (int64_t)n_sm * per_sm;
  const int64_t need = (supertiles + BLOCK / 32 - 1) / (BLOCK / 32);
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  if (info) {
    info->dmma_per_tile = S::DMMA_PER_TILE;
    info->tiles = supertiles * MTE;
    info->block = BLOCK;
    info->grid = (int)blocks;
    info->smem = SMEM;
    info->frag_doubles = S::NFRAG * 32;
    info->table = 0;
    info->flops_issued = (double)supertiles * MTE * S::DMMA_PER_TILE * 512.0;
    return cudaSuccess;
  }
  kern<<<(unsigned)blocks, BLOCK, SMEM, st>>>(a);
  return cudaGetLastError();
}

// Reference-tensor engine (cell_tensor_kernel.cuh)
template <int N, bool MASS, bool DG, int BLOCK, int MT, int MINB, bool PEER = false, bool PF = false>
static cudaError_t launch_cell_x(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info) {
  using S = TensorShape<N, MASS>;
  auto kern = cell_tensor_kernel<N, MASS, DG, BLOCK, MT, MINB, PEER, PF>;
  if (cudaError_t e = opt_in_smem(kern, S::SMEM); e != cudaSuccess) return e;
  int per_sm = 0;
  cudaError_t e = blocks_per_sm(kern, BLOCK, S::SMEM, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t supertiles = ((a.n_cells + 8 * MT - 1) / (8 * MT)) * a.nc;
  int64_t blocks = (int64_t)n_sm * per_sm;
  const int64_t need = (supertiles + BLOCK / 32 - 1) / (BLOCK / 32);
  if (blocks > need) blocks = need;
  if (blocks < 1) blocks = 1;
  if (info) {
    info->dmma_per_tile = S::DMMA_PER_TILE;
    info->tiles = supertiles * MT;
    info->block = BLOCK;
    info->grid = (int)blocks;
    info->smem = S::SMEM;
    info->frag_doubles = S::NFRAG * 32;
    info->table = 2;
    // DMMAs + the (6 | 7)-term contraction per output DoF
    info->flops_issued = (double)supertiles * MT * (S::DMMA_PER_TILE * 512.0 + 8.0 * S::KK * 4 * 2 * (MASS ? 7 : 6));
    return cudaSuccess;
  }
  if (a.n_cells == 0) return cudaSuccess;
  kern<<<(unsigned)blocks, BLOCK, S::SMEM, st>>>(a);
  return cudaGetLastError();
}

// P1 thread-per-cell kernel (cell_p1_thread_kernel): needs the plan's constant-gradient
// table (a.hP1, set when the P1 gradient tables are point-independent)
template <bool DG, int BLOCK, int MINB>
static cudaError_t launch_cell_p1(const CellArgs& a, int n_sm, cudaStream_t st) {
  if (a.n_cells == 0) return cudaSuccess;
  P1Tab T;
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < 4; ++i) T.a[k][i] = a.hP1[4 * k + i];
  T.w = a.hP1[12];
  auto kern = cell_p1_thread_kernel<DG, BLOCK, MINB>;
  int per_sm = 0;
  cudaError_t e = blocks_per_sm(kern, BLOCK, 0, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t need = (a.n_cells * a.nc + BLOCK - 1) / BLOCK;
  int64_t blocks = (int64_t)n_sm * per_sm;
  if (blocks > need) blocks = need;
  kern<<<(unsigned)blocks, BLOCK, 0, st>>>(a, T);
  return cudaGetLastError();
}

// variants: 0 = per-degree default; 1..7 = tuning (bench sweeps only)
template <int N, bool MASS, bool DG>
static cudaError_t launch_cell_xt(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info,
                                  int variant) {
  if (!DG && a.peer.u != nullptr && !info) {   // multi-GPU peer ghosts: the default shapes
    if (N <= 4) return launch_cell_x<N, MASS, DG, 768, 2, 1, true>(a, n_sm, st, info);
    if (N <= 20) return launch_cell_x<N, MASS, DG, 1024, 1, 1, true>(a, n_sm, st, info);
    return launch_cell_x<N, MASS, DG, 512, 2, 1, true>(a, n_sm, st, info);
  }
  if (variant == 1) return launch_cell_x<N, MASS, DG, 256, 1, 1>(a, n_sm, st, info);
  if (variant == 2) return launch_cell_x<N, MASS, DG, 512, 2, 1>(a, n_sm, st, info);
  if (variant == 3) return launch_cell_x<N, MASS, DG, 128, 2, 4>(a, n_sm, st, info);
  if (variant == 4) return launch_cell_x<N, MASS, DG, 256, 4, 1>(a, n_sm, st, info);
  if (variant == 5) return launch_cell_x<N, MASS, DG, 768, 2, 1>(a, n_sm, st, info);
  if (variant == 6) return launch_cell_x<N, MASS, DG, 1024, 1, 1>(a, n_sm, st, info);
  if (variant == 7) return launch_cell_x<N, MASS, DG, 256, 3, 1>(a, n_sm, st, info);
  if constexpr (N <= 10) {   // data prefetch (low degrees: latency-bound gathers)
    if (variant == 8) return launch_cell_x<N, MASS, DG, 768, 2, 1, false, true>(a, n_sm, st, info);
    if (variant == 9) return launch_cell_x<N, MASS, DG, 1024, 1, 1, false, true>(a, n_sm, st, info);
    if (variant == 10) return launch_cell_x<N, MASS, DG, 512, 2, 2, false, true>(a, n_sm, st, info);
    if (variant == 11) return launch_cell_x<N, MASS, DG, 256, 1, 6, false, true>(a, n_sm, st, info);
    if (variant == 12) return launch_cell_x<N, MASS, DG, 512, 1, 3, false, true>(a, n_sm, st, info);
    if (variant == 14) return launch_cell_x<N, MASS, DG, 256, 2, 4, false, true>(a, n_sm, st, info);
    if (N == 4 && !MASS && a.peer.u == nullptr && a.hP1 != nullptr && !info) {   // P1 thread per cell
      if (variant == 15) return launch_cell_p1<DG, 256, 4>(a, n_sm, st);
      if (variant == 7) return launch_cell_p1<DG, 512, 2>(a, n_sm, st);
    }
  }
  // per-degree defaults, measured on CG 48^3 reordered (tools/gpu_tensor1.sh, variants 0-7):
  //   P1 768 threads x 2 tiles 31.5 us (256 x 2: 34.6), P2 1024 x 1 65.0 us (67.8),
  //   P3 1024 x 1 132 us (135), P4 512 x 2 350 us (375)
  if (N <= 4) return launch_cell_x<N, MASS, DG, 768, 2, 1>(a, n_sm, st, info);
  if (N <= 10 && !MASS) return launch_cell_x<N, MASS, DG, 1024, 1, 1>(a, n_sm, st, info);
  if (N <= 10) return launch_cell_x<N, MASS, DG, 512, 2, 1>(a, n_sm, st, info);
  if (N <= 20) return launch_cell_x<N, MASS, DG, 1024, 1, 1>(a, n_sm, st, info);
  return launch_cell_x<N, MASS, DG, 512, 2, 1>(a, n_sm, st, info);
}

// DFMA engine (cell_dfma_kernel.cuh): one thread per MC cells, point-major tables.
// OVER: CTAs per SM slot launched (1 = persistent grid-stride; > 1 oversubscribes so
// the block scheduler refills SMs as CTAs finish)
template <int N, int Q, bool MASS, bool DG, int BLOCK, int MC, int MINB, int OVER = 1>
static cudaError_t launch_cell_d(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info) {
  using S = DfmaShape<N, Q, MASS>;
  constexpr int CH = BLOCK * MC;
  auto kern = cell_dfma_kernel<N, Q, MASS, DG, BLOCK, MC, MINB>;
  if (cudaError_t e = opt_in_smem(kern, S::SMEM); e != cudaSuccess) return e;
  if (info) {
    info->dmma_per_tile = 0;
    info->tiles = (a.n_cells + 7) / 8 * a.nc;
    info->block = BLOCK;
    info->smem = S::SMEM;
    info->frag_doubles = 2 * S::TAB;
    info->table = 1;
    info->flops_issued = 2.0 * a.n_cells * a.nc * Q * (2.0 * S::NC * N + 9 + (MASS ? 1 : 0));
    return cudaSuccess;
  }
  if (a.n_cells == 0) return cudaSuccess;
  int per_sm = 0;
  cudaError_t e = blocks_per_sm(kern, BLOCK, S::SMEM, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t chunks = ((a.n_cells + CH - 1) / CH) * a.nc;
  int64_t blocks = (int64_t)n_sm * per_sm * OVER;
  if (blocks > chunks) blocks = chunks;
  if (blocks < 1) blocks = 1;
  kern<<<(unsigned)blocks, BLOCK, S::SMEM, st>>>(a);
  return cudaGetLastError();
}

// CG warp-patch-local assembly (cell_patch_kernel.cuh); runs when the plan built
// patch records (a.pmeta), whatever the engine; uses the DFMA point-major tables
template <int N, int Q, int BLOCK, int MINB>
static cudaError_t launch_cell_p(const CellArgs& a, int n_sm, cudaStream_t st) {
  using S = PatchShape<N, Q>;
  auto kern = cell_patch_kernel<N, Q, BLOCK, MINB>;
  const size_t smem = S::smem_bytes(a.recmax, a.numax, BLOCK / 32);
  if (smem > 227 * 1024) return cudaErrorNotSupported;   // caller falls back to the global kernel
  if (cudaError_t e = opt_in_smem(kern, 227 * 1024); e != cudaSuccess) return e;
  if (a.n_cells == 0) return cudaSuccess;
  int per_sm = 0;
  cudaError_t e = blocks_per_sm(kern, BLOCK, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t warps = ((a.n_cells + S::CH - 1) / S::CH) * a.nc;
  int64_t blocks = (int64_t)n_sm * per_sm;
  const int64_t need = (warps + BLOCK / 32 - 1) / (BLOCK / 32);
  if (blocks > need) blocks = need;
  kern<<<(unsigned)blocks, BLOCK, smem, st>>>(a);
  return cudaGetLastError();
}

// DFMA variants (engine 2): 0 = per-degree default; 1..8 tuning (bench sweeps only)
template <int N, int Q, bool MASS, bool DG>
static cudaError_t launch_cell_dt(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info,
                                  int variant) {
  if (variant == 1) return launch_cell_d<N, Q, MASS, DG, 256, 1, 1>(a, n_sm, st, info);
  if (variant == 2) return launch_cell_d<N, Q, MASS, DG, 256, 2, 1>(a, n_sm, st, info);
  if (variant == 3) return launch_cell_d<N, Q, MASS, DG, 256, 1, 2>(a, n_sm, st, info);
  if (variant == 4) return launch_cell_d<N, Q, MASS, DG, 256, 1, 3>(a, n_sm, st, info);
  if (variant == 5) return launch_cell_d<N, Q, MASS, DG, 256, 1, 4>(a, n_sm, st, info);
  if (variant == 6) return launch_cell_d<N, Q, MASS, DG, 256, 2, 2>(a, n_sm, st, info);
  if (variant == 7) return launch_cell_d<N, Q, MASS, DG, 128, 1, 6>(a, n_sm, st, info);
  if (variant == 8) return launch_cell_d<N, Q, MASS, DG, 256, 1, 4, 4>(a, n_sm, st, info);
  if (N <= 4) return launch_cell_d<N, Q, MASS, DG, 256, 1, 4>(a, n_sm, st, info);
  return launch_cell_d<N, Q, MASS, DG, 256, 1, 3>(a, n_sm, st, info);
}

// variant: 0 = default; 1..3 = tuning variants of the CG kernel (bench sweeps only)
template <int N, int Q, bool MASS, bool DG>
static cudaError_t launch_cell_t(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info,
                                 int variant) {
  using S = CellShape<N, Q, MASS>;
  constexpr int BLOCK = S::SMEM > 96 * 1024 ? 512 : 256;
  if (!DG && a.peer.u != nullptr && !info) {   // multi-GPU peer ghosts: the default CTA shape
    if (N == 20 && !MASS) return launch_cell_v<N, Q, MASS, DG, 768, 0, 1, false, false, false, true>(a, n_sm, st, info);
    if (N == 35) return launch_cell_v<N, Q, MASS, DG, 640, 0, 1, false, false, false, true>(a, n_sm, st, info);
    return launch_cell_v<N, Q, MASS, DG, BLOCK, 0, 1, false, false, false, true>(a, n_sm, st, info);
  }
  if constexpr (Q < N) {   // modal tables: asynchronous gather ring (AS stages), default CTA shapes
    constexpr int DB = N == 20 ? 768 : N == 35 ? 512 : (N == 10 && DG) ? 512 : BLOCK;
    if (variant == 5) return launch_cell_v<N, Q, MASS, DG, DB, 0, 1, false, false, false, false, 3>(a, n_sm, st, info);
    if (variant == 6) return launch_cell_v<N, Q, MASS, DG, DB, 0, 1, false, false, false, false, 2>(a, n_sm, st, info);
    if (variant == 7) return launch_cell_v<N, Q, MASS, DG, DB, 0, 1, false, false, false, false, 4>(a, n_sm, st, info);
    if (variant == 9) return launch_cell_v<N, Q, MASS, DG, 1024, 0, 1>(a, n_sm, st, info);   // 64 registers, 32 warps
  }
  if (!DG && !MASS) {
    if (variant == 1) return launch_cell_v<N, Q, MASS, DG, BLOCK, 2, 1>(a, n_sm, st, info);
    if (variant == 2) return launch_cell_v<N, Q, MASS, DG, BLOCK, 1, (BLOCK == 256 ? 3 : 1)>(a, n_sm, st, info);
    if (variant == 3) return launch_cell_v<N, Q, MASS, DG, 128, 1, 4>(a, n_sm, st, info);
    if (variant == 4) return launch_cell_v<N, Q, MASS, DG, BLOCK, 0, 1, true>(a, n_sm, st, info);
    if (variant == 5) return launch_cell_v<N, Q, MASS, DG, BLOCK, 1, 1, true>(a, n_sm, st, info);
    if (variant == 6) return launch_cell_v<N, Q, MASS, DG, BLOCK, 3, 1>(a, n_sm, st, info);
    if (variant == 7) return launch_cell_v<N, Q, MASS, DG, 128, 2, 1>(a, n_sm, st, info);
    if (variant == 9) return launch_cell_v<N, Q, MASS, DG, 384, 0, 1>(a, n_sm, st, info);
    if (variant == 12) return launch_cell_v<N, Q, MASS, DG, 768, 1, 1>(a, n_sm, st, info);
  }
  // block-size variants for every kernel family (registers are capped by the bounds)
  if (variant == 8) return launch_cell_v<N, Q, MASS, DG, 640, 0, 1>(a, n_sm, st, info);
  if (variant == 10) return launch_cell_v<N, Q, MASS, DG, 768, 0, 1>(a, n_sm, st, info);
  if (variant == 11) return launch_cell_v<N, Q, MASS, DG, 512, 0, 1>(a, n_sm, st, info);
  if (variant == 14) {   // skewed GEMM1/D-action pipeline with the per-degree default CTA size
    if (N == 20 && !MASS) return launch_cell_v<N, Q, MASS, DG, 768, 0, 1, false, false, true>(a, n_sm, st, info);
    if (N == 35 && !DG) return launch_cell_v<N, Q, MASS, DG, 640, 0, 1, false, false, true>(a, n_sm, st, info);
    if (N == 10 && DG) return launch_cell_v<N, Q, MASS, DG, 512, 0, 1, false, false, true>(a, n_sm, st, info);
    return launch_cell_v<N, Q, MASS, DG, BLOCK, 0, 1, false, false, true>(a, n_sm, st, info);
  }
  if (variant == 15) {   // data prefetch (next tile's u and G) with a CTA size that leaves the registers
    if (N == 20 && !MASS) return launch_cell_v<N, Q, MASS, DG, 640, 0, 1, true>(a, n_sm, st, info);
    if (N == 35 && !DG) return launch_cell_v<N, Q, MASS, DG, 512, 0, 1, true>(a, n_sm, st, info);
    if (N == 10 && DG) return launch_cell_v<N, Q, MASS, DG, 384, 0, 1, true>(a, n_sm, st, info);
    return launch_cell_v<N, Q, MASS, DG, BLOCK, 0, 1, true>(a, n_sm, st, info);
  }
  if (variant == 13) {   // blocked tile runs with the per-degree default CTA size
    if (N == 20 && !MASS) return launch_cell_v<N, Q, MASS, DG, 768, 0, 1, false, true>(a, n_sm, st, info);
    if (N == 35 && !DG) return launch_cell_v<N, Q, MASS, DG, 640, 0, 1, false, true>(a, n_sm, st, info);
    if (N == 10 && DG) return launch_cell_v<N, Q, MASS, DG, 512, 0, 1, false, true>(a, n_sm, st, info);
    return launch_cell_v<N, Q, MASS, DG, BLOCK, 0, 1, false, true>(a, n_sm, st, info);
  }
  // One large CTA per SM (a single staged table copy, more warps than the smem-limited
  // default allows), measured with tools/quick_bench.py variants 8/10/11:
  //   P3 (CG and DG) 768 threads: -5.6 % / -5 %;  CG P4 640: -1.4 %;
  //   DG P2 512: -26 %, Helmholtz P2 512: -17 %;  CG P2 keeps 2 tiles per warp at 256.
  //   (the skewed GEMM1/D-action pipeline, variant 14, helped CG P3 by 2.7 % before
  //   the remainder-point group; with it the plain loop is 5 % faster)
  //   modal tables (Q = M < N, tools/gpu_modal1.sh): P4 512 threads 0.268 ms (640: 0.306),
  //   P3 768 0.1075 ms, P2 256 x 2 tiles 0.0516 ms
  if (N == 20 && !MASS) return launch_cell_v<N, Q, MASS, DG, 768, 0, 1>(a, n_sm, st, info);
  //   P4 modal with the 2-stage async gather ring (variant 6): 48^3 0.276 -> 0.253 ms
  //   (unordered), 0.267 -> 0.245 (reordered); P2 / P3 lose 5-8 % with any ring
  if constexpr (N == 35 && Q < N) return launch_cell_v<N, Q, MASS, DG, 512, 0, 1, false, false, false, false, 2>(a, n_sm, st, info);
  if (N == 35 && !DG) return launch_cell_v<N, Q, MASS, DG, 640, 0, 1>(a, n_sm, st, info);
  if (N == 10 && DG) return launch_cell_v<N, Q, MASS, DG, 512, 0, 1>(a, n_sm, st, info);
  return launch_cell_v<N, Q, MASS, DG, BLOCK, 0, 1>(a, n_sm, st, info);
}

// engine: 0 = per-degree default, 1 = DMMA quadrature points (cell_kernel.cuh), 2 = DFMA
// (cell_dfma_kernel.cuh), 3 = DMMA reference tensor (cell_tensor_kernel.cuh)
template <int N, int Q>
static cudaError_t cell_variant(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                                CellLaunchInfo* info, int variant, int engine) {
  if constexpr (N <= 20) {   // CG warp-patch-local assembly (32-cell patches)
    if (!dg && info) info->patch_cells = PatchShape<N, Q>::CH;
    if (!dg && !info && a.pmeta) {
      // variants (bench sweeps): CTA size / minimum CTAs per SM (register cap)
      cudaError_t e;
      if (variant == 1) e = launch_cell_p<N, Q, 128, 4>(a, n_sm, st);
      else if (variant == 2) e = launch_cell_p<N, Q, 128, 8>(a, n_sm, st);
      else if (variant == 3) e = launch_cell_p<N, Q, 256, 2>(a, n_sm, st);
      else if (variant == 4) e = launch_cell_p<N, Q, 256, 3>(a, n_sm, st);
      else if (variant == 5) e = launch_cell_p<N, Q, 64, 12>(a, n_sm, st);
      else if (variant == 6) e = launch_cell_p<N, Q, 128, 2>(a, n_sm, st);
      else if (N <= 4) e = launch_cell_p<N, Q, 128, 6>(a, n_sm, st);
      else if (N <= 10) e = launch_cell_p<N, Q, 128, 4>(a, n_sm, st);
      else e = launch_cell_p<N, Q, 128, 2>(a, n_sm, st);
      if (e != cudaErrorNotSupported) return e;
      // patch records too large for shared memory (tiny or unordered meshes)
      CellArgs g = a;
      g.pmeta = nullptr;
      return cell_variant<N, Q>(mass, dg, g, n_sm, st, info, 0, engine);
    }
  }
  // default: the reference-tensor engine (measured 1.2-2.0x faster than the quadrature-point
  // DMMA engine at P1-P4, tools/gpu_tensor1.sh; DFMA was P1 ~= DMMA, P2 +20 %, tools/gpu_dfma1.sh)
  if (engine == 0) engine = 3;
  if (engine == 3) {
    if (!dg) return launch_cell_xt<N, false, false>(a, n_sm, st, info, variant);
    if (mass) return launch_cell_xt<N, true, true>(a, n_sm, st, info, variant);
    return launch_cell_xt<N, false, true>(a, n_sm, st, info, variant);
  }
  if constexpr (N <= 20) {   // P4 rows do not fit the DFMA register budget
    if (engine == 2) {
      if (!dg) return launch_cell_dt<N, Q, false, false>(a, n_sm, st, info, variant);
      if (mass) return launch_cell_dt<N, Q, true, true>(a, n_sm, st, info, variant);
      return launch_cell_dt<N, Q, false, true>(a, n_sm, st, info, variant);
    }
  }
  if (!dg) return launch_cell_t<N, Q, false, false>(a, n_sm, st, info, variant);
  if (mass) return launch_cell_t<N, Q, true, true>(a, n_sm, st, info, variant);
  return launch_cell_t<N, Q, false, true>(a, n_sm, st, info, variant);
}

#define TMF_CELL_TU(NN, QQ)                                                                        \
  cudaError_t cell_dispatch_##NN##_##QQ(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st, \
                                        CellLaunchInfo* info, int variant, int engine) {             \
    return cell_variant<NN, QQ>(mass, dg, a, n_sm, st, info, variant, engine);                        \
  }

}  // namespace tmf
