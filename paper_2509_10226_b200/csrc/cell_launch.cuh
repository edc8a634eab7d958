// Cell-kernel launchers: the per-degree CTA shapes of the DMMA point-loop kernel
// (cell_kernel.cuh: n_q quadrature points, or the M exact modes of the modal form) and
// of the reference-tensor kernel (cell_tensor_kernel.cuh).  Each degree is instantiated
// in its own translation unit (cell_p*.cu) through TMF_CELL_TU so the kernels compile
// in parallel; kernels.cu dispatches on (n_dpc, n_q).
#pragma once
#include <cuda_runtime.h>

#include "cell_kernel.cuh"
#include "cell_tensor_kernel.cuh"
#include "launch.h"
#include "launch_common.cuh"

namespace tmf {

// Persistent grid: n_sm x (resident CTAs per SM), capped by the work.
template <typename K>
static cudaError_t persistent_grid(K kern, int block, int smem, int64_t warps_of_work, int n_sm, int64_t* out) {
  int per_sm = 0;
  cudaError_t e = blocks_per_sm(kern, block, smem, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)n_sm * per_sm;
  const int64_t need = (warps_of_work + block / 32 - 1) / (block / 32);
  if (blocks > need) blocks = need;
  *out = blocks < 1 ? 1 : blocks;
  return cudaSuccess;
}

// MT_: 8-cell tiles per warp iteration sharing every B-fragment load (0 = CellShape default)
template <int N, int Q, bool MASS, bool DG, int BLOCK, bool PEER = false, int AS = 0, int MT_ = 0, bool MM = false,
          bool GS = false>
static cudaError_t launch_cell_v(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info) {
  using S = CellShape<N, Q, MASS, MM>;
  constexpr int MT = MT_ ? MT_ : S::MT;
  // tables + the per-warp async rings
  constexpr int SMEM = S::SMEM + (AS > 0 ? AS * MT * (S::KK * 32 + 64 + S::KK * 16) * 8 * (BLOCK / 32) : 0) +
                       (GS ? 2 * MT * 64 * 8 * (BLOCK / 32) : 0);
  static_assert(SMEM <= 227 * 1024, "shared memory");
  auto kern = cell_apply_kernel<N, Q, MASS, DG, BLOCK, PEER, AS, MT_, MM, GS>;
  if (cudaError_t e = opt_in_smem(kern, SMEM); e != cudaSuccess) return e;
  const int64_t supertiles = ((a.n_cells + 8 * MT - 1) / (8 * MT)) * a.nc;
  int64_t blocks = 1;
  if (cudaError_t e = persistent_grid(kern, BLOCK, SMEM, supertiles, n_sm, &blocks); e != cudaSuccess) return e;
  if (info) {
    info->dmma_per_tile = S::DMMA_PER_TILE;
    info->tiles = supertiles * MT;
    info->block = BLOCK;
    info->grid = (int)blocks;
    info->smem = SMEM;
    info->frag_doubles = S::NFRAG * 32;
    info->table = 0;
    info->flops_issued = (double)supertiles * MT * S::DMMA_PER_TILE * 512.0;
    return cudaSuccess;
  }
  if (a.n_cells == 0) return cudaSuccess;
  return launch_kernel(kern, (unsigned)blocks, BLOCK, SMEM, st, a);
}

// Reference-tensor engine (cell_tensor_kernel.cuh)
template <int N, bool MASS, bool DG, int BLOCK, int MT, bool PEER = false>
static cudaError_t launch_cell_x(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info) {
  using S = TensorShape<N, MASS>;
  auto kern = cell_tensor_kernel<N, MASS, DG, BLOCK, MT, 1, PEER>;
  if (cudaError_t e = opt_in_smem(kern, S::SMEM); e != cudaSuccess) return e;
  const int64_t supertiles = ((a.n_cells + 8 * MT - 1) / (8 * MT)) * a.nc;
  int64_t blocks = 1;
  if (cudaError_t e = persistent_grid(kern, BLOCK, S::SMEM, supertiles, n_sm, &blocks); e != cudaSuccess) return e;
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
  return launch_kernel(kern, (unsigned)blocks, BLOCK, S::SMEM, st, a);
}

// Per-degree CTA shapes, measured on 48^3 (CG reordered) / 64^3 (DG) meshes in round 1
// (profiles/r01/*.jsonl; the tuning sweeps are in git history):
//   tensor  P1 768 threads x 2 tiles per warp 31.5 us (256 x 2: 34.6), P2 1024 x 1, P3 1024 x 1,
//           P4 512 x 2 (P2 with mass 512 x 2)
//   points  one large CTA per SM: P3 768 threads (-5.6 %), P4 640 (-1.4 %), DG P2 512 (-26 %);
//   modal   P2 256 x 2 tiles 0.0516 ms, P3 768 0.1075 ms, P4 512 with the 2-stage async
//           gather ring (0.267 -> 0.245 ms reordered; P2 / P3 lose 5-8 % with any ring);
//           two 8-cell tiles per warp sharing every B-fragment load (half the shared-memory
//           wavefronts) measured 7-36 % SLOWER at P3 / P4 (fewer warps, round 2:
//           profiles/r02/modal_two_tiles.jsonl)
template <int N, bool MASS, bool DG>
static cudaError_t launch_tensor(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info) {
  if (!DG && a.peer.u != nullptr && !info) {   // multi-GPU peer ghosts
    if (N <= 4) return launch_cell_x<N, MASS, DG, 768, 2, true>(a, n_sm, st, info);
    if (N <= 20) return launch_cell_x<N, MASS, DG, 1024, 1, true>(a, n_sm, st, info);
    return launch_cell_x<N, MASS, DG, 512, 2, true>(a, n_sm, st, info);
  }
  if (N <= 4) return launch_cell_x<N, MASS, DG, 768, 2>(a, n_sm, st, info);
  if (N <= 10 && !MASS) return launch_cell_x<N, MASS, DG, 1024, 1>(a, n_sm, st, info);
  if (N <= 10) return launch_cell_x<N, MASS, DG, 512, 2>(a, n_sm, st, info);
  if (N <= 20) return launch_cell_x<N, MASS, DG, 1024, 1>(a, n_sm, st, info);
  return launch_cell_x<N, MASS, DG, 512, 2>(a, n_sm, st, info);
}

template <int N, int Q, bool MASS, bool DG>
static cudaError_t launch_points(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info) {
  using S = CellShape<N, Q, MASS>;
  constexpr int BLOCK = S::SMEM > 96 * 1024 ? 512 : 256;
  if (!DG && a.peer.u != nullptr && !info) {   // multi-GPU peer ghosts
    if (N == 20 && !MASS) return launch_cell_v<N, Q, MASS, DG, 768, true>(a, n_sm, st, info);
    if (N == 35) return launch_cell_v<N, Q, MASS, DG, 640, true>(a, n_sm, st, info);
    return launch_cell_v<N, Q, MASS, DG, BLOCK, true>(a, n_sm, st, info);
  }
  // CG P3 on the modal tables.  Up to ~1 M cells (vectors and indices L2-resident): the 2-stage
  // gather ring, 768 threads; larger meshes: no ring, geometry records staged one tile ahead
  // through shared memory (GS), 640 threads.  48^3 reordered 0.108 -> 0.100 ms (ring; GS 0.103),
  // 96^3 0.728 -> 0.672 ms (GS; ring 0.693): profiles/r02/cell_kernel_experiments.jsonl.  (Before
  // the scatter reused the gather's indices the ring lost 5-8 % at P3.)  DG P3 and CG P2 are
  // slower with either.
  if constexpr (N == 20 && !MASS && !DG && Q < N) {
    if (a.n_cells <= 1000000) return launch_cell_v<N, Q, MASS, DG, 768, false, 2>(a, n_sm, st, info);
    return launch_cell_v<N, Q, MASS, DG, 640, false, 0, 0, false, true>(a, n_sm, st, info);
  }
  if (N == 20 && !MASS) return launch_cell_v<N, Q, MASS, DG, 768>(a, n_sm, st, info);
  if constexpr (N == 35 && Q < N) return launch_cell_v<N, Q, MASS, DG, 512, false, 2>(a, n_sm, st, info);
  if (N == 35 && !DG) return launch_cell_v<N, Q, MASS, DG, 640>(a, n_sm, st, info);
  // DG P2 on the modal tables: 3-stage gather ring (cells -23 % at 64^3: the rows stream from HBM)
  if constexpr (N == 10 && DG && !MASS && Q < N) return launch_cell_v<N, Q, MASS, DG, 512, false, 3>(a, n_sm, st, info);
  if (N == 10 && DG) return launch_cell_v<N, Q, MASS, DG, 512>(a, n_sm, st, info);
  return launch_cell_v<N, Q, MASS, DG, BLOCK>(a, n_sm, st, info);
}

// engine: 1 = DMMA point loop (n_q quadrature points, or the modal tables' M modes),
// 3 = DMMA reference tensor
template <int N, int Q>
static cudaError_t cell_engine_launch(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                                      CellLaunchInfo* info, int engine) {
  if (engine == 3) {
    if (!dg) return launch_tensor<N, false, false>(a, n_sm, st, info);
    if (mass) return launch_tensor<N, true, true>(a, n_sm, st, info);
    return launch_tensor<N, false, true>(a, n_sm, st, info);
  }
  if (!dg) return launch_points<N, Q, false, false>(a, n_sm, st, info);
  if constexpr (Q < N) {
    // Helmholtz on the modal tables: the mass term as its own GEMM (cell_kernel.cuh MM); the
    // plan refuses modal + mass at P1, and no kernel with the mass term in a modal point loop exists
    if (mass) {
      if constexpr (N >= 10) {
        // P2: 3-stage gather ring, two 256-thread CTAs per SM (DG rows stream from HBM; cells
        // -19 % at 96^3, profiles/r02/dg_cell_ring.jsonl; P3 gains nothing from a ring)
        if (N == 10) return launch_cell_v<N, Q, false, true, 256, false, 3, 0, true>(a, n_sm, st, info);
        if (N == 20) return launch_cell_v<N, Q, false, true, 768, false, 0, 0, true>(a, n_sm, st, info);
        return launch_cell_v<N, Q, false, true, 512, false, 0, 0, true>(a, n_sm, st, info);
      } else {
        return cudaErrorInvalidValue;
      }
    }
    return launch_points<N, Q, false, true>(a, n_sm, st, info);
  } else {
    if (mass) return launch_points<N, Q, true, true>(a, n_sm, st, info);
    return launch_points<N, Q, false, true>(a, n_sm, st, info);
  }
}

#define TMF_CELL_TU(NN, QQ)                                                                        \
  cudaError_t cell_dispatch_##NN##_##QQ(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st, \
                                        CellLaunchInfo* info, int engine) {                         \
    return cell_engine_launch<NN, QQ>(mass, dg, a, n_sm, st, info, engine);                         \
  }

}  // namespace tmf
