// Face-kernel instantiations and launchers (sm_100a).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "face_kernel.cuh"
#include "launch.h"
#include "launch_common.cuh"

namespace tmf {

template <int N, int QF, bool BND, int PF = 2, int MINB = 2, int BLOCK = 256, bool BLOCKED = false,
          bool PEER = false, bool RESIDENT = false, bool HIER = false, bool SG = false, bool RT = false>
static cudaError_t launch_face_v(const FaceArgs& a, int n_sm, cudaStream_t st, FaceLaunchInfo* info) {
  using S = FaceShapeSel<N, QF, HIER>;
  constexpr int SMEM = ((RT && !RESIDENT) ? 0 : RESIDENT ? 24 * S::NFRAG * 32 * 8 : (BND ? 1 : 2) * S::NFRAG * 32 * 8) +
                       (SG ? (BLOCK / 32) * 128 * 8 : 0);   // + the per-warp staged face records
  static_assert(SMEM <= 227 * 1024, "shared memory");
  auto kern = face_apply_kernel<N, QF, BND, PF, MINB, BLOCK, BLOCKED, PEER, RESIDENT, HIER, SG, RT>;
  if (cudaError_t e = opt_in_smem(kern, SMEM); e != cudaSuccess) return e;
  if (info) {
    info->nfrag = S::NFRAG;
    info->chunk = S::CHUNK;
    info->dmma_per_batch = BND ? (S::NB1 + S::NB2) : 2 * (S::NB1 + S::NB2);
    return cudaSuccess;
  }
  int per_sm = 0;
  cudaError_t e = blocks_per_sm(kern, BLOCK, SMEM, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t work = a.n_chunks * a.nc;
  if (work == 0) return cudaSuccess;
  int64_t blocks = (int64_t)n_sm * per_sm;
  if (blocks > work) blocks = work;
  return launch_kernel(kern, (unsigned)blocks, BLOCK, SMEM, st, a);
}

// interior faces with the asynchronous gather ring (face_async_kernel), blocked chunk runs
template <int N, int QF, int AS, int MINB, int BLOCK = 256, bool HIER = false>
static cudaError_t launch_face_a(const FaceArgs& a, int n_sm, cudaStream_t st) {
  using S = FaceShapeSel<N, QF, HIER>;
  constexpr int SLOT = 2 * S::KK * 32 + 64 + 16;
  constexpr int SMEM = (2 * S::NFRAG * 32 + (4 * N + 1) / 2 + (BLOCK / 32) * AS * SLOT) * 8;
  if constexpr (SMEM > 227 * 1024) {
    return cudaErrorNotSupported;   // tables + rings do not fit (n_qf-point P4): caller falls back
  } else {
    auto kern = face_async_kernel<N, QF, AS, MINB, BLOCK, true, HIER>;
    if (cudaError_t e = opt_in_smem(kern, SMEM); e != cudaSuccess) return e;
    int per_sm = 0;
    cudaError_t e = blocks_per_sm(kern, BLOCK, SMEM, &per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    const int64_t work = a.n_chunks * a.nc;
    if (work == 0) return cudaSuccess;
    int64_t blocks = (int64_t)n_sm * per_sm;
    if (blocks > work) blocks = work;
    return launch_kernel(kern, (unsigned)blocks, BLOCK, SMEM, st, a);
  }
}

// Per-degree defaults, measured in round 1 (tuning sweeps in git history, profiles/r01):
// contiguous chunk runs per CTA (tables restaged only when the signature changes: -7 % /
// -8 % at P3 / P2); low degrees have short batches, so occupancy beats prefetch depth;
// P >= 3 prefers the fully prefetching 2-CTA kernel.  Modal tables: P2 prefers round-robin
// chunks with record prefetch at 3 CTAs/SM (Helmholtz 96^3 1.55 ms vs 1.90 blocked); P4
// interior faces take the 3-stage asynchronous gather ring (DG 48^3 1.05 -> 0.85 ms; P2 / P3
// gain nothing from it).
// Split-mode modal layout (HierShape), interior faces.  TMF_FACE_VARIANT (environment,
// experiments only) picks another CTA shape / pipeline.
template <int N>
static cudaError_t launch_face_h(const FaceArgs& a, int n_sm, cudaStream_t st, FaceLaunchInfo* info) {
  constexpr int QF = HierShape<N>::NF;
  static const int variant = [] {
    const char* e = std::getenv("TMF_FACE_VARIANT");
    return e ? std::atoi(e) : 0;
  }();
  if (info) return launch_face_v<N, QF, false, 1, 2, 256, false, false, false, true>(a, n_sm, st, info);
  if (a.peer.u != nullptr) {
    if (N <= 10) return launch_face_v<N, QF, false, 1, 3, 256, true, true, false, true>(a, n_sm, st, info);
    return launch_face_v<N, QF, false, 2, 2, 256, true, true, false, true>(a, n_sm, st, info);
  }
  if constexpr (N == 35) {
    if (variant == 1) return launch_face_v<N, QF, false, 2, 2, 256, true, false, false, true>(a, n_sm, st, info);
    if (variant == 2) return launch_face_a<N, QF, 2, 2, 256, true>(a, n_sm, st);
    return launch_face_a<N, QF, 3, 2, 256, true>(a, n_sm, st);
  } else if constexpr (N == 20) {
    if (variant == 1) return launch_face_v<N, QF, false, 1, 1, 512, false, false, true, true>(a, n_sm, st, info);
    if (variant == 2) return launch_face_v<N, QF, false, 2, 1, 512, false, false, true, true>(a, n_sm, st, info);
    if (variant == 3) return launch_face_v<N, QF, false, 1, 1, 768, false, false, true, true>(a, n_sm, st, info);
    if (variant == 4) return launch_face_a<N, QF, 3, 2, 256, true>(a, n_sm, st);
    if (variant == 5) return launch_face_v<N, QF, false, 1, 3, 256, true, false, false, true>(a, n_sm, st, info);
    if (variant == 10) return launch_face_v<N, QF, false, 2, 2, 256, true, false, false, true>(a, n_sm, st, info);
    if (variant == 11) return launch_face_v<N, QF, false, 2, 2, 256, true, false, false, true, true>(a, n_sm, st, info);
    if (variant == 12) return launch_face_v<N, QF, false, 2, 8, 64, true, false, false, true, true>(a, n_sm, st, info);
    // default: full prefetch, face records staged through shared memory (SG: faces -1.9 %), four
    // 128-thread CTAs per SM instead of two of 256 (fewer warps wait at each table restage:
    // DG P3 64^3 faces 0.677 -> 0.631 ms, profiles/r02/face_runs.jsonl)
    return launch_face_v<N, QF, false, 2, 4, 128, true, false, false, true, true>(a, n_sm, st, info);
  } else if constexpr (N == 10) {
    // P2: both tables of a chunk (2 x 10 fragments) live in REGISTERS, loaded once per chunk from
    // global memory (no table shared memory, no barriers); small CTAs (2 warps, 8 per SM) so a
    // warp serves 16 batches per table load; face records staged through shared memory.
    // kappa-Helmholtz P2 96^3 faces 1.032 -> 0.895 ms (-13 %) against round 2's resident-table
    // 512-thread kernel (variant 1), profiles/r02/face_register_tables.jsonl
    if (variant == 1) return launch_face_v<N, QF, false, 1, 1, 512, false, false, true, true>(a, n_sm, st, info);
    if (variant == 2) return launch_face_v<N, QF, false, 1, 4, 128, false, false, false, true, true, true>(a, n_sm, st, info);
    return launch_face_v<N, QF, false, 1, 8, 64, false, false, false, true, true, true>(a, n_sm, st, info);
  } else {
    return launch_face_v<N, QF, false, 1, 3, 256, true, false, false, true>(a, n_sm, st, info);
  }
}

template <int N, int QF, bool BND>
static cudaError_t launch_face_t(const FaceArgs& a, int n_sm, cudaStream_t st, FaceLaunchInfo* info) {
  if (!BND && a.peer.u != nullptr && !info) {   // multi-GPU: plus-side ghost cells from peer memory
    if (N <= 10) return launch_face_v<N, QF, BND, 1, 3, 256, true, true>(a, n_sm, st, info);
    return launch_face_v<N, QF, BND, 2, 2, 256, true, true>(a, n_sm, st, info);
  }
  if constexpr (!BND && N == 35) {
    if (!info && QF < N) {
      cudaError_t e = launch_face_a<N, QF, 3, 2>(a, n_sm, st);
      if (e != cudaErrorNotSupported) return e;
    }
  }
  // P2 modal interior faces: all 24 (lf, code) tables resident in shared memory (123 KB), one
  // 512-thread CTA per SM, no restaging and no barriers between chunks: faces -6 to -7 % at
  // 64^3 / 96^3 against the restaging 3-CTA kernel (round 2, profiles/r02/face_resident.jsonl)
  if constexpr (!BND && N == 10 && QF < 10) {
    if (!info && a.peer.u == nullptr) return launch_face_v<N, QF, BND, 1, 1, 512, false, false, true>(a, n_sm, st, info);
  }
  if (N == 10 && QF < 10) return launch_face_v<N, QF, BND, 1, 3>(a, n_sm, st, info);
  if (N <= 10) return launch_face_v<N, QF, BND, 1, 3, 256, true>(a, n_sm, st, info);
  return launch_face_v<N, QF, BND, 2, 2, 256, true>(a, n_sm, st, info);
}

cudaError_t launch_face(int n_dpc, int n_qf, bool boundary, const FaceArgs& a, int n_sm,
                        cudaStream_t st, FaceLaunchInfo* info, bool* supported) {
  *supported = true;
  if (a.hier && !boundary) {
    if (n_dpc == 4) return launch_face_h<4>(a, n_sm, st, info);
    if (n_dpc == 10) return launch_face_h<10>(a, n_sm, st, info);
    if (n_dpc == 20) return launch_face_h<20>(a, n_sm, st, info);
    if (n_dpc == 35) return launch_face_h<35>(a, n_sm, st, info);
    *supported = false;
    return cudaSuccess;
  }
#define TMF_FACE(NN, QQ)                                                          \
  if (n_dpc == NN && n_qf == QQ) {                                                \
    if (boundary) return launch_face_t<NN, QQ, true>(a, n_sm, st, info);          \
    return launch_face_t<NN, QQ, false>(a, n_sm, st, info);                       \
  }
  TMF_FACE(4, 3)
  TMF_FACE(4, 4)
  TMF_FACE(10, 6)
  TMF_FACE(10, 10)
  TMF_FACE(20, 12)
  TMF_FACE(20, 20)
  TMF_FACE(20, 10)   // modal face tables (NF = dim P_p on the face)
  TMF_FACE(35, 35)
  TMF_FACE(35, 15)
#undef TMF_FACE
  *supported = false;
  return cudaSuccess;
}

cudaError_t launch_face_geometry(bool boundary, const FaceGeoArgs& a, int n_sm, cudaStream_t st) {
  if (a.n_chunks == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)std::min<int64_t>(a.n_chunks, (int64_t)n_sm * 8);
  if (boundary)
    face_geometry_kernel<true><<<blocks, 256, 0, st>>>(a);
  else
    face_geometry_kernel<false><<<blocks, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace tmf
