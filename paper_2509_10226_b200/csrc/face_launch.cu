// Face-kernel instantiations and launchers (sm_100a).
#include <cuda_runtime.h>

#include <algorithm>

#include "face_kernel.cuh"
#include "face_tensor_kernel.cuh"
#include "launch.h"
#include "launch_common.cuh"

namespace tmf {

template <int N, int QF, bool BND, int PF = 2, int MINB = 2, int BLOCK = 256, bool BLOCKED = false,
          bool TPF = false, bool PEER = false>
static cudaError_t launch_face_v(const FaceArgs& a, int n_sm, cudaStream_t st, FaceLaunchInfo* info) {
  using S = FaceShape<N, QF>;
  constexpr int SMEM = (TPF ? 2 : 1) * (BND ? 1 : 2) * S::NFRAG * 32 * 8;
  auto kern = face_apply_kernel<N, QF, BND, PF, MINB, BLOCK, BLOCKED, TPF, PEER>;
  if (cudaError_t e = opt_in_smem(kern, SMEM); e != cudaSuccess) return e;
  if (info) {
    info->nfrag = S::NFRAG;
    info->chunk = S::CHUNK;
    info->dmma_per_batch = BND ? (S::NB1 + S::NB2) : 2 * (S::NB1 + S::NB2);
    info->blocked_grid = 0;
    if (BLOCKED && !TPF) {
      int ps = 0;
      if (blocks_per_sm(kern, BLOCK, SMEM, &ps) == cudaSuccess) info->blocked_grid = n_sm * (ps < 1 ? 1 : ps);
    }
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
  kern<<<(unsigned)blocks, BLOCK, SMEM, st>>>(a);
  return cudaGetLastError();
}

// Interior faces, MB batches per warp iteration (face_mb_kernel)
template <int N, int QF, int MB, int MINB, bool BLOCKED>
static cudaError_t launch_face_mb(const FaceArgs& a, int n_sm, cudaStream_t st) {
  using S = FaceShape<N, QF>;
  constexpr int SMEM = 2 * S::NFRAG * 32 * 8;
  auto kern = face_mb_kernel<N, QF, MB, MINB, 256, BLOCKED>;
  if (cudaError_t e = opt_in_smem(kern, SMEM); e != cudaSuccess) return e;
  int per_sm = 0;
  cudaError_t e = blocks_per_sm(kern, 256, SMEM, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t work = a.n_chunks * a.nc;
  if (work == 0) return cudaSuccess;
  int64_t blocks = (int64_t)n_sm * per_sm;
  if (blocks > work) blocks = work;
  kern<<<(unsigned)blocks, 256, SMEM, st>>>(a);
  return cudaGetLastError();
}

// Reference-tensor interior-face kernel (face_tensor_kernel.cuh)
template <int N, int BLOCK, int MINB, bool PF>
static cudaError_t launch_face_x(const FaceArgs& a, int n_sm, cudaStream_t st) {
  using S = FaceTensorShape<N>;
  auto kern = face_tensor_kernel<N, BLOCK, MINB, PF>;
  if (cudaError_t e = opt_in_smem(kern, S::SMEM); e != cudaSuccess) return e;
  int per_sm = 0;
  cudaError_t e = blocks_per_sm(kern, BLOCK, S::SMEM, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t work = a.n_chunks * a.nc;
  if (work == 0) return cudaSuccess;
  int64_t blocks = (int64_t)n_sm * per_sm;
  if (blocks > work) blocks = work;
  kern<<<(unsigned)blocks, BLOCK, S::SMEM, st>>>(a);
  return cudaGetLastError();
}

// variants of the tensor face kernel: 0 = by degree; 1..6 tuning (bench sweeps)
template <int N>
static cudaError_t launch_face_xt(const FaceArgs& a, int n_sm, cudaStream_t st, int variant) {
  if (variant == 1) return launch_face_x<N, 256, 3, false>(a, n_sm, st);
  if (variant == 2) return launch_face_x<N, 256, 2, true>(a, n_sm, st);
  if (variant == 3) return launch_face_x<N, 256, 2, false>(a, n_sm, st);
  if (variant == 4) return launch_face_x<N, 512, 1, true>(a, n_sm, st);
  if (variant == 5) return launch_face_x<N, 128, 4, true>(a, n_sm, st);
  if (variant == 6) return launch_face_x<N, 256, 3, true>(a, n_sm, st);
  // measured (tools/gpu_face3.sh): P2 Helmholtz 96^3 128 x 4 CTAs with prefetch 1.77 ms
  // (256 x 3 without: 1.80); P3 64^3 256 x 2 with prefetch 1.14 ms (best of 7)
  if (N <= 10) return launch_face_x<N, 128, 4, true>(a, n_sm, st);
  return launch_face_x<N, 256, 2, true>(a, n_sm, st);
}

// interior faces with the asynchronous gather ring (face_async_kernel)
template <int N, int QF, int AS, int MINB, int BLOCK = 256, bool BLOCKED = false>
static cudaError_t launch_face_a(const FaceArgs& a, int n_sm, cudaStream_t st) {
  using S = FaceShape<N, QF>;
  constexpr int SLOT = 2 * S::KK * 32 + 64 + 16;
  constexpr int SMEM = (2 * S::NFRAG * 32 + (4 * N + 1) / 2 + (BLOCK / 32) * AS * SLOT) * 8;
  if constexpr (SMEM > 227 * 1024) {
    return cudaErrorNotSupported;   // tables + rings do not fit (n_qf-point P4): caller falls back
  }
  auto kern = face_async_kernel<N, QF, AS, MINB, BLOCK, BLOCKED>;
  if (cudaError_t e = opt_in_smem(kern, SMEM); e != cudaSuccess) return e;
  int per_sm = 0;
  cudaError_t e = blocks_per_sm(kern, BLOCK, SMEM, &per_sm);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t work = a.n_chunks * a.nc;
  if (work == 0) return cudaSuccess;
  int64_t blocks = (int64_t)n_sm * per_sm;
  if (blocks > work) blocks = work;
  kern<<<(unsigned)blocks, BLOCK, SMEM, st>>>(a);
  return cudaGetLastError();
}

// variant: 0 = default (by degree, below, blocked chunk runs); 1 = no prefetch, 3 CTAs/SM;
// 2 = record prefetch, 3 CTAs/SM; 3 = record prefetch, 2 CTAs/SM; 4 = full prefetch, 2 CTAs/SM
template <int N, int QF, bool BND>
static cudaError_t launch_face_t(const FaceArgs& a, int n_sm, cudaStream_t st, FaceLaunchInfo* info,
                                 int variant) {
  if (!BND && info) {
    info->tnfrag = FaceTensorShape<N>::NFRAG;
    info->tdmma_per_batch = FaceTensorShape<N>::DMMA_PER_BATCH;
  }
  if (!BND && !info && a.tfrags != nullptr && a.peer.u == nullptr) return launch_face_xt<N>(a, n_sm, st, variant);
  if (!BND && a.peer.u != nullptr && !info) {   // multi-GPU: plus-side ghost cells from peer memory
    if (N <= 10) return launch_face_v<N, QF, BND, 1, 3, 256, true, false, true>(a, n_sm, st, info);
    return launch_face_v<N, QF, BND, 2, 2, 256, true, false, true>(a, n_sm, st, info);
  }
  if (variant == 1) return launch_face_v<N, QF, BND, 0, 3>(a, n_sm, st, info);
  if (variant == 2) return launch_face_v<N, QF, BND, 1, 3>(a, n_sm, st, info);
  if (variant == 3) return launch_face_v<N, QF, BND, 1, 2>(a, n_sm, st, info);
  if (variant == 4) return launch_face_v<N, QF, BND, 2, 2>(a, n_sm, st, info);
  if (variant == 5) return launch_face_v<N, QF, BND, 1, 1, 512>(a, n_sm, st, info);
  if (variant == 6) return launch_face_v<N, QF, BND, 2, 1, 512>(a, n_sm, st, info);
  if (variant == 7) return launch_face_v<N, QF, BND, 1, 4>(a, n_sm, st, info);          // 64 registers
  if (variant == 8) return launch_face_v<N, QF, BND, 1, 6, 128>(a, n_sm, st, info);
  if (variant == 9) return launch_face_v<N, QF, BND, 1, 3, 256, true>(a, n_sm, st, info);
  if (variant == 10) return launch_face_v<N, QF, BND, 2, 2, 256, true>(a, n_sm, st, info);
  // (variants 11 / 12 were round-robin chunks + cp.async table prefetch, TPF: measured 5-15 %
  // slower than the blocked default at C3 / C4 sizes; they now select the two-batch kernel)
  if constexpr (!BND) {
    if (!info && a.peer.u == nullptr && (variant == 11 || variant == 12)) {
      if (variant == 11) return launch_face_mb<N, QF, 2, 2, false>(a, n_sm, st);
      return launch_face_mb<N, QF, 2, 2, true>(a, n_sm, st);
    }
  }
  if constexpr (!BND) {   // asynchronous gather ring (no peers)
    if (!info && a.peer.u == nullptr && variant >= 13) {
      cudaError_t e = cudaErrorNotSupported;
      if (variant == 13) e = launch_face_a<N, QF, 2, 3>(a, n_sm, st);
      if (variant == 14) e = launch_face_a<N, QF, 3, 2>(a, n_sm, st);
      if (variant == 15) e = launch_face_a<N, QF, 3, 2, 256, true>(a, n_sm, st);
      if (e != cudaErrorNotSupported) return e;
      variant = 0;   // does not fit in shared memory: the default kernel
    }
  }
  // default: contiguous chunk runs per CTA (tables restaged only when the signature
  // changes: -7 % / -8 % at P3 / P2); low degrees have short batches, so occupancy
  // beats prefetch depth (P2 96^3: 2.39 vs 2.48 ms); P >= 3 prefers the fully
  // prefetching 2-CTA kernel
  //   modal tables (QF = NF < n_qf, tools/gpu_modal2.sh): P2 prefers round-robin chunks
  //   with record prefetch at 3 CTAs/SM (Helmholtz 96^3 1.55 ms vs 1.90 blocked), P3 / P4
  //   the default below (DG 64^3 P3 0.94 ms, 48^3 P4 1.04 ms)
  //   P4 interior faces (modal) with the 3-stage asynchronous gather ring, blocked chunk runs
  //   (variant 15): DG 48^3 1.05 -> 0.85 ms; P2 / P3 gain nothing from the ring (-2 % / +7 %)
  if constexpr (!BND && N == 35) {
    if (!info && a.peer.u == nullptr && QF < N) {
      cudaError_t e = launch_face_a<N, QF, 3, 2, 256, true>(a, n_sm, st);
      if (e != cudaErrorNotSupported) return e;
    }
  }
  if (N == 10 && QF < 10) return launch_face_v<N, QF, BND, 1, 3>(a, n_sm, st, info);
  if (N <= 10) return launch_face_v<N, QF, BND, 1, 3, 256, true>(a, n_sm, st, info);
  return launch_face_v<N, QF, BND, 2, 2, 256, true>(a, n_sm, st, info);
}

cudaError_t launch_face(int n_dpc, int n_qf, bool boundary, const FaceArgs& a, int n_sm,
                        cudaStream_t st, FaceLaunchInfo* info, bool* supported, int variant) {
  *supported = true;
#define TMF_FACE(NN, QQ)                                                          \
  if (n_dpc == NN && n_qf == QQ) {                                                \
    if (boundary) return launch_face_t<NN, QQ, true>(a, n_sm, st, info, variant); \
    return launch_face_t<NN, QQ, false>(a, n_sm, st, info, variant);              \
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
