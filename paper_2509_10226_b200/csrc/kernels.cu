// Kernel instantiations and launchers for tetmf_b200 (sm_100a).
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <unordered_map>

#include "cell_kernel.cuh"
#include "face_kernel.cuh"
#include "launch.h"

namespace tmf {

// Dynamic shared memory above 48 KB needs a per-kernel, per-DEVICE opt-in; remember
// which (kernel, device) pairs have been configured (kernels sharing a signature share
// a function-pointer type, so the key is the pointer itself).
template <typename K>
static cudaError_t opt_in_smem(K kern, int bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, unsigned long long> done;  // bit d = device d (< 64)
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> lock(mu);
  unsigned long long& mask = done[reinterpret_cast<const void*>(kern)];
  if (mask & bit) return cudaSuccess;
  if (cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      e != cudaSuccess)
    return e;
  mask |= bit;
  return cudaSuccess;
}

template <int N, int Q, bool MASS, bool DG, int BLOCK, int MT, int MINB, bool PF = false, bool BLK = false,
          bool SKEW = false>
static cudaError_t launch_cell_v(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info) {
  using S = CellShape<N, Q, MASS>;
  constexpr int MTE = MT ? MT : S::MT;
  auto kern = cell_apply_kernel<N, Q, MASS, DG, BLOCK, MT, MINB, PF, BLK, SKEW>;
  if (cudaError_t e = opt_in_smem(kern, S::SMEM); e != cudaSuccess) return e;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BLOCK, S::SMEM);
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
    info->smem = S::SMEM;
    info->frag_doubles = S::NFRAG * 32;
    return cudaSuccess;
  }
  kern<<<(unsigned)blocks, BLOCK, S::SMEM, st>>>(a);
  return cudaGetLastError();
}

// variant: 0 = default; 1..3 = tuning variants of the CG kernel (bench sweeps only)
template <int N, int Q, bool MASS, bool DG>
static cudaError_t launch_cell_t(const CellArgs& a, int n_sm, cudaStream_t st, CellLaunchInfo* info,
                                 int variant) {
  using S = CellShape<N, Q, MASS>;
  constexpr int BLOCK = S::SMEM > 96 * 1024 ? 512 : 256;
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
  //   CG P3 additionally skews GEMM1(t+1) ahead of the D action of tile t (-2.7 %;
  //   slower for the other families, variant 14)
  if (N == 20 && !MASS && !DG) return launch_cell_v<N, Q, MASS, DG, 768, 0, 1, false, false, true>(a, n_sm, st, info);
  if (N == 20 && !MASS) return launch_cell_v<N, Q, MASS, DG, 768, 0, 1>(a, n_sm, st, info);
  if (N == 35 && !DG) return launch_cell_v<N, Q, MASS, DG, 640, 0, 1>(a, n_sm, st, info);
  if (N == 10 && DG) return launch_cell_v<N, Q, MASS, DG, 512, 0, 1>(a, n_sm, st, info);
  return launch_cell_v<N, Q, MASS, DG, BLOCK, 0, 1>(a, n_sm, st, info);
}

template <int N, int Q>
static cudaError_t cell_variant(bool mass, bool dg, const CellArgs& a, int n_sm, cudaStream_t st,
                                CellLaunchInfo* info, int variant) {
  if (!dg) return launch_cell_t<N, Q, false, false>(a, n_sm, st, info, variant);
  if (mass) return launch_cell_t<N, Q, true, true>(a, n_sm, st, info, variant);
  return launch_cell_t<N, Q, false, true>(a, n_sm, st, info, variant);
}

cudaError_t launch_cell(int n_dpc, int n_q, bool mass, bool dg, const CellArgs& a, int n_sm,
                        cudaStream_t st, CellLaunchInfo* info, bool* supported, int variant) {
  *supported = true;
#define TMF_CELL(NN, QQ) \
  if (n_dpc == NN && n_q == QQ) return cell_variant<NN, QQ>(mass, dg, a, n_sm, st, info, variant);
  TMF_CELL(4, 4)
  TMF_CELL(4, 5)
  TMF_CELL(10, 14)
  TMF_CELL(10, 15)
  TMF_CELL(20, 35)
  TMF_CELL(35, 70)
#undef TMF_CELL
  *supported = false;
  return cudaSuccess;
}

template <int N, int QF, bool BND, int PF = 2, int MINB = 2, int BLOCK = 256, bool BLOCKED = false>
static cudaError_t launch_face_v(const FaceArgs& a, int n_sm, cudaStream_t st, FaceLaunchInfo* info) {
  using S = FaceShape<N, QF>;
  constexpr int SMEM = (BND ? 1 : 2) * S::NFRAG * 32 * 8;
  auto kern = face_apply_kernel<N, QF, BND, PF, MINB, BLOCK, BLOCKED>;
  if (cudaError_t e = opt_in_smem(kern, SMEM); e != cudaSuccess) return e;
  if (info) {
    info->nfrag = S::NFRAG;
    info->chunk = S::CHUNK;
    info->dmma_per_batch = BND ? (S::NB1 + S::NB2) : 2 * (S::NB1 + S::NB2);
    return cudaSuccess;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BLOCK, SMEM);
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
  if (variant == 1) return launch_face_v<N, QF, BND, 0, 3>(a, n_sm, st, info);
  if (variant == 2) return launch_face_v<N, QF, BND, 1, 3>(a, n_sm, st, info);
  if (variant == 3) return launch_face_v<N, QF, BND, 1, 2>(a, n_sm, st, info);
  if (variant == 4) return launch_face_v<N, QF, BND, 2, 2>(a, n_sm, st, info);
  if (variant == 5) return launch_face_v<N, QF, BND, 1, 1, 512>(a, n_sm, st, info);
  if (variant == 6) return launch_face_v<N, QF, BND, 2, 1, 512>(a, n_sm, st, info);
  if (variant == 7) return launch_face_v<N, QF, BND, 1, 1, 768>(a, n_sm, st, info);
  if (variant == 8) return launch_face_v<N, QF, BND, 1, 2, 384>(a, n_sm, st, info);
  if (variant == 9) return launch_face_v<N, QF, BND, 1, 3, 256, true>(a, n_sm, st, info);
  if (variant == 10) return launch_face_v<N, QF, BND, 2, 2, 256, true>(a, n_sm, st, info);
  // default: contiguous chunk runs per CTA (tables restaged only when the signature
  // changes: -7 % / -8 % at P3 / P2); low degrees have short batches, so occupancy
  // beats prefetch depth (P2 96^3: 2.39 vs 2.48 ms); P >= 3 prefers the fully
  // prefetching 2-CTA kernel
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
  TMF_FACE(35, 35)
#undef TMF_FACE
  *supported = false;
  return cudaSuccess;
}

cudaError_t launch_cell_geometry(const CellGeoArgs& a, int n_sm, cudaStream_t st) {
  cell_geometry_kernel<<<n_sm * 8, 256, 0, st>>>(a);
  return cudaGetLastError();
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

cudaError_t launch_fixup(const double* u, double* y, const int* list, int64_t n, int n_sm,
                         cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 4 * n_sm) blocks = 4 * n_sm;
  dirichlet_fixup_kernel<<<(unsigned)blocks, 256, 0, st>>>(u, y, list, n);
  return cudaGetLastError();
}

}  // namespace tmf
