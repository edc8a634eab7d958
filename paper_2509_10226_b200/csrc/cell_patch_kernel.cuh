// CG cell term with patch-local assembly and an asynchronous copy pipeline.
//
// Same arithmetic as cell_dfma_kernel.cuh (operator.py:255-278; DFMA point
// loop), reorganised around the locality that hierarchical reordering gives
// (PAPER.md:274-280): the cells are cut into patches of CH = BLOCK consecutive
// cells, one thread per cell, one patch per CTA iteration.  A patch of a
// reordered mesh touches few DoFs (P1: ~0.17 unique DoFs per cell-DoF slot),
// so instead of N scattered global gathers and N global atomics per cell:
//
//   1. TMA bulk copies (cp.async.bulk, mbarrier completion) bring the patch's
//      contiguous records into a STAGES-deep shared-memory ring, two patches
//      ahead: G (6 x CH, component-major), the 16-bit local DoF indices
//      (word-major), the unique-DoF list and the incidence lists;
//   2. one patch ahead, the unique DoFs' u values are gathered from L2 with
//      8-byte cp.async into a double-buffered shared array;
//   3. the cells read u and G from shared memory, run the point loop, and
//      write their residuals to a shared contribution array sc[j][CHP];
//   4. one thread per unique DoF sums its incidences (deterministic order)
//      and issues ONE global RED.
//
// So the only long-latency traffic on the critical path is prefetched, and
// global atomics drop from N per cell to ~N * ratio per cell.
#pragma once
#include "cell_dfma_kernel.cuh"

namespace tmf {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory");
}

template <int N, int Q, int BLOCK>
struct PatchShape {
  using D = DfmaShape<N, Q, false>;
  static constexpr int NP = D::NP;
  static constexpr int CH = BLOCK;          // cells per patch
  static constexpr int CHP = CH + 4;        // contribution row stride (conflict-free)
  static constexpr int NW = NP / 2;         // 32-bit words of local indices per cell
  // shared-memory bytes for a plan with numax / icmax (see CellArgs)
  __host__ __device__ static constexpr size_t fixed_bytes() { return (size_t)2 * D::TAB * 8 + (size_t)N * CHP * 8; }
  __host__ __device__ static size_t stage_bytes(int numax, int icmax) {
    return (size_t)6 * CH * 8 + (size_t)numax * 4 + (size_t)NW * CH * 4 + (size_t)icmax * 2;
  }
  __host__ __device__ static size_t smem_bytes(int numax, int icmax, int stages) {   // + 32 B barriers + metadata
    return fixed_bytes() + (size_t)2 * numax * 8 + stages * stage_bytes(numax, icmax) + 32 + 16 * stages;
  }
};

template <int N, int Q, int BLOCK, int STAGES, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) cell_patch_kernel(CellArgs a) {
  static_assert(STAGES >= 3 && STAGES <= 4, "bulk data runs two patches ahead");
  using S = PatchShape<N, Q, BLOCK>;
  using D = DfmaShape<N, Q, false>;
  constexpr int NP = S::NP, CH = S::CH, CHP = S::CHP, NW = S::NW;
  extern __shared__ __align__(16) unsigned char sbytes[];
  double* tab = reinterpret_cast<double*>(sbytes);
  double* sc = tab + 2 * D::TAB;                            // [N][CHP]
  double* su = sc + N * CHP;                                // [2][numax]
  unsigned char* stage0 = reinterpret_cast<unsigned char*>(su + 2 * a.numax);
  const size_t sbytes_stage = S::stage_bytes(a.numax, a.icmax);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stage0 + STAGES * sbytes_stage);
  int4* smeta = reinterpret_cast<int4*>(bars + 4);          // 16-byte aligned
  auto st_geo = [&](int s) { return reinterpret_cast<double*>(stage0 + s * sbytes_stage); };
  auto st_pd = [&](int s) { return reinterpret_cast<int*>(stage0 + s * sbytes_stage + 6 * CH * 8); };
  auto st_lid = [&](int s) {
    return reinterpret_cast<uint32_t*>(stage0 + s * sbytes_stage + 6 * CH * 8 + a.numax * 4);
  };
  auto st_ic = [&](int s) {
    return reinterpret_cast<uint16_t*>(stage0 + s * sbytes_stage + 6 * CH * 8 + a.numax * 4 + NW * CH * 4);
  };

  const int tid = threadIdx.x;
  const int64_t cpc = (a.n_cells + CH - 1) / CH;
  const int64_t nch = cpc * a.nc;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  {
    const double2* src = reinterpret_cast<const double2*>(a.frags);
    double2* dst = reinterpret_cast<double2*>(tab);
    for (int i = tid; i < D::TAB; i += BLOCK) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const double2* T1 = reinterpret_cast<const double2*>(tab);
  const double2* T2 = reinterpret_cast<const double2*>(tab + D::TAB);

  // patch k of this CTA -> chunk (component-major), patch id
  auto chunk = [&](int64_t k) { return (int64_t)blockIdx.x + k * gridDim.x; };
  auto issue = [&](int64_t k) {   // tid 0: bulk copies of patch k into stage k % STAGES
    const int64_t ch = chunk(k);
    if (ch >= nch) return;
    const int64_t p = ch % cpc;
    const int s = (int)(k % STAGES);
    const int4 m = __ldg(a.pmeta + p);
    smeta[s] = m;
    // the stage was last read through the generic proxy (iteration k - STAGES)
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    const uint32_t b_geo = 6 * CH * 8, b_pd = (uint32_t)((m.y + 3) & ~3) * 4, b_lid = NW * CH * 4,
                   b_ic = (uint32_t)m.w * 2;
    mbar_expect_tx(bars + s, b_geo + b_pd + b_lid + b_ic);
    bulk_g2s(st_geo(s), a.pgeo + p * 6 * CH, b_geo, bars + s);
    if (b_pd) bulk_g2s(st_pd(s), a.pdofs + m.x, b_pd, bars + s);
    bulk_g2s(st_lid(s), a.plidw + p * NW * CH, b_lid, bars + s);
    bulk_g2s(st_ic(s), a.pic + m.z, b_ic, bars + s);
  };
  auto gather = [&](int64_t k) {  // all threads: u of patch k's unique DoFs -> su[k & 1]
    const int64_t ch = chunk(k);
    if (ch < nch) {
      const int s = (int)(k % STAGES);
      mbar_wait(bars + s, (uint32_t)((k / STAGES) & 1));
      const int comp = (int)(ch / cpc);
      const int nu = smeta[s].y;
      const int* pd = st_pd(s);
      double* dst = su + (k & 1) * a.numax;
      for (int i = tid; i < nu; i += BLOCK) cp_async8(dst + i, a.u + (int64_t)pd[i] * a.nc + comp);
    }
    cp_async_commit();
  };

  if (tid == 0)
    for (int k = 0; k < STAGES - 1; ++k) issue(k);
  __syncthreads();   // smeta of the first stages
  gather(0);
  for (int64_t k = 0; chunk(k) < nch; ++k) {
    const int64_t ch = chunk(k);
    const int comp = (int)(ch / cpc);
    const int s = (int)(k % STAGES);
    if (tid == 0) issue(k + STAGES - 1);   // its stage was released by iteration k-1
    gather(k + 1);
    cp_async_wait<1>();                     // this thread's gathers of patch k
    __syncthreads();

    // ---- cells: one per thread
    const double* sk = su + (k & 1) * a.numax;
    double uu[1][NP], yy[1][NP], G[1][6], md[1] = {0.0};
    {
      const uint32_t* lid = st_lid(s);
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const uint32_t x = lid[w * CH + tid];
        const uint32_t l0 = x & 0xFFFFu, l1 = x >> 16;
        uu[0][2 * w] = l0 != 0xFFFFu ? sk[l0] : 0.0;
        uu[0][2 * w + 1] = l1 != 0xFFFFu ? sk[l1] : 0.0;
      }
      const double* geo = st_geo(s);
#pragma unroll
      for (int i = 0; i < 6; ++i) G[0][i] = geo[i * CH + tid];
    }
    dfma_cell_points<N, Q, false, 1>(T1, T2, uu, G, md, yy);
#pragma unroll
    for (int j = 0; j < N; ++j) sc[j * CHP + tid] = yy[0][j];
    __syncthreads();

    // ---- unique DoFs: sum the incidences, one RED each
    {
      const int nu = smeta[s].y;
      const int* pd = st_pd(s);
      const uint16_t* ic = st_ic(s);
      const uint16_t* pos = ic + ((nu + 1 + 7) & ~7);
      for (int i = tid; i < nu; i += BLOCK) {
        const int k0 = ic[i], k1 = ic[i + 1];
        double s0 = 0.0, s1 = 0.0;
        int kk = k0;
        for (; kk + 1 < k1; kk += 2) {
          s0 += sc[pos[kk]];
          s1 += sc[pos[kk + 1]];
        }
        if (kk < k1) s0 += sc[pos[kk]];
        atomicAdd(a.y + (int64_t)pd[i] * a.nc + comp, s0 + s1);
      }
    }
    __syncthreads();   // stage s, su[k & 1] and sc are reused
  }
}

}  // namespace tmf
