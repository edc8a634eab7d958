// CG cell term with warp-patch-local assembly and an asynchronous copy pipeline.
//
// Same arithmetic as cell_dfma_kernel.cuh (operator.py:255-278; DFMA point
// loop), reorganised around the locality that hierarchical reordering gives
// (PAPER.md:274-280).  The cells are cut into patches of 32 consecutive cells,
// one patch per warp iteration, one cell per lane.  A 32-cell patch of a
// reordered mesh touches few distinct DoFs (P1: ~0.2 per cell-DoF slot), so
// instead of N scattered global gathers and N global atomics per cell:
//
//   1. each patch is ONE contiguous, 16-byte aligned record in HBM
//        [G: 6 x 32 doubles, component-major] [local DoF indices: NW x 32 words]
//        [unique DoFs: nu ints] [incidence offsets: nu+1 u16 | contribution slots: u16]
//      copied into a 3-deep per-warp shared ring with 16-byte cp.async, two
//      patches ahead;
//   2. one patch ahead, the unique DoFs' u values are gathered from L2 with
//      8-byte cp.async into a double-buffered per-warp array;
//   3. the lanes read u and G from shared memory, run the point loop and write
//      their residuals to a per-warp contribution array sc[j][32];
//   4. lanes take the unique DoFs, sum their incidences in a fixed order and
//      issue ONE global RED per DoF.
//
// Only __syncwarp() separates the phases (no CTA barriers), so the latency of
// the prefetches is hidden by the other warps' compute.
#pragma once
#include "cell_dfma_kernel.cuh"

namespace tmf {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory");
}

template <int N, int Q>
struct PatchShape {
  using D = DfmaShape<N, Q, false>;
  static constexpr int NP = D::NP;
  static constexpr int CH = 32;             // cells per (warp) patch
  static constexpr int NW = NP / 2;         // 32-bit words of local indices per cell
  static constexpr int GEO_B = 6 * CH * 8;  // record layout (bytes)
  static constexpr int LID_B = NW * CH * 4;
  static constexpr int STAGES = 3;
  // per-warp shared bytes for a plan whose largest record is recmax bytes and whose
  // largest patch has numax unique DoFs (multiple of 2)
  __host__ __device__ static size_t warp_bytes(int recmax, int numax) {
    return (size_t)STAGES * recmax + (size_t)2 * numax * 8 + (size_t)N * CH * 8;
  }
  __host__ __device__ static size_t smem_bytes(int recmax, int numax, int warps) {
    return (size_t)2 * D::TAB * 8 + (size_t)warps * warp_bytes(recmax, numax);
  }
};

template <int N, int Q, int BLOCK, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) cell_patch_kernel(CellArgs a) {
  using S = PatchShape<N, Q>;
  using D = DfmaShape<N, Q, false>;
  constexpr int NP = S::NP, CH = S::CH, NW = S::NW, STAGES = S::STAGES, WARPS = BLOCK / 32;
  extern __shared__ __align__(16) unsigned char sbytes[];
  double* tab = reinterpret_cast<double*>(sbytes);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int recmax = a.recmax;                               // bytes, multiple of 16
  unsigned char* wbase = sbytes + 2 * D::TAB * 8 + wid * S::warp_bytes(recmax, a.numax);
  double* su = reinterpret_cast<double*>(wbase + STAGES * recmax);   // [2][numax]
  double* sc = su + 2 * a.numax;                                     // [N][32]
  {
    const double2* src = reinterpret_cast<const double2*>(a.frags);
    double2* dst = reinterpret_cast<double2*>(tab);
    for (int i = threadIdx.x; i < D::TAB; i += BLOCK) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const double2* T1 = reinterpret_cast<const double2*>(tab);
  const double2* T2 = reinterpret_cast<const double2*>(tab + D::TAB);

  // 32-bit patch arithmetic (n_cells < 2^31); components only when nc > 1
  const int cpc = (int)((a.n_cells + CH - 1) / CH);
  const int nch = cpc * a.nc;
  const int gw = blockIdx.x * WARPS + wid, nwarps = gridDim.x * WARPS;
  auto chunk = [&](int k) { return gw + k * nwarps; };
  auto comp_of = [&](int ch) { return a.nc == 1 ? 0 : ch / cpc; };
  auto meta = [&](int k) {   // {record offset (16 B units), nu, n incidences, record size (16 B)}
    const int ch = chunk(k);
    return ch < nch ? __ldg(a.pmeta + (ch - comp_of(ch) * cpc)) : make_int4(0, 0, 0, 0);
  };
  auto stage = [&](int k) { return wbase + (k % STAGES) * recmax; };
  auto issue_record = [&](int k, int4 m) {
    const uint4* src = reinterpret_cast<const uint4*>(a.prec) + m.x;
    uint4* dst = reinterpret_cast<uint4*>(stage(k));
    for (int i = lane; i < m.w; i += 32) cp_async16(dst + i, src + i);
  };
  auto issue_gather = [&](int k, int4 m) {
    const int ch = chunk(k);
    if (ch >= nch) return;
    const int comp = comp_of(ch);
    const int* pd = reinterpret_cast<const int*>(stage(k) + S::GEO_B + S::LID_B);
    double* dst = su + (k & 1) * a.numax;
    for (int i = lane; i < m.y; i += 32) cp_async8(dst + i, a.u + (int64_t)pd[i] * a.nc + comp);
  };

  int4 m0 = meta(0), m1 = meta(1);
  issue_record(0, m0);
  cp_async_commit();
  issue_record(1, m1);
  cp_async_commit();
  cp_async_wait<1>();   // record 0
  __syncwarp();
  issue_gather(0, m0);
  cp_async_commit();
  int4 m2 = meta(2);
  for (int k = 0; chunk(k) < nch; ++k) {
    const int comp = comp_of(chunk(k));
    cp_async_wait<0>();   // record k+1 and the u gather of patch k
    __syncwarp();
    issue_gather(k + 1, m1);
    issue_record(k + 2, m2);
    cp_async_commit();
    const int4 mk = m0;
    m0 = m1;
    m1 = m2;
    m2 = meta(k + 3);

    // ---- cells: one per lane
    const unsigned char* rec = stage(k);
    const double* sk = su + (k & 1) * a.numax;
    double uu[1][NP], yy[1][NP], G[1][6], md[1] = {0.0};
    {
      const uint32_t* lid = reinterpret_cast<const uint32_t*>(rec + S::GEO_B);
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        const uint32_t x = lid[w * CH + lane];
        const uint32_t l0 = x & 0xFFFFu, l1 = x >> 16;
        uu[0][2 * w] = l0 != 0xFFFFu ? sk[l0] : 0.0;
        uu[0][2 * w + 1] = l1 != 0xFFFFu ? sk[l1] : 0.0;
      }
      const double* geo = reinterpret_cast<const double*>(rec);
#pragma unroll
      for (int i = 0; i < 6; ++i) G[0][i] = geo[i * CH + lane];
    }
    dfma_cell_points<N, Q, false, 1>(T1, T2, uu, G, md, yy);
#pragma unroll
    for (int j = 0; j < N; ++j) sc[j * CH + lane] = yy[0][j];
    __syncwarp();

    // ---- unique DoFs: sum the incidences, one RED each
    {
      const int nu = mk.y;
      const int* pd = reinterpret_cast<const int*>(rec + S::GEO_B + S::LID_B);
      const uint16_t* ic = reinterpret_cast<const uint16_t*>(pd + ((nu + 3) & ~3));
      const uint16_t* pos = ic + ((nu + 1 + 7) & ~7);
      for (int i = lane; i < nu; i += 32) {
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
    __syncwarp();   // sc, su[k & 1] and the record stage are reused
  }
  cp_async_wait<0>();
}

}  // namespace tmf
