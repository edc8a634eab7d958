// CG Laplace cell term by BLOCK ASSEMBLY (low degrees, sm_100a): one CTA per block of B
// consecutive cells of a locality order the plan chooses (Morton order of the cell
// centroids), the block's unique DoFs gathered and scattered ONCE, the per-cell work on
// the FP64 vector pipe with the table operands in the constant bank.
//
// Restates the same cell loop as cell_kernel.cuh (operator.py:255-278; gather
// numpy_backend.py:23-35, E u :48-55, D :68-76, E^T :58-65, scatter_add :38-40) in the
// modal form of DESIGN §4: y_e = sum_m E'_m^T G_e (E'_m u_e), with the M = dim P_{p-1}
// unit-weight modes E'(k, m, j) built from the plan's own gradient tables and G_e =
// scale * kappa_e * det J * J^-1 J^-T recomputed from the cell's 4 vertices (the same
// affine_from_vertices / stiffness_metric as the other kernels).
//
// Why: at P1 / P2 the cell term is a few hundred flops per cell, and the tile kernels are
// bound by their per-cell-slot global traffic -- an fp64 RED and a gather per (cell, DoF)
// slot plus a 64 B geometry record per cell (round-1 ncu: P1 3.6x its algorithmic bytes,
// long-scoreboard stalls; P2 L1TEX 78 %).  On a compact block the DoFs are shared by many
// cells (P1: ~12 cells per vertex inside a 512-cell block), so
//   phase 1  the block's unique DoFs (sorted; the vertex DoFs -- ids < n_vertices in the
//            reference numbering, dofmap.py:113-114 -- come first) gather u and, for the
//            vertices, their coordinates into shared memory;
//   phase 2  one thread per cell: local DoF indices (u16), coordinates and u from shared
//            memory, G from the vertices, M x (3N + 9 + 3N) DFMAs whose E' operands are
//            kernel parameters (constant bank, warp-uniform), the cell's N results stored
//            to a shared slot array R[j][cell];
//   phase 3  one thread per unique DoF sums its slots (host-built incidence list, u16) in
//            a fixed order and issues ONE fp64 RED (Dirichlet DoFs: none).
// Global traffic per cell: 2 NP + 2 N bytes of u16 indices plus the unique-DoF lists,
// instead of 4 N + 64 bytes and N scattered REDs.
#pragma once
#include <cstdint>

#include "cell_kernel.cuh"
#include "common.cuh"

namespace tmf {

template <int N, int M>
struct BlockTab {
  double e[M * 3 * N];   // e[(m * 3 + k) * N + j] = E'(k, m, j)
};

struct BlockArgs {
  const double* __restrict__ u;
  double* __restrict__ y;
  const double* __restrict__ verts;
  const double* __restrict__ kappa;     // per processed cell (plan order), or nullptr
  const int* __restrict__ boff;         // (n_blocks + 1): block b's unique DoFs uniq[boff[b], boff[b+1])
  const int* __restrict__ bnv;          // (n_blocks): how many of them are vertices (at the front)
  const int* __restrict__ uniq;         // global DoF, ~g for Dirichlet DoFs (gathered 0, never written)
  const uint16_t* __restrict__ loc;     // (n_cells, NP) local DoF index per slot, processing order
  const uint16_t* __restrict__ inc;     // block b's B*N slot ids (j*B + cl), grouped by unique DoF
  const uint16_t* __restrict__ ioff;    // block b: nu_b + 1 offsets into its inc, at boff[b] + b
  int64_t n_cells;
  int64_t n_blocks;
  int numax, nvmax;                     // largest block: unique DoFs / vertex DoFs
  double scale;                         // stiff_scale
  double* energy;                       // += sum_e u_e^T A_e u_e (PCG's fused p.Ap), or nullptr
  TMF_DBG_FIELDS
};

template <int N>
struct BlockShape {
  static constexpr int NP = (N + 3) & ~3;   // loc row length (u16), 8-byte aligned rows
};

// dynamic shared memory: R[N*B] doubles | us[numax] | xs[3*nvmax] | (16-byte aligned)
// inc[N*B] u16 | ioff[numax+1] u16
__host__ __device__ inline size_t block_smem_doubles(int N, int B, int numax, int nvmax) {
  return (((size_t)N * B + numax + 3 * (size_t)nvmax) + 1) & ~(size_t)1;
}
__host__ __device__ inline size_t block_smem_bytes(int N, int B, int numax, int nvmax) {
  return sizeof(double) * block_smem_doubles(N, B, numax, nvmax) + sizeof(uint16_t) * ((size_t)N * B + numax + 1);
}

template <int N, int M, int BLOCK, int CPT, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) cell_block_kernel(BlockArgs a, const BlockTab<N, M> T) {
  constexpr int B = BLOCK * CPT;
  constexpr int NP = BlockShape<N>::NP;
  extern __shared__ __align__(16) double smem[];
  double* R = smem;                                   // R[j * B + cl]
  double* us = R + N * B;                             // u of the block's unique DoFs
  double* xs = us + a.numax;                          // vertex coordinates (x, y, z)
  uint16_t* sinc = reinterpret_cast<uint16_t*>(smem + block_smem_doubles(N, B, a.numax, a.nvmax));
  uint16_t* sioff = sinc + N * B;

  const int64_t b = blockIdx.x;
  const int off = __ldg(a.boff + b), nu = __ldg(a.boff + b + 1) - off, nv = __ldg(a.bnv + b);
  const int64_t c0 = b * B;
  const int ncb = (int)(a.n_cells - c0 < B ? a.n_cells - c0 : B);

  // the cells' local indices (and kappa) do not depend on phase 1: load them first, so
  // their latency overlaps the gathers
  uint2 lraw[CPT][NP / 4];
  double kap[CPT];
#pragma unroll
  for (int r = 0; r < CPT; ++r) {
    const int cl = threadIdx.x + r * BLOCK;
    const int64_t pc = c0 + (cl < ncb ? cl : 0);
    const uint2* lp = reinterpret_cast<const uint2*>(a.loc + pc * NP);
#pragma unroll
    for (int q = 0; q < NP / 4; ++q) lraw[r][q] = __ldg(lp + q);
    kap[r] = a.kappa ? a.scale * __ldg(a.kappa + pc) : a.scale;
  }

  // ---- phase 1: unique DoFs -> u, vertex coordinates; incidence lists -> shared
  // (two entries per thread per round: their loads are independent and issued together)
  for (int i0 = threadIdx.x; i0 < nu; i0 += 2 * BLOCK) {
    const int i1 = i0 + BLOCK;
    const int e0 = __ldg(a.uniq + off + i0);
    const int e1 = i1 < nu ? __ldg(a.uniq + off + i1) : -1;
    const int g0 = e0 < 0 ? ~e0 : e0, g1 = e1 < 0 ? ~e1 : e1;
    TMF_CHECK(a, g0 < a.dbg_n_dofs && (i1 >= nu || g1 < a.dbg_n_dofs), TMF_DBG_DOF);
    TMF_CHECK(a, nu <= a.numax && nv <= a.nvmax && nv <= nu, TMF_DBG_LOCAL);
    const double u0 = e0 < 0 ? 0.0 : __ldg(a.u + g0);
    const double u1 = e1 < 0 ? 0.0 : __ldg(a.u + g1);
    double x0[3], x1[3];
    if (i0 < nv) {
#pragma unroll
      for (int k = 0; k < 3; ++k) x0[k] = __ldg(a.verts + 3 * (int64_t)g0 + k);
    }
    if (i1 < nv) {
#pragma unroll
      for (int k = 0; k < 3; ++k) x1[k] = __ldg(a.verts + 3 * (int64_t)g1 + k);
    }
    us[i0] = u0;
    if (i1 < nu) us[i1] = u1;
    if (i0 < nv) {
#pragma unroll
      for (int k = 0; k < 3; ++k) xs[3 * i0 + k] = x0[k];
    }
    if (i1 < nv) {
#pragma unroll
      for (int k = 0; k < 3; ++k) xs[3 * i1 + k] = x1[k];
    }
  }
  {
    // the block's slot ids: B*N u16 at b*B*N (16-byte aligned for every b: B*N*2 % 16 == 0)
    const uint4* src = reinterpret_cast<const uint4*>(a.inc + b * (int64_t)B * N);
    uint4* dst = reinterpret_cast<uint4*>(sinc);
    const int n16 = (ncb * N + 7) / 8;
    for (int i = threadIdx.x; i < n16; i += BLOCK) dst[i] = __ldg(src + i);
    const uint16_t* io = a.ioff + off + b;
    for (int i = threadIdx.x; i <= nu; i += BLOCK) sioff[i] = __ldg(io + i);
  }
  __syncthreads();

  // ---- phase 2: one thread per cell
  double en = 0.0;
#pragma unroll
  for (int r = 0; r < CPT; ++r) {
    const int cl = threadIdx.x + r * BLOCK;
    if (cl >= ncb) break;
    uint16_t l[NP];
#pragma unroll
    for (int q = 0; q < NP / 4; ++q) {
      const uint2 v = lraw[r][q];
      l[4 * q] = (uint16_t)(v.x & 0xFFFFu);
      l[4 * q + 1] = (uint16_t)(v.x >> 16);
      l[4 * q + 2] = (uint16_t)(v.y & 0xFFFFu);
      l[4 * q + 3] = (uint16_t)(v.y >> 16);
    }
#pragma unroll
    for (int j = 0; j < N; ++j) TMF_CHECK(a, l[j] < nu && (j >= 4 || l[j] < nv), TMF_DBG_LOCAL);
    Vec3 x[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = Vec3{xs[3 * l[i]], xs[3 * l[i] + 1], xs[3 * l[i] + 2]};
    Affine g;
    affine_from_vertices(x[0], x[1], x[2], x[3], g);
    double G[6];
    stiffness_metric(g, kap[r], G);
    double uu[N], yy[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      uu[j] = us[l[j]];
      yy[j] = 0.0;
    }
#pragma unroll
    for (int m = 0; m < M; ++m) {
      double v0 = 0.0, v1 = 0.0, v2 = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        v0 = fma(T.e[(m * 3 + 0) * N + j], uu[j], v0);
        v1 = fma(T.e[(m * 3 + 1) * N + j], uu[j], v1);
        v2 = fma(T.e[(m * 3 + 2) * N + j], uu[j], v2);
      }
      const double d0 = G[0] * v0 + G[1] * v1 + G[2] * v2;
      const double d1 = G[1] * v0 + G[3] * v1 + G[4] * v2;
      const double d2 = G[2] * v0 + G[4] * v1 + G[5] * v2;
      en = fma(v0, d0, fma(v1, d1, fma(v2, d2, en)));
#pragma unroll
      for (int j = 0; j < N; ++j)
        yy[j] = fma(T.e[(m * 3 + 0) * N + j], d0,
                    fma(T.e[(m * 3 + 1) * N + j], d1, fma(T.e[(m * 3 + 2) * N + j], d2, yy[j])));
    }
#pragma unroll
    for (int j = 0; j < N; ++j) R[j * B + cl] = yy[j];
  }
  __syncthreads();

  // ---- phase 3: one thread per unique DoF, its slots summed in list order, one RED
  for (int i = threadIdx.x; i < nu; i += BLOCK) {
    const int e = __ldg(a.uniq + off + i);
    if (e < 0) continue;
    double s = 0.0;
    TMF_CHECK(a, sioff[i] <= sioff[i + 1] && sioff[i + 1] <= ncb * N && e < a.dbg_n_dofs, TMF_DBG_SLOT);
    for (int k = sioff[i]; k < sioff[i + 1]; ++k) {
      TMF_CHECK(a, sinc[k] < N * B && (int)(sinc[k] % B) < ncb, TMF_DBG_SLOT);
      s += R[sinc[k]];
    }
    atomicAdd(a.y + e, s);
  }
  if (a.energy != nullptr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) en += __shfl_xor_sync(0xffffffffu, en, o);
    if ((threadIdx.x & 31) == 0 && en != 0.0) atomicAdd(a.energy, en);
  }
}


// ===================================================================================
// Pipelined block assembly on FP64 tensor cores: cell_bpipe_kernel
//
// The same three phases as cell_block_kernel (unique-DoF gather, per-cell work, per-DoF
// reduction + one RED), with the per-cell work done by the modal DMMA tile of
// cell_kernel.cuh (8 cells per warp tile, A fragments read from the block's staged u,
// G from a per-block shared array), and the block's global loads PIPELINED across the
// blocks a persistent CTA walks:
//   contiguous data (unique DoFs, local indices, slot lists, offsets) of block k+2 and the
//   indirect gathers (u, vertex coordinates) of block k+1 are in flight, as cp.async
//   groups, while block k computes -- 3 stages of contiguous data, 2 of gathered data.
// Host layout (capi.cu build_blocks): per block a header {uniq offset, nu, nv, ioff offset}
// whose segments start 16-byte aligned, so every contiguous copy is 16-byte cp.async.
// ===================================================================================

struct BpipeLayout {
  int numax, nvmax, B, N, NP, NFRAG;
  // byte offsets in dynamic shared memory
  __host__ __device__ static int r16(int x) { return (x + 15) & ~15; }
  __host__ __device__ int frag_bytes() const { return NFRAG * 32 * 8; }
  __host__ __device__ int rstride() const { return B + 2; }   // doubles per R row (bank spread)
  __host__ __device__ int r_bytes() const { return N * rstride() * 8; }
  __host__ __device__ int g_bytes() const { return B * 6 * 8; }
  __host__ __device__ int gath_bytes() const { return r16((numax + 3 * nvmax) * 8); }
  __host__ __device__ int uq_bytes() const { return r16(numax * 4); }
  __host__ __device__ int loc_bytes() const { return r16(B * NP * 2); }
  __host__ __device__ int inc_bytes() const { return r16(B * N * 2); }
  __host__ __device__ int io_bytes() const { return r16((numax + 1) * 2); }
  __host__ __device__ int cont_bytes() const { return uq_bytes() + loc_bytes() + inc_bytes() + io_bytes(); }
  __host__ __device__ int off_r() const { return frag_bytes(); }
  __host__ __device__ int off_g() const { return off_r() + r_bytes(); }
  __host__ __device__ int off_gath(int s) const { return off_g() + g_bytes() + s * gath_bytes(); }
  __host__ __device__ int off_cont(int s) const { return off_gath(2) + s * cont_bytes(); }
  __host__ __device__ int total() const { return off_cont(3); }
};

struct BpipeArgs {
  const double* __restrict__ u;
  double* __restrict__ y;
  const double* __restrict__ verts;
  const double* __restrict__ kappa;     // per processed cell (plan order), or nullptr
  const double* __restrict__ frags;     // modal DMMA fragments (CellShape<N, M, false> layout)
  const int4* __restrict__ head;        // (n_blocks): {uniq offset, nu, nv, ioff offset}, offsets 16-B aligned
  const int* __restrict__ uniq;         // global DoF, ~g for Dirichlet DoFs
  const uint16_t* __restrict__ loc;     // (n_cells, NP) local DoF index per slot, processing order
  const uint16_t* __restrict__ inc;     // block b's B*N slot ids (j*B + cl), grouped by unique DoF
  const uint16_t* __restrict__ ioff;    // block b: nu_b + 1 offsets into its slot list
  int64_t n_cells;
  int64_t n_blocks;
  int numax, nvmax;
  double scale;
  double* energy;
  TMF_DBG_FIELDS
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool ok) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <int N, int M, int BLOCK, int B>
__global__ void __launch_bounds__(BLOCK, 1) cell_bpipe_kernel(BpipeArgs a) {
  using S = CellShape<N, M, false>;
  constexpr int NP = BlockShape<N>::NP;
  constexpr int MT = S::MT;
  constexpr int NT = B / 8;                   // 8-cell tiles per block
  constexpr int NW = BLOCK / 32;
  static_assert(B % 8 == 0 && (B & (B - 1)) == 0, "block size");
  extern __shared__ __align__(16) unsigned char sm[];
  const BpipeLayout L{a.numax, a.nvmax, B, N, NP, S::NFRAG};
  double* sF = reinterpret_cast<double*>(sm);
  double* sR = reinterpret_cast<double*>(sm + L.off_r());
  double* sG = reinterpret_cast<double*>(sm + L.off_g());
  constexpr int RS = B + 2;
  {
    const double2* src = reinterpret_cast<const double2*>(a.frags);
    double2* dst = reinterpret_cast<double2*>(sF);
    for (int i = threadIdx.x; i < S::NFRAG * 16; i += BLOCK) dst[i] = __ldg(src + i);
  }
  const double* sB1 = sF;
  const double* sB2 = sF + S::NB1 * 32;
  auto cont_uq = [&](int s) { return reinterpret_cast<int*>(sm + L.off_cont(s)); };
  auto cont_loc = [&](int s) { return reinterpret_cast<uint16_t*>(sm + L.off_cont(s) + L.uq_bytes()); };
  auto cont_inc = [&](int s) {
    return reinterpret_cast<uint16_t*>(sm + L.off_cont(s) + L.uq_bytes() + L.loc_bytes());
  };
  auto cont_io = [&](int s) {
    return reinterpret_cast<uint16_t*>(sm + L.off_cont(s) + L.uq_bytes() + L.loc_bytes() + L.inc_bytes());
  };
  auto gath_u = [&](int s) { return reinterpret_cast<double*>(sm + L.off_gath(s)); };
  auto gath_x = [&](int s) { return reinterpret_cast<double*>(sm + L.off_gath(s)) + a.numax; };

  // contiguous data of block b into stage s (16-byte copies; the host pads every segment)
  auto issue_cont = [&](int64_t b, int s) {
    const int4 h = __ldg(a.head + b);
    const int64_t c0 = b * B;
    const int ncb = (int)(a.n_cells - c0 < B ? a.n_cells - c0 : B);
    const int nu = h.y;
    {
      const int n16 = (nu + 3) / 4;
      const int4* src = reinterpret_cast<const int4*>(a.uniq + h.x);
      int4* dst = reinterpret_cast<int4*>(cont_uq(s));
      for (int i = threadIdx.x; i < n16; i += BLOCK) cp_async16(dst + i, src + i);
    }
    {
      const int n16 = (ncb * NP * 2 + 15) / 16;
      const int4* src = reinterpret_cast<const int4*>(a.loc + c0 * NP);
      int4* dst = reinterpret_cast<int4*>(cont_loc(s));
      for (int i = threadIdx.x; i < n16; i += BLOCK) cp_async16(dst + i, src + i);
    }
    {
      const int n16 = (ncb * N * 2 + 15) / 16;
      const int4* src = reinterpret_cast<const int4*>(a.inc + b * (int64_t)B * N);
      int4* dst = reinterpret_cast<int4*>(cont_inc(s));
      for (int i = threadIdx.x; i < n16; i += BLOCK) cp_async16(dst + i, src + i);
    }
    {
      const int n16 = ((nu + 1) * 2 + 15) / 16;
      const int4* src = reinterpret_cast<const int4*>(a.ioff + h.w);
      int4* dst = reinterpret_cast<int4*>(cont_io(s));
      for (int i = threadIdx.x; i < n16; i += BLOCK) cp_async16(dst + i, src + i);
    }
  };
  // indirect gathers of block b (its unique DoFs in contiguous stage sc) into gather stage sg
  auto issue_gath = [&](int64_t b, int sc, int sg) {
    const int4 h = __ldg(a.head + b);
    const int* uq = cont_uq(sc);
    double* us = gath_u(sg);
    double* xs = gath_x(sg);
    for (int i = threadIdx.x; i < h.y; i += BLOCK) {
      const int e = uq[i];
      const int g = e < 0 ? ~e : e;
      TMF_CHECK(a, g < a.dbg_n_dofs && h.y <= a.numax && h.z <= a.nvmax, TMF_DBG_DOF);
      cp_async8(us + i, a.u + g, e >= 0);
      if (i < h.z) {
#pragma unroll
        for (int k = 0; k < 3; ++k) cp_async8(xs + 3 * i + k, a.verts + 3 * (int64_t)g + k, true);
      }
    }
  };

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cs = lane >> 2, q4 = lane & 3;
  double en = 0.0;
  const int64_t b0 = blockIdx.x, bstep = gridDim.x;
  // prologue: contiguous data of the first two blocks, the gathers of the first
  if (b0 < a.n_blocks) issue_cont(b0, 0);
  cp_commit();
  if (b0 + bstep < a.n_blocks) issue_cont(b0 + bstep, 1);
  cp_commit();
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  __syncthreads();
  if (b0 < a.n_blocks) issue_gath(b0, 0, 0);
  cp_commit();

  int k = 0;
  for (int64_t b = b0; b < a.n_blocks; b += bstep, ++k) {
    const int sc = k % 3, sg = k & 1;
    cp_wait_all();       // this block's gathers and the next block's contiguous data
    __syncthreads();
    if (b + bstep < a.n_blocks) issue_gath(b + bstep, (k + 1) % 3, sg ^ 1);
    cp_commit();
    if (b + 2 * bstep < a.n_blocks) issue_cont(b + 2 * bstep, (k + 2) % 3);
    cp_commit();

    const int4 h = __ldg(a.head + b);
    const int64_t c0 = b * B;
    const int ncb = (int)(a.n_cells - c0 < B ? a.n_cells - c0 : B);
    const uint16_t* loc = cont_loc(sc);
    const double* us = gath_u(sg);
    const double* xs = gath_x(sg);

    // ---- geometry: G per cell from its 4 staged vertices
    for (int cl = threadIdx.x; cl < ncb; cl += BLOCK) {
      const uint16_t* l = loc + cl * NP;
      Vec3 x[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        TMF_CHECK(a, l[i] < h.z, TMF_DBG_LOCAL);
        x[i] = Vec3{xs[3 * l[i]], xs[3 * l[i] + 1], xs[3 * l[i] + 2]};
      }
      Affine g;
      affine_from_vertices(x[0], x[1], x[2], x[3], g);
      double G[6];
      stiffness_metric(g, a.kappa ? a.scale * __ldg(a.kappa + c0 + cl) : a.scale, G);
      double2* o = reinterpret_cast<double2*>(sG + 6 * cl);
      o[0] = make_double2(G[0], G[1]);
      o[1] = make_double2(G[2], G[3]);
      o[2] = make_double2(G[4], G[5]);
    }
    __syncthreads();

    // ---- DMMA tiles: 8 cells per warp tile, MT tiles per warp iteration
    for (int st = warp; st * MT < NT; st += NW) {
      int cell[MT];
      bool valid[MT];
      double av[MT][S::KK], G[MT][6];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        cell[m] = (st * MT + m) * 8 + cs;
        valid[m] = (st * MT + m) < NT && cell[m] < ncb;
        const int cl = valid[m] ? cell[m] : 0;
#pragma unroll
        for (int kk = 0; kk < S::KK; ++kk) {
          const int j = 4 * kk + q4;
          double v = 0.0;
          if (valid[m] && j < N) {
            const int li = loc[cl * NP + j];
            TMF_CHECK(a, li < h.y, TMF_DBG_LOCAL);
            v = us[li];
          }
          av[m][kk] = v;
        }
        const double2* gp = reinterpret_cast<const double2*>(sG + 6 * cl);
        const double2 g01 = gp[0], g23 = gp[1], g45 = gp[2];
        G[m][0] = g01.x; G[m][1] = g01.y; G[m][2] = g23.x;
        G[m][3] = g23.y; G[m][4] = g45.x; G[m][5] = g45.y;
      }
      double yacc[MT][S::NJ][2];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int nj = 0; nj < S::NJ; ++nj) yacc[m][nj][0] = yacc[m][nj][1] = 0.0;
      auto dact = [&](int m, double g0, double g1, double g2, double& d0, double& d1, double& d2) {
        d0 = G[m][0] * g0 + G[m][1] * g1 + G[m][2] * g2;
        d1 = G[m][1] * g0 + G[m][3] * g1 + G[m][4] * g2;
        d2 = G[m][2] * g0 + G[m][4] * g1 + G[m][5] * g2;
        en = fma(g0, d0, fma(g1, d1, fma(g2, d2, en)));
      };
#pragma unroll
      for (int t = 0; t < S::T; ++t) {
        double v[MT][3][2];
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int c = 0; c < 3; ++c) v[m][c][0] = v[m][c][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < S::KK; ++kk)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const double bb = sB1[((t * 3 + c) * S::KK + kk) * 32 + lane];
#pragma unroll
            for (int m = 0; m < MT; ++m) dmma(v[m][c], av[m][kk], bb);
          }
        double d[MT][3][2];
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int i = 0; i < 2; ++i) dact(m, v[m][0][i], v[m][1][i], v[m][2][i], d[m][0][i], d[m][1][i], d[m][2][i]);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int nj = 0; nj < S::NJ; ++nj) {
              const double bb = sB2[(((t * 3 + c) * 2 + i) * S::NJ + nj) * 32 + lane];
#pragma unroll
              for (int m = 0; m < MT; ++m) dmma(yacc[m][nj], d[m][c][i], bb);
            }
      }
      if (S::GRP) {
        double v[MT][2][2];
#pragma unroll
        for (int m = 0; m < MT; ++m) v[m][0][0] = v[m][0][1] = v[m][1][0] = v[m][1][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < S::KK; ++kk)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const double bb = sB1[(S::NB1T + hh * S::KK + kk) * 32 + lane];
#pragma unroll
            for (int m = 0; m < MT; ++m) dmma(v[m][hh], av[m][kk], bb);
          }
        double d[MT][3];
#pragma unroll
        for (int m = 0; m < MT; ++m) dact(m, v[m][0][0], v[m][0][1], v[m][1][0], d[m][0], d[m][1], d[m][2]);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int nj = 0; nj < S::NJ; ++nj) {
            const double bb = sB2[(S::NB2T + c * S::NJ + nj) * 32 + lane];
#pragma unroll
            for (int m = 0; m < MT; ++m) dmma(yacc[m][nj], d[m][c], bb);
          }
      }
      // lane owns output DoFs 8nj + 2q4 + {0,1} of its cell: to the slot array
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        if (!valid[m]) continue;
#pragma unroll
        for (int nj = 0; nj < S::NJ; ++nj)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int j = 8 * nj + 2 * q4 + i;
            if (j < N) sR[j * RS + cell[m]] = yacc[m][nj][i];
          }
      }
    }
    __syncthreads();

    // ---- one thread per unique DoF: its slots in list order, one RED
    {
      const int* uq = cont_uq(sc);
      const uint16_t* sinc = cont_inc(sc);
      const uint16_t* sio = cont_io(sc);
      for (int i = threadIdx.x; i < h.y; i += BLOCK) {
        const int e = uq[i];
        if (e < 0) continue;
        double s = 0.0;
        TMF_CHECK(a, sio[i] <= sio[i + 1] && sio[i + 1] <= ncb * N, TMF_DBG_SLOT);
        for (int q = sio[i]; q < sio[i + 1]; ++q) {
          const int slot = sinc[q];
          TMF_CHECK(a, slot < N * B && (slot & (B - 1)) < ncb, TMF_DBG_SLOT);
          s += sR[(slot / B) * RS + (slot & (B - 1))];
        }
        atomicAdd(a.y + e, s);
      }
    }
    __syncthreads();     // stage sc / sg, sG and sR are free for the next blocks
  }
  cp_wait_all();
  if (a.energy != nullptr) {
    // DMMA lanes accumulate two points' g.(G g) per 8-point tile once; the geometry threads none
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) en += __shfl_xor_sync(0xffffffffu, en, o);
    if (lane == 0 && en != 0.0) atomicAdd(a.energy, en);
  }
}

}  // namespace tmf
