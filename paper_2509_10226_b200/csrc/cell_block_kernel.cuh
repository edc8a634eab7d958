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
  pdl_wait_prior_grid();   // y cleared (common.cuh); phases 1-2 do not touch y
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

}  // namespace tmf
