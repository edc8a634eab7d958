// Cell-term kernel of the matrix-free apply on FP64 tensor cores (sm_100a).
//
// Restates the reference cell loop (operator.py:255-278):
//     U = gather(u)                      numpy_backend.py:23-35
//     V = E_grad @ U                     numpy_backend.py:48-55
//     D = J^-1 (jxw * J^-T V)            numpy_backend.py:68-76
//     R = E_grad^T @ D  (+ E_val^T (mass_scale jxw E_val U))  :58-65, :86-88
//     y += scatter(R)                    numpy_backend.py:38-40
// as two chained DMMA GEMMs per warp over a tile of 8 cells (M = cells):
//
//   GEMM1  V^T[8 cells, (t,c,pt)] = U^T[8, N] . E^T[N, (t,c,pt)]
//          component-major point tiles: tile (t, c) holds component c of the
//          8 quadrature points 8t..8t+7, so each lane ends up owning ALL
//          components of points 8t + 2(lane&3) + {0,1} for its cell;
//   D      in registers: d = w_q (G g)  (w_q folded into the GEMM2 table)
//   GEMM2  Y^T[8, N] += D^T[8, (t,c,i,lane&3)] . Ew[(t,c,i,k), N]
//          the C fragment of GEMM1 *is* the A fragment of GEMM2 once the K
//          index of GEMM2 is ordered (t, c, i, lane&3): no shuffles, no smem.
//          GEMM2's output columns are ordered so that column 2q+i of n-tile nj is
//          DoF 4(2nj+i)+q: a lane ends up with the results of exactly the DoFs
//          4kk + (lane&3) whose u it gathered, and scatters them through the index
//          registers of the gather (no second index load).
//
// Both B operands are constant tables, pre-swizzled on the host into
// lane-major fragments (frag[f][lane]) and staged once per CTA in shared
// memory (one conflict-free LDS.64 per DMMA).  Per-cell geometry (6 entries
// of G = det J^-1 J^-T, plus the mass factor) is precomputed once per plan by
// cell_geometry_kernel and read as 64 B per cell.
//
// CG: masked (Dirichlet) DoFs are encoded as ~idx (< 0): gathered as 0 and
// never scattered (operator.py:327-328 fixes y on them afterwards).  The
// scatter uses fp64 RED (red.global.add.f64); DG cells own their DoFs, so
// the DG variant stores y directly and the face kernel adds onto it.
#pragma once
#include "common.cuh"

namespace tmf {

struct CellArgs {
  const double* __restrict__ u;
  double* __restrict__ y;
  const int* __restrict__ dofs;    // CG: (n_cells, N) encoded; DG: nullptr (contiguous)
  const double* __restrict__ cgeo; // (n_cells, 8): G[6] (scaled), mass factor, 0
  const double* __restrict__ frags;  // B1 then B2 fragments (global; staged to smem)
  int64_t n_cells;
  int nc;                          // interleaved components
  // kernel-parameter layout: the cell kernels' code generation depends on it (a tighter
  // struct measured 4-9 % slower at P3 / P4, same SASS otherwise); keep these reserved slots
  int reserved0 = 0;
  const void* reserved1[2] = {nullptr, nullptr};
  int reserved2[2] = {0, 0};
  PeerArgs peer;                   // multi-GPU: ghost DoFs read / scattered over peer memory
  double* energy = nullptr;        // CG tensor / modal engines: += sum_e u_e^T A_e u_e (PCG's p.Ap)
  const double* reserved3 = nullptr;
  TMF_DBG_FIELDS
};

// Per-cell geometry, computed once per plan by cell_geometry_kernel (the
// reference stores J^-T and JxW per cell, geometry.py:145-151; 8 doubles here):
//   G = stiff_scale * kappa_e * det J * J^-1 J^-T  (packed 00,01,02,11,12,22)
//   m = mass_scale * det J
struct CellGeoArgs {
  const int* __restrict__ cells;
  const double* __restrict__ verts;
  const double* __restrict__ kappa;
  double* __restrict__ cgeo;
  int64_t n_cells;
  double stiff_scale;
  double mass_scale;
};

static __global__ void cell_geometry_kernel(CellGeoArgs a) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.n_cells;
       e += (int64_t)gridDim.x * blockDim.x) {
    int vid[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) vid[i] = __ldg(a.cells + 4 * e + i);
    Affine g;
    affine_from_vertices(load_vertex(a.verts, vid[0]), load_vertex(a.verts, vid[1]),
                         load_vertex(a.verts, vid[2]), load_vertex(a.verts, vid[3]), g);
    double sc = a.stiff_scale;
    if (a.kappa) sc *= a.kappa[e];
    double G[6];
    stiffness_metric(g, sc, G);
    double* o = a.cgeo + 8 * e;
#pragma unroll
    for (int i = 0; i < 6; ++i) o[i] = G[i];
    o[6] = a.mass_scale * g.det;
    o[7] = 0.0;
  }
}

// MM: the mass term as its own GEMM (modal Helmholtz): Y += diag(m_e) U M with the exact
// reference mass matrix M = sum_q w_q phi_i phi_j as KK x NJ more table fragments
template <int N, int Q, bool MASS, bool MM = false>
struct CellShape {
  static constexpr int KK = (N + 3) / 4;     // GEMM1 k-steps (DoFs)
  static constexpr int NJ = (N + 7) / 8;     // GEMM2 n-tiles (DoFs)
  static constexpr int NC = MASS ? 4 : 3;    // value (mass) + 3 reference gradients
  // Points: T full 8-point tiles; a remainder of 1..4 points goes to one 4-point
  // group (GEMM1 columns (point, component) with components padded to 4, the
  // face-kernel layout), which takes 2 KK + NC NJ DMMAs instead of the
  // NC KK + 2 NC NJ of an 8-point tile (P3, n_q 35: 165 -> 151 per tile).
  // A remainder of 1..2 points goes to one 2-point pair group: ONE 8-column GEMM1 tile
  // with columns (point, component padded to 4); a lane holds two components of its
  // point and gets the others from its neighbour lane with one shuffle each, so the
  // pair takes KK + 2 NJ DMMAs (modal P3, 10 modes: 52 -> 44 per tile).
  static constexpr int R = Q % 8;
  static constexpr bool PAIR = R >= 1 && R <= 2;
  static constexpr bool GRP = R >= 3 && R <= 4;
  static constexpr int T = (GRP || PAIR) ? Q / 8 : (Q + 7) / 8;
  static constexpr int NB1T = T * NC * KK;   // GEMM1 fragments of the 8-point tiles
  static constexpr int NB2T = T * NC * 2 * NJ;
  static constexpr int NB1 = NB1T + (GRP ? 2 * KK : 0) + (PAIR ? KK : 0);
  static constexpr int NB2 = NB2T + (GRP ? NC * NJ : 0) + (PAIR ? 2 * NJ : 0);
  static constexpr int NB3 = MM ? KK * NJ : 0;   // mass-matrix fragments
  static constexpr int NFRAG = NB1 + NB2 + NB3;
  static constexpr int SMEM = NFRAG * 32 * 8;
  static constexpr int DMMA_PER_TILE = NB1 + NB2 + NB3;
  // tiles per warp iteration: two independent 8-cell tiles share every B
  // fragment load (half the LDS traffic) and double the DMMA chains in flight
  static constexpr int MT = (KK + 2 * NJ) <= 7 ? 2 : 1;
};

// PEER: ghost DoFs through peer memory (multi-GPU, CellArgs::peer); a separate
// instantiation so the single-GPU kernel carries no ghost test (it costs 10-20 %)
// AS: asynchronous gather pipeline with AS stages -- each warp cp.async's the gathered u
// (8-byte copies, zero-filled for masked DoFs) and the 64-byte geometry records of the
// super-tile AS-1 ahead into its own shared-memory ring, so AS-1 tiles' loads are in
// flight without holding registers (measured: pays at P4 only)
// MT_: 8-cell tiles per warp iteration sharing every B-fragment load (0 = CellShape::MT)
// MM: mass term as a separate GEMM on the gathered u (CellShape; Helmholtz on the modal tables)
// GS (kernels without the ring): the geometry records of the NEXT super-tile are staged one
// iteration ahead into a per-warp shared-memory slot (one coalesced 16-byte cp.async per lane)
// and read back as broadcast LDS.64s, instead of three LDG.128s per lane at the tile start
template <int N, int Q, bool MASS, bool DG, int BLOCK, bool PEER = false, int AS = 0, int MT_ = 0, bool MM = false,
          bool GS = false>
__global__ void __launch_bounds__(BLOCK, 1) cell_apply_kernel(CellArgs a) {
  static_assert(!GS || AS == 0, "the ring stages the geometry itself");
  static_assert(!(MASS && MM), "the mass term is either in the point loop or a separate GEMM");
  using S = CellShape<N, Q, MASS, MM>;
  constexpr int MT = MT_ ? MT_ : S::MT;
  static_assert(AS == 0 || !PEER, "the async ring has no peer gathers");
  extern __shared__ __align__(16) double smem[];
  {
    const double2* src = reinterpret_cast<const double2*>(a.frags);
    double2* dst = reinterpret_cast<double2*>(smem);
    for (int i = threadIdx.x; i < S::NFRAG * 16; i += BLOCK) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const double* sB1 = smem;
  const double* sB2 = smem + S::NB1 * 32;
  const int lane = threadIdx.x & 31;
  auto B1 = [&](int f) -> double { return sB1[f * 32 + lane]; };
  auto B2 = [&](int f) -> double { return sB2[f * 32 + lane]; };

  const int cs = lane >> 2;  // cell slot in the tile
  const int q4 = lane & 3;
  const int64_t ctiles = (a.n_cells + 7) / 8;
  const int64_t cst = (ctiles + MT - 1) / MT;       // super-tiles per component
  const int64_t nst = cst * a.nc;
  const int64_t nwarps = (int64_t)gridDim.x * (BLOCK / 32);

  // Index prefetch: the DoF indices of the warp's next super-tile are loaded
  // while the current one computes, so each start pays one memory round trip
  // (u and the per-cell geometry, issued together) instead of two.
  int64_t st = (int64_t)blockIdx.x * (BLOCK / 32) + (threadIdx.x >> 5);
  const int64_t step = nwarps;
  int nidx[MT][S::KK];
  auto load_indices = [&](int64_t t) {
    const int cmp = a.nc == 1 ? 0 : (int)(t / cst);
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int64_t c = ((t - (int64_t)cmp * cst) * MT + m) * 8 + cs;
      const bool ok = t < nst && c < a.n_cells;
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk) {
        const int j = 4 * kk + q4;
        nidx[m][kk] = -1;
        if (ok && j < N) nidx[m][kk] = DG ? (int)(c * N + j) : __ldg(a.dofs + c * N + j);
      }
    }
  };
  // gathered u (A fragments) and geometry of one super-tile, from the indices in nidx
  auto load_data = [&](int64_t t, double (&av)[MT][S::KK], double (&G)[MT][6], double (&mdet)[MT]) {
    const int cmp = a.nc == 1 ? 0 : (int)(t / cst);
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int64_t c = ((t - (int64_t)cmp * cst) * MT + m) * 8 + cs;
      const bool ok = t < nst && c < a.n_cells;
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk) {
        const int g = nidx[m][kk];
        TMF_CHECK(a, g < 0 || (int64_t)g * a.nc + cmp < a.dbg_n_dofs, TMF_DBG_DOF);
        TMF_CHECK(a, !ok || c < a.dbg_n_cells, TMF_DBG_CELL);
        if (PEER)
          av[m][kk] = (g >= 0) ? __ldg(peer_src(a.peer, a.u, g, a.nc, cmp)) : 0.0;
        else
          av[m][kk] = (g >= 0) ? __ldg(a.u + (int64_t)g * a.nc + cmp) : 0.0;
      }
      if (!GS) {
        const double2* gp = reinterpret_cast<const double2*>(a.cgeo + 8 * (ok ? c : 0));
        const double2 g01 = __ldg(gp), g23 = __ldg(gp + 1), g45 = __ldg(gp + 2);
        G[m][0] = g01.x; G[m][1] = g01.y; G[m][2] = g23.x;
        G[m][3] = g23.y; G[m][4] = g45.x; G[m][5] = g45.y;
        mdet[m] = (MASS || MM) ? __ldg(a.cgeo + 8 * (ok ? c : 0) + 6) : 0.0;
      }
    }
  };
  // GS: two slots of MT x 64 doubles per warp behind the tables
  double* sgeo = smem + S::NFRAG * 32 + (threadIdx.x >> 5) * 2 * MT * 64;
  int gslot = 0;
  auto stage_geo = [&](int64_t t) {   // records of super-tile t into the other slot
    const int cmp = a.nc == 1 ? 0 : (int)(t / cst);
    gslot ^= 1;
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int64_t c = ((t - (int64_t)cmp * cst) * MT + m) * 8 + cs;
      const bool ok = t < nst && c < a.n_cells;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(sgeo + (gslot * MT + m) * 64 + cs * 8 + 2 * q4)),
                   "l"(a.cgeo + 8 * (ok ? c : 0) + 2 * q4), "r"(ok ? 16 : 0) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  // async ring: per stage MT x (KK x 32 gathered u, 8 cells x 8 geometry doubles, and the
  // KK x 32 gather indices as ints, read back by the scatter)
  constexpr int STAGE = MT * (S::KK * 32 + 64 + S::KK * 16);
  double* ring = smem + S::NFRAG * 32 + (threadIdx.x >> 5) * (AS > 0 ? AS : 1) * STAGE;
  auto issue = [&](int64_t t, int slot) {
    double* r = ring + slot * STAGE;
    const int cmp = a.nc == 1 ? 0 : (int)(t / cst);
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      const int64_t c = ((t - (int64_t)cmp * cst) * MT + m) * 8 + cs;
      const bool ok = t < nst && c < a.n_cells;
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk) {
        const int g = nidx[m][kk];
        TMF_CHECK(a, g < 0 || (int64_t)g * a.nc + cmp < a.dbg_n_dofs, TMF_DBG_DOF);
        const double* src = g >= 0 ? a.u + (int64_t)g * a.nc + cmp : a.u;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(r + (m * S::KK + kk) * 32 + lane)),
                     "l"(src), "r"(g >= 0 ? 8 : 0) : "memory");
        if (!DG) reinterpret_cast<int*>(r + MT * (S::KK * 32 + 64))[(m * S::KK + kk) * 32 + lane] = g;
      }
      // lane copies 16-byte piece q4 of its cell's 64-byte geometry record
      const double* gsrc = a.cgeo + 8 * (ok ? c : 0) + 2 * q4;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(r + MT * S::KK * 32 + m * 64 + cs * 8 + 2 * q4)),
                   "l"(gsrc), "r"(ok ? 16 : 0) : "memory");
    }
  };
  load_indices(st);
  if (GS) stage_geo(st);
  int slot = 0;
  if (AS > 0) {
#pragma unroll
    for (int s = 0; s < AS - 1; ++s) {
      issue(st + s * step, s);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      load_indices(st + (s + 1) * step);
    }
  }
  // sum over the lane's points of g . (G g) = u_e^T A_e u_e when the point weights are 1:
  // compiled for the modal tables only (fewer "points" than DoFs), CG; CellArgs::energy
  constexpr bool EN = !DG && Q < N;
  double en = 0.0;

  if (!DG) pdl_wait_prior_grid();   // y cleared (common.cuh); nothing above touches y
  for (; st < nst; st += step) {
    const int comp = a.nc == 1 ? 0 : (int)(st / cst);
    int64_t cell[MT];
    bool valid[MT];
    double av[MT][S::KK];
    double G[MT][6];
    double mdet[MT];
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      cell[m] = ((st - (int64_t)comp * cst) * MT + m) * 8 + cs;
      valid[m] = cell[m] < a.n_cells;
    }
    int cidx[MT][S::KK];               // this tile's gather indices (CG scatter; AS: in the ring slot)
    const int* ridx = nullptr;
    if (AS > 0) {
      // refill the slot of tile st + (AS-1) step (the slot the previous tile was read
      // from: every lane has its values in registers), then wait for this tile's group
      __syncwarp();
      issue(st + (AS - 1) * step, (slot + AS - 1) % AS);
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      load_indices(st + AS * step);
      asm volatile("cp.async.wait_group %0;\n" ::"n"(AS > 0 ? AS - 1 : 0) : "memory");
      __syncwarp();
      const double* r = ring + slot * STAGE;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
#pragma unroll
        for (int kk = 0; kk < S::KK; ++kk) av[m][kk] = r[(m * S::KK + kk) * 32 + lane];
        const double* gg = r + MT * S::KK * 32 + m * 64 + cs * 8;
#pragma unroll
        for (int i = 0; i < 6; ++i) G[m][i] = gg[i];
        mdet[m] = (MASS || MM) ? gg[6] : 0.0;
      }
      ridx = reinterpret_cast<const int*>(r + MT * (S::KK * 32 + 64));   // refilled only next iteration
      slot = slot + 1 == AS ? 0 : slot + 1;
    } else {
      load_data(st, av, G, mdet);
      if (GS) {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
#pragma unroll
        for (int m = 0; m < MT; ++m) {
          const double* gg = sgeo + (gslot * MT + m) * 64 + cs * 8;
#pragma unroll
          for (int i = 0; i < 6; ++i) G[m][i] = gg[i];
          mdet[m] = (MASS || MM) ? gg[6] : 0.0;
        }
        stage_geo(st + step);   // the other slot: read two iterations ago
      }
      if (!DG) {
#pragma unroll
        for (int m = 0; m < MT; ++m)
#pragma unroll
          for (int kk = 0; kk < S::KK; ++kk) cidx[m][kk] = nidx[m][kk];
      }
      load_indices(st + step);
    }

    double yacc[MT][S::NJ][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
      for (int nj = 0; nj < S::NJ; ++nj) yacc[m][nj][0] = yacc[m][nj][1] = 0.0;
    if (MM) {
      // mass term: (U M) rows scaled by the cell's m_e = mass_scale det J (operator.py:86-88)
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk)
#pragma unroll
        for (int nj = 0; nj < S::NJ; ++nj) {
          const double b = sB2[(S::NB2 + kk * S::NJ + nj) * 32 + lane];
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma(yacc[m][nj], av[m][kk], b);
        }
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int nj = 0; nj < S::NJ; ++nj) {
          yacc[m][nj][0] *= mdet[m];
          yacc[m][nj][1] *= mdet[m];
        }
    }

    auto gemm1 = [&](int t, double (&v)[MT][S::NC][2]) {
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int c = 0; c < S::NC; ++c) v[m][c][0] = v[m][c][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk) {
#pragma unroll
        for (int c = 0; c < S::NC; ++c) {
          const double b = B1((t * S::NC + c) * S::KK + kk);
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma(v[m][c], av[m][kk], b);
        }
      }
    };
    // D action at the lane's two points (w_q lives in the GEMM2 table), then GEMM2
    auto daction_gemm2 = [&](int t, const double (&v)[MT][S::NC][2]) {
      double d[MT][S::NC][2];
#pragma unroll
      for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          constexpr int o = MASS ? 1 : 0;
          const double g0 = v[m][o][i], g1 = v[m][o + 1][i], g2 = v[m][o + 2][i];
          d[m][o][i] = G[m][0] * g0 + G[m][1] * g1 + G[m][2] * g2;
          d[m][o + 1][i] = G[m][1] * g0 + G[m][3] * g1 + G[m][4] * g2;
          d[m][o + 2][i] = G[m][2] * g0 + G[m][4] * g1 + G[m][5] * g2;
          if (MASS) d[m][0][i] = mdet[m] * v[m][0][i];
          if (EN) en = fma(g0, d[m][o][i], fma(g1, d[m][o + 1][i], fma(g2, d[m][o + 2][i], en)));
        }
#pragma unroll
      for (int c = 0; c < S::NC; ++c)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int nj = 0; nj < S::NJ; ++nj) {
            const double b = B2(((t * S::NC + c) * 2 + i) * S::NJ + nj);
#pragma unroll
            for (int m = 0; m < MT; ++m) dmma(yacc[m][nj], d[m][c][i], b);
          }
    };
    // remainder 4-point group: lane owns point 8T + q4 (components 2h + i)
    auto gemm1g = [&](double (&v)[MT][2][2]) {
#pragma unroll
      for (int m = 0; m < MT; ++m) v[m][0][0] = v[m][0][1] = v[m][1][0] = v[m][1][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double b = B1(S::NB1T + h * S::KK + kk);
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma(v[m][h], av[m][kk], b);
        }
    };
    auto dgemm2g = [&](const double (&v)[MT][2][2]) {
      double d[MT][S::NC];
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        constexpr int o = MASS ? 1 : 0;
        const double c[4] = {v[m][0][0], v[m][0][1], v[m][1][0], v[m][1][1]};
        const double g0 = c[o], g1 = c[o + 1], g2 = c[o + 2];
        d[m][o] = G[m][0] * g0 + G[m][1] * g1 + G[m][2] * g2;
        d[m][o + 1] = G[m][1] * g0 + G[m][3] * g1 + G[m][4] * g2;
        d[m][o + 2] = G[m][2] * g0 + G[m][4] * g1 + G[m][5] * g2;
        if (MASS) d[m][0] = mdet[m] * c[0];
        // lane q4 owns group point 8T + q4 (all its components), so each point counts once
        if (EN) en = fma(g0, d[m][o], fma(g1, d[m][o + 1], fma(g2, d[m][o + 2], en)));
      }
#pragma unroll
      for (int c = 0; c < S::NC; ++c)
#pragma unroll
        for (int nj = 0; nj < S::NJ; ++nj) {
          const double b = B2(S::NB2T + c * S::NJ + nj);
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma(yacc[m][nj], d[m][c], b);
        }
    };
    // remainder pair group: lane owns components 2(q4&1) + {0,1} of point 8T + (q4>>1)
    auto gemm1p = [&](double (&v)[MT][2]) {
#pragma unroll
      for (int m = 0; m < MT; ++m) v[m][0] = v[m][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk) {
        const double b = B1(S::NB1T + kk);
#pragma unroll
        for (int m = 0; m < MT; ++m) dmma(v[m], av[m][kk], b);
      }
    };
    auto dgemm2p = [&](const double (&v)[MT][2]) {
      static_assert(!(S::PAIR && MASS), "no rule with a mass term in the point loop leaves a 1-2 point remainder");
      double d[MT][2];
      const bool odd = (q4 & 1) != 0;
#pragma unroll
      for (int m = 0; m < MT; ++m) {
        const double x0 = __shfl_xor_sync(0xffffffffu, v[m][0], 1);
        const double x1 = __shfl_xor_sync(0xffffffffu, v[m][1], 1);
        {
          // components (g0, g1 | g2, pad): even lanes integrate d0 and d1, odd lanes d2
          const double g0 = odd ? x0 : v[m][0], g1 = odd ? x1 : v[m][1], g2 = odd ? v[m][0] : x0;
          const double a0 = odd ? G[m][2] : G[m][0], a1 = odd ? G[m][4] : G[m][1], a2 = odd ? G[m][5] : G[m][2];
          d[m][0] = a0 * g0 + a1 * g1 + a2 * g2;
          d[m][1] = odd ? 0.0 : G[m][1] * g0 + G[m][3] * g1 + G[m][4] * g2;
          if (EN) en = odd ? fma(g2, d[m][0], en) : fma(g0, d[m][0], fma(g1, d[m][1], en));
        }
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int nj = 0; nj < S::NJ; ++nj) {
          const double b = B2(S::NB2T + i * S::NJ + nj);
#pragma unroll
          for (int m = 0; m < MT; ++m) dmma(yacc[m][nj], d[m][i], b);
        }
    };
    double vg[MT][2][2];
#pragma unroll
    for (int t = 0; t < S::T; ++t) {
      double v[MT][S::NC][2];
      gemm1(t, v);
      daction_gemm2(t, v);
    }
    if (S::GRP) {
      gemm1g(vg);
      dgemm2g(vg);
    }
    if (S::PAIR) {
      double vp[MT][2];
      gemm1p(vp);
      dgemm2p(vp);
    }

    // ---- scatter / store: accumulator (nj, i) of a lane is DoF 4(2nj+i) + q4, the DoF of
    // its gather k-step kk = 2nj+i
#pragma unroll
    for (int m = 0; m < MT; ++m) {
      if (!valid[m]) continue;
#pragma unroll
      for (int nj = 0; nj < S::NJ; ++nj)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          constexpr int KKc = S::KK;
          const int kk = 2 * nj + i;
          if (kk >= KKc) continue;
          const int j = 4 * kk + q4;
          if (j < N) {
            if (DG) {
              TMF_CHECK(a, (cell[m] * N + j) * a.nc + comp < a.dbg_n_dofs, TMF_DBG_DOF);
              a.y[(cell[m] * N + j) * a.nc + comp] = yacc[m][nj][i];
            } else {
              const int64_t g = AS > 0 ? ridx[(m * S::KK + kk) * 32 + lane] : cidx[m][kk < KKc ? kk : 0];
              TMF_CHECK(a, g < 0 || g * a.nc + comp < a.dbg_n_dofs, TMF_DBG_DOF);
              if (g >= 0) {
                if (PEER)
                  peer_red_add(peer_dst(a.peer, a.y, g, a.nc, comp), yacc[m][nj][i]);
                else
                  atomicAdd(a.y + g * a.nc + comp, yacc[m][nj][i]);
              }
            }
          }
        }
    }
  }
  if (EN && a.energy != nullptr) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) en += __shfl_xor_sync(0xffffffffu, en, o);
    if (lane == 0) atomicAdd(a.energy, en);
  }
  // peer REDs must be visible system-wide before the caller's cross-rank barrier
  if (PEER && a.peer.y != nullptr) __threadfence_system();
}

// y[c] = u[c] on strongly constrained DoFs (identity rows, operator.py:327-328)
// energy != nullptr: also += sum over the list of u[g] y[g] = u[g]^2 (the identity rows'
// share of u.Au, which the cell kernels' element energies leave out)
static __global__ void dirichlet_fixup_kernel(const double* __restrict__ u, double* __restrict__ y,
                                       const int* __restrict__ list, int64_t n, double* energy) {
  double e = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = list[i];
    const double v = u[g];
    y[g] = v;
    e += v * v;
  }
  if (energy) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
    if ((threadIdx.x & 31) == 0 && e != 0.0) atomicAdd(energy, e);
  }
}

}  // namespace tmf
