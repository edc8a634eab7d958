// SIPG face-term kernel on FP64 tensor cores (sm_100a).
//
// Restates the reference face loop (operator.py:387-437) with the
// quadrature-point arithmetic of face_qpoint / boundary_qpoint
// (numpy_backend.py:91-119):
//     jump = V- - V+,  avg = (m-.G- + m+.G+)/2,  w = |t_s x t_t| w_q scale
//     qv = w (tau jump - avg),   qg± = -w jump m± / 2
//     R- = Fv-^T qv + Fg-^T qg-,   R+ = -Fv+^T qv + Fg+^T qg+
//   boundary (Dirichlet): qv = w (tau V - m.G),  qg = -w V m
//
// Work decomposition.  One warp handles a batch of 8 faces (M = faces) that
// share the signature (lf-, lf+, code), so the tables (lf-, 0) and
// (lf+, code) are common B operands -- the reference's grouping of faces by
// signature (operator.py:152-170).  The host sorts faces by signature, pads
// each group to a multiple of 8 and cuts it into chunks of <= CHUNK batches;
// one CTA per chunk stages the two tables' DMMA fragments in shared memory
// once and its warps stream over the chunk's batches.
//
// Face frame.  Each side's reference gradient is rotated into the frame of
// its local face lf: D = A_lf^T grad, A_lf = [c1-c0, c2-c0, v_lf-c0] (two
// tangent directions of the reference face and one transversal), and
// m.grad = (A_lf^-1 m).D, so the geometry record stores m~ = A^-1 m.  With
// a nodal (Lagrange) basis the value and the two tangential derivatives on a
// face only involve the NF = (p+1)(p+2)/2 DoFs on that face; DoFs are gathered
// in the order perm_lf = (face DoFs, other DoFs) so those three components
// only need ceil(NF/4) GEMM1 k-steps and ceil(NF/8) GEMM2 n-tiles (the
// transversal component keeps all of them): 29 % (P2), 23 % (P3) and 37 % (P4)
// fewer DMMAs than the plain 4-component layout, same quadrature.
//
// Point layout (4 components per point: value, D0, D1 | D2): points are taken
// in groups of 4; GEMM1 n-tile (g, h) holds columns 2*q + i = (point 4g + q,
// component 2h + i), so lane (q = lane&3) owns all four components of point
// 4g + q after the two tiles of group g, and those four values are directly
// the A fragments of the four GEMM2 k-steps (g, c), k = lane&3 <-> point
// 4g + k.  Points pad to a multiple of 4 (n_qf 20 -> 20, 10 -> 12), not 8.
// Geometry (unit normal outward from the minus cell, |t_s x t_t|,
// m = J^-1 n on each side, geometry.py:202-236) is computed once per plan by
// face_geometry_kernel.  Contributions are added to y with fp64 RED.
#pragma once
#include "common.cuh"

namespace tmf {

struct FaceArgs {
  const double* __restrict__ u;
  double* __restrict__ y;
  const double* __restrict__ frags;   // per (lf, code) combo: B1 then B2 fragments
  const int4* __restrict__ chunks;    // (combo-, combo+ or -1, first batch, n batches)
  const int* __restrict__ cm;         // (n_batches*8) minus cell, -1 = padding
  const int* __restrict__ cp;         // (n_batches*8) plus cell (interior)
  const double* __restrict__ geo;     // (n_batches*8, 8): m~-[3], m~+[3], s, tau (see below)
  const int* __restrict__ perm;       // (4, n_dpc): gather order per local face (face DoFs first)
  int64_t n_chunks;
  int n_dpc;
  int nc;
  PeerArgs peer;                      // multi-GPU: ghost cells' u read from their owner (n_own = cells)
  int hier = 0;                       // host-side: frags hold the split-mode layout (HierShape) -> HIER kernels
  int run = 0;                        // BLOCKED kernels: chunk-run length of the CTA walk (ChunkWalk), 0 = one run per CTA
  // the (4, n_dpc) gather orders again, as a kernel parameter: face_apply_kernel reads them
  // from the constant bank (LDC), off the L1 data pipe its gathers and REDs saturate
  int permc[4 * 35] = {};
  TMF_DBG_FIELDS
};

// Which chunks a CTA takes, in which order (work item w = component * n_chunks + chunk):
//   round-robin (not BLOCKED): w = blockIdx + i * grid;
//   BLOCKED, run 0: one contiguous run per CTA -- consecutive chunks of a (window,
//     signature) group share their tables, so restaging and its barriers are skipped;
//   BLOCKED, run R: runs of R consecutive chunks dealt round-robin, so all CTAs advance
//     through the window-sorted face list together and the four faces of a cell find its
//     u / y rows in L2 (DG P3 64^3 reordered: faces -10 %), while a run still shares tables.
struct ChunkWalk {
  int64_t nwork, nit, per;
  int64_t grid, block;   // CTAs of the launch, this CTA
  int run;
  bool blocked;
  __host__ __device__ ChunkWalk(int64_t nwork_, bool blocked_, int run_, int64_t grid_, int64_t block_)
      : nwork(nwork_), grid(grid_), block(block_), run(run_), blocked(blocked_) {
    per = (nwork + grid - 1) / grid;
    if (!blocked || run <= 0) nit = per;
    else nit = ((nwork + run - 1) / run + grid - 1) / grid * run;
  }
  // work item of this CTA's iteration i (>= nwork: none)
  __host__ __device__ int64_t at(int64_t i) const {
    if (!blocked) return block + i * grid;
    if (run <= 0) return block * per + i;
    return ((i / run) * grid + block) * run + i % run;
  }
};

// Per-face geometry, computed once at plan creation by face_geometry_kernel and
// streamed (64 B per face, coalesced) by the apply -- the reference stores the
// same factors in GeometryData (face_jxw, face_m_minus/plus, geometry.py:44-53):
//   m± = kappa± J±^-1 n,  s = |t_s x t_t| * scale,  tau_eff = tau * max(kappa-, kappa+)
struct FaceGeoArgs {
  const int* __restrict__ cells;
  const double* __restrict__ verts;
  const double* __restrict__ kappa;
  const int4* __restrict__ chunks;
  const int* __restrict__ cm;
  const int* __restrict__ cp;
  const double* __restrict__ tau;     // raw penalty per slot
  double* __restrict__ geo;
  int64_t n_chunks;
  double scale;
};

template <int N, int QF>
struct FaceShape {
  static constexpr int NF = N == 4 ? 3 : N == 10 ? 6 : N == 20 ? 10 : 15;  // DoFs on a face
  static constexpr int KK = (N + 3) / 4;
  static constexpr int KKF = (NF + 3) / 4;
  static constexpr int G = (QF + 3) / 4;       // point groups of 4
  static constexpr int NJ = (N + 7) / 8;
  static constexpr int NJF = (NF + 7) / 8;
  static constexpr int B1G = KKF + KK;         // GEMM1 fragments per group: h=0 (V,D0) | h=1 (D1,D2)
  static constexpr int B2G = 3 * NJF + NJ;     // GEMM2 fragments per group: V, D0, D1 face-only | D2
  static constexpr int NB1 = G * B1G;
  static constexpr int NB2 = G * B2G;
  static constexpr int NFRAG = NB1 + NB2;      // per (lf, code) combo
  static constexpr int CHUNK = 32;             // default batches per CTA chunk
  __host__ __device__ static constexpr int b1(int g, int h, int kk) { return g * B1G + (h ? KKF + kk : kk); }
  __host__ __device__ static constexpr int b2(int g, int c, int nj) {
    return NB1 + g * B2G + (c < 3 ? c * NJF + nj : 3 * NJF + nj);
  }
};

// Split-mode layout of the modal interior-face kernel (HIER).  With a degree-ordered
// orthonormal basis psi_0.. of P_p on the face (the first MD = dim P_{p-1} modes span
// P_{p-1}), the derivative components of every trace are polynomials of degree p-1, so they
// only have MD modal coefficients; the NVO = p+1 modes of exact degree p carry a value only,
// and their share of the face term is linear: qv_m = -s tau (V+_m - V-_m).
//
// Each lane (q = lane&3) owns NS "quad slots" of four registers per side.  Quad slot
// idx = 4 s + q is
//   * full   (idx < MD):  (V, D0, D1, D2) of mode idx        -> (qv, qg0, qg1, qg2)
//   * triple (idx >= MD): V of modes MD + 3 (idx-MD) + {0,1,2} -> their three qv, and 0
// (triples only occur in the last slot row).  GEMM1 n-tiles pair the lane's registers:
// face-only entries e = 3 s + r (r < 3: V, D0, D1 need the NF face DoFs = KKF k-steps),
// then the D2 entries (all N DoFs, KK k-steps; an odd NS leaves a spare column that takes
// the last face-only entry).  GEMM2 k-steps: one per (s, r), NJF n-tiles for r < 3, NJ for
// the transversal derivative.  DMMAs per 8-face batch (both sides): 20 / 64 / 134 at
// P2 / P3 / P4 against 40 / 102 / 192 for the flat 4-components-per-mode layout.
template <int N>
struct HierShape {
  static constexpr int P = N == 4 ? 1 : N == 10 ? 2 : N == 20 ? 3 : 4;
  static constexpr int NF = (P + 1) * (P + 2) / 2;   // value modes = DoFs on a face
  static constexpr int MD = P * (P + 1) / 2;         // derivative modes
  static constexpr int NVO = NF - MD;                // value-only modes
  static constexpr int NTRI = (NVO + 2) / 3;
  static constexpr int NS = (MD + NTRI + 3) / 4;     // quad slots per lane
  static_assert(4 * (NS - 1) <= MD, "triple slots must sit in the last slot row");
  static constexpr int KK = (N + 3) / 4;
  static constexpr int KKF = (NF + 3) / 4;
  static constexpr int NJ = (N + 7) / 8;
  static constexpr int NJF = (NF + 7) / 8;
  static constexpr int NTF = (3 * NS) / 2;           // face-only GEMM1 tiles
  static constexpr int NTD = (NS + 1) / 2;           // GEMM1 tiles with the D2 entries
  static constexpr int NB1 = NTF * KKF + NTD * KK;
  static constexpr int NB2 = 3 * NS * NJF + NS * NJ;
  static constexpr int NFRAG = NB1 + NB2;            // per (lf, code) combo
  static constexpr int CHUNK = 32;
  __host__ __device__ static constexpr int b1f(int t, int kk) { return t * KKF + kk; }
  __host__ __device__ static constexpr int b1d(int d, int kk) { return NTF * KKF + d * KK + kk; }
  __host__ __device__ static constexpr int b2(int s, int r, int nj) {
    return NB1 + (r < 3 ? (s * 3 + r) * NJF + nj : 3 * NS * NJF + s * NJ + nj);
  }
  // register (s, r) of column i of face-only tile t / D2 tile d; s < 0: empty column
  __host__ __device__ static constexpr int tf_s(int t, int i) { return (2 * t + i) / 3; }
  __host__ __device__ static constexpr int tf_r(int t, int i) { return (2 * t + i) % 3; }
  __host__ __device__ static constexpr int td_s(int d, int i) {
    return i == 0 ? 2 * d : (2 * d + 1 < NS ? 2 * d + 1 : ((3 * NS) % 2 ? (3 * NS - 1) / 3 : -1));
  }
  __host__ __device__ static constexpr int td_r(int d, int i) {
    return (i == 0 || 2 * d + 1 < NS) ? 3 : (3 * NS - 1) % 3;
  }
  // (component, mode) held by register (s, r) of lane slot q: mode < 0 = empty
  __host__ __device__ static constexpr int item_mode(int q, int s, int r) {
    const int idx = 4 * s + q;
    if (idx < MD) return idx;
    const int m = MD + 3 * (idx - MD) + r;
    return (r < 3 && m < NF) ? m : -1;
  }
  __host__ __device__ static constexpr int item_comp(int q, int s, int r) { return 4 * s + q < MD ? r : 0; }
};

// Either layout behind the names the kernels use
template <int N, int QF, bool HIER>
struct FaceShapeSel : FaceShape<N, QF> {};
template <int N, int QF>
struct FaceShapeSel<N, QF, true> : HierShape<N> {};

// Interior-face arithmetic of one 8-face batch in the split-mode layout: GEMM1 of both
// sides, the modal face_qpoint (numpy_backend.py:91-105 on modes), GEMM2 of both sides.
// Bm(f) / Bp(f): fragment f of the minus / plus table for this lane (shared memory, or
// registers loaded once per chunk: face_apply_kernel RT)
template <int N, class TM, class TP>
__device__ __forceinline__ void face_hier_core_t(const double (&am)[HierShape<N>::KK], const double (&ap)[HierShape<N>::KK],
                                                 const double (&hm)[3], const double (&hp)[3], double stau,
                                                 TM Bm, TP Bp, int lane, double (&ym)[HierShape<N>::NJ][2],
                                                 double (&yp)[HierShape<N>::NJ][2]) {
  using S = HierShape<N>;
  const int q4 = lane & 3;
  double vm[S::NS][4], vp[S::NS][4];
#pragma unroll
  for (int s = 0; s < S::NS; ++s)
#pragma unroll
    for (int r = 0; r < 4; ++r) vm[s][r] = vp[s][r] = 0.0;
#pragma unroll
  for (int t = 0; t < S::NTF; ++t) {
    double cm[2] = {0.0, 0.0}, cp[2] = {0.0, 0.0};
#pragma unroll
    for (int kk = 0; kk < S::KKF; ++kk) {
      dmma(cm, am[kk], Bm(S::b1f(t, kk)));
      dmma(cp, ap[kk], Bp(S::b1f(t, kk)));
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      vm[S::tf_s(t, i)][S::tf_r(t, i)] = cm[i];
      vp[S::tf_s(t, i)][S::tf_r(t, i)] = cp[i];
    }
  }
#pragma unroll
  for (int d = 0; d < S::NTD; ++d) {
    double cm[2] = {0.0, 0.0}, cp[2] = {0.0, 0.0};
#pragma unroll
    for (int kk = 0; kk < S::KK; ++kk) {
      dmma(cm, am[kk], Bm(S::b1d(d, kk)));
      dmma(cp, ap[kk], Bp(S::b1d(d, kk)));
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
      if (S::td_s(d, i) >= 0) {
        vm[S::td_s(d, i)][S::td_r(d, i)] = cm[i];
        vp[S::td_s(d, i)][S::td_r(d, i)] = cp[i];
      }
  }
#pragma unroll
  for (int s = 0; s < S::NS; ++s) {
    const bool may_tri = 4 * s + 3 >= S::MD;            // compile time per unrolled s
    const bool tri = may_tri && (4 * s + q4 >= S::MD);
    const double d0 = vp[s][0] - vm[s][0];              // -[[u]] of the slot's (first) mode
    double hmf[3], hpf[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      hmf[k] = tri ? 0.0 : hm[k];
      hpf[k] = tri ? 0.0 : hp[k];
    }
    double qv = -stau * d0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      qv = fma(-hmf[k], vm[s][1 + k], qv);
      qv = fma(-hpf[k], vp[s][1 + k], qv);
    }
    double om[4], op[4];
    om[0] = qv;
    op[0] = -qv;
    if (may_tri) {
      const double t1 = stau * (vp[s][1] - vm[s][1]), t2 = stau * (vp[s][2] - vm[s][2]);
      om[1] = tri ? -t1 : d0 * hm[0];
      om[2] = tri ? -t2 : d0 * hm[1];
      op[1] = tri ? t1 : d0 * hp[0];
      op[2] = tri ? t2 : d0 * hp[1];
    } else {
      om[1] = d0 * hm[0];
      om[2] = d0 * hm[1];
      op[1] = d0 * hp[0];
      op[2] = d0 * hp[1];
    }
    om[3] = d0 * hmf[2];
    op[3] = d0 * hpf[2];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int nj = 0; nj < (r < 3 ? S::NJF : S::NJ); ++nj) {
        dmma(ym[nj], om[r], Bm(S::b2(s, r, nj)));
        dmma(yp[nj], op[r], Bp(S::b2(s, r, nj)));
      }
  }
}

template <int N>
__device__ __forceinline__ void face_hier_core(const double (&am)[HierShape<N>::KK], const double (&ap)[HierShape<N>::KK],
                                               const double (&hm)[3], const double (&hp)[3], double stau,
                                               const double* __restrict__ Fm, const double* __restrict__ Fp,
                                               int lane, double (&ym)[HierShape<N>::NJ][2],
                                               double (&yp)[HierShape<N>::NJ][2]) {
  face_hier_core_t<N>(
      am, ap, hm, hp, stau, [&](int f) { return Fm[f * 32 + lane]; }, [&](int f) { return Fp[f * 32 + lane]; },
      lane, ym, yp);
}

// A_lf^-1 for the face frame (reference vertices (0,0,0),(1,0,0),(0,1,0),(0,0,1)).
__host__ __device__ inline void face_frame_inverse(int lf, double (&Ai)[3][3]) {
  const double R[4][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  const int fv[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
  double A[3][3];
  for (int k = 0; k < 3; ++k) {
    A[k][0] = R[fv[lf][1]][k] - R[fv[lf][0]][k];
    A[k][1] = R[fv[lf][2]][k] - R[fv[lf][0]][k];
    A[k][2] = R[lf][k] - R[fv[lf][0]][k];
  }
  const double c00 = A[1][1] * A[2][2] - A[1][2] * A[2][1], c01 = A[1][2] * A[2][0] - A[1][0] * A[2][2],
               c02 = A[1][0] * A[2][1] - A[1][1] * A[2][0];
  const double det = A[0][0] * c00 + A[0][1] * c01 + A[0][2] * c02;
  Ai[0][0] = c00 / det;
  Ai[1][0] = c01 / det;
  Ai[2][0] = c02 / det;
  Ai[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) / det;
  Ai[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / det;
  Ai[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) / det;
  Ai[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / det;
  Ai[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) / det;
  Ai[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / det;
}

__device__ __forceinline__ void to_face_frame(int lf, double (&m)[3]) {
  double Ai[3][3];
  face_frame_inverse(lf, Ai);
  const double x = m[0], y = m[1], z = m[2];
#pragma unroll
  for (int i = 0; i < 3; ++i) m[i] = Ai[i][0] * x + Ai[i][1] * y + Ai[i][2] * z;
}

__device__ __forceinline__ void cell_affine(const int* __restrict__ cells, const double* __restrict__ verts,
                                            int c, Affine& g, Vec3& opp_base, int lf, Vec3& face_v0) {
  int vid[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) vid[i] = __ldg(cells + 4 * (int64_t)c + i);
  const Vec3 x0 = load_vertex(verts, vid[0]), x1 = load_vertex(verts, vid[1]),
             x2 = load_vertex(verts, vid[2]), x3 = load_vertex(verts, vid[3]);
  affine_from_vertices(x0, x1, x2, x3, g);
  // local face lf is opposite local vertex lf; its first corner is v1 (lf 0) or v0
  opp_base = lf == 0 ? x0 : (lf == 1 ? x1 : (lf == 2 ? x2 : x3));
  face_v0 = lf == 0 ? x1 : x0;
}

__device__ __forceinline__ void apply_inv(const Affine& g, const double (&n)[3], double (&m)[3]) {
  const double inv = 1.0 / g.det;
#pragma unroll
  for (int i = 0; i < 3; ++i) m[i] = inv * (g.adj[i][0] * n[0] + g.adj[i][1] * n[1] + g.adj[i][2] * n[2]);
}

// One thread per face slot: unit normal outward from the minus cell
// (geometry.py:207-225), surface JxW factor and m = J^-1 n on each side, the
// latter expressed in the side's face frame (m~ = A_lf^-1 m).
template <bool BOUNDARY>
__global__ void face_geometry_kernel(FaceGeoArgs a) {
  for (int64_t ci = blockIdx.x; ci < a.n_chunks; ci += gridDim.x) {
    const int4 ch = __ldg(a.chunks + ci);
    const int lfm = ch.x / 6;
    for (int k = threadIdx.x; k < ch.w * 8; k += blockDim.x) {
      const int64_t slot = (int64_t)ch.z * 8 + k;
      double* out = a.geo + slot * 8;
      const int c_m = a.cm[slot];
      if (c_m < 0) {
#pragma unroll
        for (int i = 0; i < 8; ++i) out[i] = 0.0;
        continue;
      }
      Affine Jm;
      Vec3 opp, fv0;
      cell_affine(a.cells, a.verts, c_m, Jm, opp, lfm, fv0);
      double ds[3], dt[3];
      face_tangents_ref(lfm, ds, dt);
      double ts[3], tt[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        ts[i] = Jm.J[i][0] * ds[0] + Jm.J[i][1] * ds[1] + Jm.J[i][2] * ds[2];
        tt[i] = Jm.J[i][0] * dt[0] + Jm.J[i][1] * dt[1] + Jm.J[i][2] * dt[2];
      }
      double n[3] = {ts[1] * tt[2] - ts[2] * tt[1], ts[2] * tt[0] - ts[0] * tt[2],
                     ts[0] * tt[1] - ts[1] * tt[0]};
      const double area2 = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
      const double side = n[0] * (fv0.x - opp.x) + n[1] * (fv0.y - opp.y) + n[2] * (fv0.z - opp.z);
      const double inv = (side < 0 ? -1.0 : 1.0) / area2;
#pragma unroll
      for (int i = 0; i < 3; ++i) n[i] *= inv;
      double mm[3], mp[3] = {0.0, 0.0, 0.0};
      apply_inv(Jm, n, mm);
      to_face_frame(lfm, mm);
      double tau = a.tau[slot];
      const double km = a.kappa ? a.kappa[c_m] : 1.0;
      if (!BOUNDARY) {
        const int c_p = a.cp[slot];
        Affine Jp;
        Vec3 o2, f2;
        cell_affine(a.cells, a.verts, c_p, Jp, o2, 0, f2);
        apply_inv(Jp, n, mp);
        to_face_frame(ch.y / 6, mp);
        const double kp = a.kappa ? a.kappa[c_p] : 1.0;
#pragma unroll
        for (int i = 0; i < 3; ++i) mp[i] *= kp;
        tau *= fmax(km, kp);
      } else {
        tau *= km;
      }
      // pre-scaled record: interior h+- = s m~+- / 2, boundary h = s m~;  out[6] = s tau
      const double sc = area2 * a.scale;
      const double hs = BOUNDARY ? sc : 0.5 * sc;
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        out[i] = hs * mm[i] * km;
        out[3 + i] = hs * mp[i];
      }
      out[6] = sc * tau;
      out[7] = 0.0;
    }
  }
}

// PF: prefetch depth (0 none, 1 face record, 2 record + geometry + gathered u); MINB: CTAs/SM hint
// BLOCKED: each CTA takes a contiguous run of chunks (consecutive chunks of one
// (window, signature) group share their tables, so restaging and both barriers are
// skipped); otherwise chunks are dealt round-robin.
// RESIDENT: all 24 (lf, code) tables are staged once per CTA, so a chunk never restages
// and the warps never wait for each other (small tables: P1 / P2 modal faces)
// HIER: the split-mode modal layout (HierShape, interior faces only; QF is not used)
// SG: the batch's 8 face records (64 B each) are staged through a per-warp shared-memory
// slot with ONE coalesced 16-byte cp.async per lane and read back as broadcast LDS.64s,
// instead of four LDG.128s per lane that every lane of a face repeats (32 -> 15 L1
// wavefronts per batch, 8 fewer registers in the prefetch state)
template <int N, int QF, bool BOUNDARY, int PF = 2, int MINB = 2, int BLOCK = 256, bool BLOCKED = false,
          bool PEER = false, bool RESIDENT = false, bool HIER = false, bool SG = false, bool RT = false>
__global__ void __launch_bounds__(BLOCK, MINB) face_apply_kernel(FaceArgs a) {
  static_assert(!HIER || !BOUNDARY, "the split-mode layout is for interior faces");
  // RT: both tables' fragments of a chunk are loaded into registers once and serve all of the
  // warp's batches in the chunk (small tables: split-mode P2, 2 x 10 fragments)
  static_assert(!RT || HIER, "register tables are for the split-mode layout");
  using S = FaceShapeSel<N, QF, HIER>;
  extern __shared__ __align__(16) double smem[];
  // staged geometry: two 64-double slots per warp behind the tables
  double* sgeo = smem + ((RT && !RESIDENT) ? 0 : (RESIDENT ? 24 : (BOUNDARY ? 1 : 2))) * S::NFRAG * 32 +
                 (threadIdx.x >> 5) * 128;
  int gslot = 0;
  if (RESIDENT) {
    const double2* src = reinterpret_cast<const double2*>(a.frags);
    double2* dst = reinterpret_cast<double2*>(smem);
    for (int i = threadIdx.x; i < 24 * S::NFRAG * 16; i += blockDim.x) dst[i] = __ldg(src + i);
    __syncthreads();
  }
  // launched as the programmatic dependent of the kernel before it (launch_apply): the CTA and
  // its resident tables are set up while that kernel drains; its stores / REDs into y are
  // complete and visible from here on (no-op without the launch attribute)
  pdl_wait_prior_grid();
  const int lane = threadIdx.x & 31;
  const int fs = lane >> 2;
  const int q4 = lane & 3;
  const int warp = threadIdx.x >> 5;
  const int nwb = blockDim.x >> 5;

  const int64_t nwork = a.n_chunks * a.nc;
  const ChunkWalk walk(nwork, BLOCKED, a.run, gridDim.x, blockIdx.x);
  auto chunk_at = [&](int64_t w) {
    const int comp = a.nc == 1 ? 0 : (int)(w / a.n_chunks);
    return __ldg(a.chunks + (w - (int64_t)comp * a.n_chunks));
  };
  int cur_x = -1, cur_y = -2;
  for (int64_t it = 0; it < walk.nit; ++it) {
    const int64_t w = walk.at(it);
    if (w >= nwork) continue;
    const int comp = a.nc == 1 ? 0 : (int)(w / a.n_chunks);
    const int4 ch = chunk_at(w);
    // RT without RESIDENT: the register tables are loaded straight from global memory (L1 / L2
    // hold the 24 small tables), nothing is staged and the CTA needs no table shared memory
    constexpr bool GT = RT && !RESIDENT;
    if (!RESIDENT && !GT && (ch.x != cur_x || ch.y != cur_y)) {
      cur_x = ch.x;
      cur_y = ch.y;
      __syncthreads();  // previous chunk's warps are done with the staged tables
      const double2* s0 = reinterpret_cast<const double2*>(a.frags + (int64_t)ch.x * S::NFRAG * 32);
      double2* d = reinterpret_cast<double2*>(smem);
      for (int i = threadIdx.x; i < S::NFRAG * 16; i += blockDim.x) d[i] = __ldg(s0 + i);
      if (!BOUNDARY) {
        const double2* s1 = reinterpret_cast<const double2*>(a.frags + (int64_t)ch.y * S::NFRAG * 32);
        for (int i = threadIdx.x; i < S::NFRAG * 16; i += blockDim.x) d[S::NFRAG * 16 + i] = __ldg(s1 + i);
      }
      __syncthreads();
    }
    const double* Fm = GT ? a.frags + (int64_t)ch.x * S::NFRAG * 32
                          : RESIDENT ? smem + (int64_t)ch.x * S::NFRAG * 32 : smem;
    const double* Fp = GT ? a.frags + (int64_t)(BOUNDARY ? 0 : ch.y) * S::NFRAG * 32
                          : RESIDENT ? smem + (int64_t)(BOUNDARY ? 0 : ch.y) * S::NFRAG * 32 : Fm + S::NFRAG * 32;
    const int pm0 = (ch.x / 6) * N;                  // gather order, minus side
    const int pp0 = (BOUNDARY ? 0 : ch.y / 6) * N;   // plus side

    // Software pipeline over the warp's batches.  PF 2: the next batch's face
    // record, geometry and gathered u are loaded while the current batch
    // computes; PF 1: only the record (cell ids) is prefetched, so the u and
    // geometry loads of a batch are issued together (one memory round trip);
    // PF 0: no prefetch.
    double nam[S::KK], nap[S::KK], ng[8];
    int n_cm = -1, n_cp = -1;
    auto fetch_rec = [&](int bi) {
      n_cm = -1;
      n_cp = -1;
      if (bi < ch.w) {
        const int64_t slot = ((int64_t)ch.z + bi) * 8 + fs;
        n_cm = __ldg(a.cm + slot);
        if (!BOUNDARY) n_cp = __ldg(a.cp + slot);
      }
    };
    auto fetch_data = [&](int bi) {
      if (SG) {
        if (bi < ch.w)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(
                           (uint32_t)__cvta_generic_to_shared(sgeo + (gslot ^ 1) * 64 + 2 * lane)),
                       "l"(a.geo + ((int64_t)ch.z + bi) * 64 + 2 * lane) : "memory");
        asm volatile("cp.async.commit_group;\n" ::: "memory");
        gslot ^= 1;
      } else if (bi < ch.w) {
        const int64_t slot = ((int64_t)ch.z + bi) * 8 + fs;
        const double2* gp = reinterpret_cast<const double2*>(a.geo + slot * 8);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double2 v = __ldg(gp + i);
          ng[2 * i] = v.x;
          ng[2 * i + 1] = v.y;
        }
      }
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk) {
        const int j = 4 * kk + q4;
        nam[kk] = 0.0;
        nap[kk] = 0.0;
        if (n_cm >= 0 && j < N) {
          TMF_CHECK(a, n_cm < a.dbg_n_cells && a.permc[pm0 + j] < N, TMF_DBG_CELL);
          TMF_CHECK(a, BOUNDARY || (n_cp >= 0 && (PEER || n_cp < a.dbg_n_cells) && a.permc[pp0 + j] < N),
                    TMF_DBG_CELL);
          nam[kk] = __ldg(a.u + ((int64_t)n_cm * N + a.permc[pm0 + j]) * a.nc + comp);
          if (!BOUNDARY) {
            // DG ghost cell (partitioned apply): its u is read from the owner rank
            if (PEER && n_cp >= a.peer.n_own) {
              const int64_t gc = n_cp - a.peer.n_own;
              nap[kk] = __ldg(a.peer.u[__ldg(a.peer.rank + gc)] +
                              ((int64_t)__ldg(a.peer.idx + gc) * N + a.permc[pp0 + j]) * a.nc + comp);
            } else {
              nap[kk] = __ldg(a.u + ((int64_t)n_cp * N + a.permc[pp0 + j]) * a.nc + comp);
            }
          }
        }
      }
    };
    double bm[RT ? S::NFRAG : 1], bp[RT ? S::NFRAG : 1];
    if (RT && warp < ch.w) {
#pragma unroll
      for (int f = 0; f < S::NFRAG; ++f) {
        bm[f] = GT ? __ldg(Fm + f * 32 + lane) : Fm[f * 32 + lane];
        bp[f] = GT ? __ldg(Fp + f * 32 + lane) : Fp[f * 32 + lane];
      }
    }
    if (PF >= 1) fetch_rec(warp);
    if (PF == 2) fetch_data(warp);

    for (int bi = warp; bi < ch.w; bi += nwb) {
      if (PF == 0) fetch_rec(bi);
      if (PF <= 1) fetch_data(bi);
      const int c_m = n_cm, c_p = n_cp;
      double am[S::KK], ap[S::KK];
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk) {
        am[kk] = nam[kk];
        ap[kk] = nap[kk];
      }
      if (SG) {
        // the slot filled by this batch's fetch_data (PF 2: one iteration ago)
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncwarp();
        const double* g8 = sgeo + gslot * 64 + fs * 8;
#pragma unroll
        for (int i = 0; i < 7; ++i) ng[i] = g8[i];
        // (this slot is refilled two fetches from now, after the next batch's __syncwarp)
      }
      const double hm[3] = {ng[0], ng[1], ng[2]};   // s m~- / 2   (boundary: s m~)
      const double hp[3] = {ng[3], ng[4], ng[5]};   // s m~+ / 2
      const double stau = ng[6];                     // s tau
      if (PF >= 1) fetch_rec(bi + nwb);
      if (PF == 2) fetch_data(bi + nwb);

      double ym[S::NJ][2], yp[S::NJ][2];
#pragma unroll
      for (int nj = 0; nj < S::NJ; ++nj) ym[nj][0] = ym[nj][1] = yp[nj][0] = yp[nj][1] = 0.0;

      if constexpr (HIER && RT) {
        face_hier_core_t<N>(
            am, ap, hm, hp, stau, [&](int f) { return bm[f]; }, [&](int f) { return bp[f]; }, lane, ym, yp);
      } else if constexpr (HIER) {
        face_hier_core<N>(am, ap, hm, hp, stau, Fm, Fp, lane, ym, yp);
      } else {
#pragma unroll
      for (int g = 0; g < S::G; ++g) {
        double vm[2][2], vp[2][2];  // [h][i] = component 2h+i of point 4g+q4
#pragma unroll
        for (int h = 0; h < 2; ++h) vm[h][0] = vm[h][1] = vp[h][0] = vp[h][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < S::KK; ++kk)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 0 && kk >= S::KKF) continue;   // value and D0 live on the face DoFs
            const int f = S::b1(g, h, kk) * 32 + lane;
            dmma(vm[h], am[kk], Fm[f]);
            if (!BOUNDARY) dmma(vp[h], ap[kk], Fp[f]);
          }
        // face_qpoint / boundary_qpoint (numpy_backend.py:91-119) with s, 1/2 and m~
        // folded into the per-face record: 14 (interior) / 7 (boundary) FP64 ops per point
        double qm[4], qp[4];
        if (BOUNDARY) {
          const double v = vm[0][0];
          qm[0] = fma(stau, v, -(hm[0] * vm[0][1] + hm[1] * vm[1][0] + hm[2] * vm[1][1]));
#pragma unroll
          for (int k = 0; k < 3; ++k) qm[1 + k] = -v * hm[k];
        } else {
          const double nj = vp[0][0] - vm[0][0];   // -[[u]]
          double qv = -stau * nj;
          qv = fma(-hm[0], vm[0][1], qv);
          qv = fma(-hm[1], vm[1][0], qv);
          qv = fma(-hm[2], vm[1][1], qv);
          qv = fma(-hp[0], vp[0][1], qv);
          qv = fma(-hp[1], vp[1][0], qv);
          qv = fma(-hp[2], vp[1][1], qv);
          qm[0] = qv;
          qp[0] = -qv;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            qm[1 + k] = nj * hm[k];
            qp[1 + k] = nj * hp[k];
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int nj = 0; nj < S::NJ; ++nj) {
            if (c < 3 && nj >= S::NJF) continue;     // V, D0, D1 integrate onto face DoFs only
            const int f = S::b2(g, c, nj) * 32 + lane;
            dmma(ym[nj], qm[c], Fm[f]);
            if (!BOUNDARY) dmma(yp[nj], qp[c], Fp[f]);
          }
      }
      }

      if (c_m >= 0) {
#pragma unroll
        for (int nj = 0; nj < S::NJ; ++nj)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int j = 4 * (2 * nj + i) + q4;   // GEMM2 columns in the gather's lane order (capi.cu col_dof)
            if (j < N) {
              atomicAdd(a.y + ((int64_t)c_m * N + a.permc[pm0 + j]) * a.nc + comp, ym[nj][i]);
              if (!BOUNDARY) atomicAdd(a.y + ((int64_t)c_p * N + a.permc[pp0 + j]) * a.nc + comp, yp[nj][i]);
            }
          }
      }
    }
  }
}





// Interior faces with an asynchronous gather ring (the face-kernel analogue of the cell
// kernel's AS pipeline).  Each warp walks its batches of the CTA's chunks as one flat
// sequence; the gathered u of both sides and the 64-byte geometry records of the batch
// AS-1 ahead -- which may lie in a later chunk: its gather order comes from the chunk's
// signature, all four orders sit in shared memory -- are cp.async'ed into a per-warp ring,
// and the cell ids of the batch after that are loaded into registers, so AS-1 batches'
// gathers are in flight while the DMMAs of the current one run.  The chunk loop (table
// restaging and its barriers) is unchanged; round-robin or blocked chunk runs.
template <int N, int QF, int AS, int MINB = 2, int BLOCK = 256, bool BLOCKED = false, bool HIER = false>
__global__ void __launch_bounds__(BLOCK, MINB) face_async_kernel(FaceArgs a) {
  using S = FaceShapeSel<N, QF, HIER>;
  constexpr int SLOT = 2 * S::KK * 32 + 64 + 16;   // am, ap, geometry (8 x 8), cell ids (8 x 2 ints)
  extern __shared__ __align__(16) double smem[];
  double* tabs = smem;                                        // two staged tables
  int* sperm = reinterpret_cast<int*>(smem + 2 * S::NFRAG * 32);   // (4, N) gather orders
  constexpr int NW = BLOCK / 32;
  double* ring = smem + 2 * S::NFRAG * 32 + (4 * N + 1) / 2 + (threadIdx.x >> 5) * AS * SLOT;
  for (int i = threadIdx.x; i < 4 * N; i += BLOCK) sperm[i] = __ldg(a.perm + i);
  pdl_wait_prior_grid();   // see face_apply_kernel
  __syncthreads();   // the prologue's gathers read sperm
  const int lane = threadIdx.x & 31;
  const int fs = lane >> 2;
  const int q4 = lane & 3;
  const int warp = threadIdx.x >> 5;

  const int64_t nwork = a.n_chunks * a.nc;
  const ChunkWalk walk(nwork, BLOCKED, a.run, gridDim.x, blockIdx.x);
  auto chunk_at = [&](int64_t w) {
    const int comp = a.nc == 1 ? 0 : (int)(w / a.n_chunks);
    return __ldg(a.chunks + (w - (int64_t)comp * a.n_chunks));
  };
  // flat per-warp item sequence (walk iteration i -> chunk w, batch bi); i >= nit = past the end
  struct Item {
    int64_t i, w;
    int bi;
    int4 ch;
  };
  auto first_from = [&](int64_t i) {
    Item it{i, 0, warp, make_int4(0, 0, 0, 0)};
    for (; it.i < walk.nit; ++it.i) {
      it.w = walk.at(it.i);
      if (it.w >= nwork) continue;
      it.ch = chunk_at(it.w);
      if (warp < it.ch.w) break;
    }
    return it;
  };
  auto advance = [&](Item it) {
    if (it.i >= walk.nit) return it;
    if (it.bi + NW < it.ch.w) {
      it.bi += NW;
      return it;
    }
    return first_from(it.i + 1);
  };
  Item iss = first_from(0);     // next item to issue
  Item rec = iss;               // item whose cell ids are in (rcm, rcp)
  int rcm = -1, rcp = -1;
  auto load_rec = [&]() {
    rcm = rcp = -1;
    if (rec.i < walk.nit) {
      const int64_t slot = ((int64_t)rec.ch.z + rec.bi) * 8 + fs;
      rcm = __ldg(a.cm + slot);
      rcp = __ldg(a.cp + slot);
    }
  };
  int islot = 0;
  auto issue = [&]() {   // gathers of item iss (cell ids rcm / rcp) into ring slot islot
    double* r = ring + islot * SLOT;
    if (iss.i < walk.nit) {
      const int comp = a.nc == 1 ? 0 : (int)(iss.w / a.n_chunks);
      const int* pm = sperm + (iss.ch.x / 6) * N;
      const int* pp = sperm + (iss.ch.y / 6) * N;
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk) {
        const int j = 4 * kk + q4;
        const bool ok = rcm >= 0 && j < N;
        TMF_CHECK(a, !ok || (rcm < a.dbg_n_cells && rcp >= 0 && rcp < a.dbg_n_cells && pm[j] < N && pp[j] < N),
                  TMF_DBG_CELL);
        const double* sm = ok ? a.u + ((int64_t)rcm * N + pm[j]) * a.nc + comp : a.u;
        const double* sp = ok ? a.u + ((int64_t)rcp * N + pp[j]) * a.nc + comp : a.u;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(r + kk * 32 + lane)), "l"(sm), "r"(ok ? 8 : 0) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(r + (S::KK + kk) * 32 + lane)), "l"(sp), "r"(ok ? 8 : 0)
                     : "memory");
      }
      const int64_t gslot = ((int64_t)iss.ch.z + iss.bi) * 8 + fs;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(r + 2 * S::KK * 32 + fs * 8 + 2 * q4)),
                   "l"(a.geo + gslot * 8 + 2 * q4) : "memory");
      if (q4 == 0) {
        int* ids = reinterpret_cast<int*>(r + 2 * S::KK * 32 + 64);
        ids[2 * fs] = rcm;
        ids[2 * fs + 1] = rcp;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    islot = islot + 1 == AS ? 0 : islot + 1;
  };
  // prologue: AS-1 items in flight, the record of the next one in registers
  load_rec();
#pragma unroll
  for (int s = 0; s < AS - 1; ++s) {
    issue();
    iss = advance(iss);
    rec = iss;
    load_rec();
  }
  int cslot = 0;
  int cur_x = -1, cur_y = -2;
  for (int64_t wi = 0; wi < walk.nit; ++wi) {
    const int64_t w = walk.at(wi);
    if (w >= nwork) continue;
    const int comp = a.nc == 1 ? 0 : (int)(w / a.n_chunks);
    const int4 ch = chunk_at(w);
    if (ch.x != cur_x || ch.y != cur_y) {
      __syncthreads();   // previous chunk's warps are done with the tables (and sperm is set)
      const double2* s0 = reinterpret_cast<const double2*>(a.frags + (int64_t)ch.x * S::NFRAG * 32);
      const double2* s1 = reinterpret_cast<const double2*>(a.frags + (int64_t)ch.y * S::NFRAG * 32);
      double2* d = reinterpret_cast<double2*>(tabs);
      for (int i = threadIdx.x; i < S::NFRAG * 16; i += BLOCK) {
        d[i] = __ldg(s0 + i);
        d[S::NFRAG * 16 + i] = __ldg(s1 + i);
      }
      __syncthreads();
      cur_x = ch.x;
      cur_y = ch.y;
    }
    const double* Fm = tabs;
    const double* Fp = tabs + S::NFRAG * 32;
    const int* perm_m = sperm + (ch.x / 6) * N;
    const int* perm_p = sperm + (ch.y / 6) * N;
    for (int bi = warp; bi < ch.w; bi += NW) {
      // keep AS-1 items in flight: issue the next one, fetch the record after it
      __syncwarp();   // every lane is done reading the slot the issue refills
      issue();
      iss = advance(iss);
      rec = iss;
      load_rec();
      asm volatile("cp.async.wait_group %0;\n" ::"n"(AS - 1) : "memory");
      __syncwarp();
      const double* r = ring + cslot * SLOT;
      cslot = cslot + 1 == AS ? 0 : cslot + 1;
      double am[S::KK], ap[S::KK];
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk) {
        am[kk] = r[kk * 32 + lane];
        ap[kk] = r[(S::KK + kk) * 32 + lane];
      }
      const double* ng = r + 2 * S::KK * 32 + fs * 8;
      const double hm[3] = {ng[0], ng[1], ng[2]};
      const double hp[3] = {ng[3], ng[4], ng[5]};
      const double stau = ng[6];
      const int* ids = reinterpret_cast<const int*>(r + 2 * S::KK * 32 + 64);
      const int c_m = ids[2 * fs], c_p = ids[2 * fs + 1];

      double ym[S::NJ][2], yp[S::NJ][2];
#pragma unroll
      for (int nj = 0; nj < S::NJ; ++nj) ym[nj][0] = ym[nj][1] = yp[nj][0] = yp[nj][1] = 0.0;
      if constexpr (HIER) {
        face_hier_core<N>(am, ap, hm, hp, stau, Fm, Fp, lane, ym, yp);
      } else {
#pragma unroll
      for (int g = 0; g < S::G; ++g) {
        double vm[2][2], vp[2][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) vm[h][0] = vm[h][1] = vp[h][0] = vp[h][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < S::KK; ++kk)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == 0 && kk >= S::KKF) continue;
            const int f = S::b1(g, h, kk) * 32 + lane;
            dmma(vm[h], am[kk], Fm[f]);
            dmma(vp[h], ap[kk], Fp[f]);
          }
        const double nj = vp[0][0] - vm[0][0];
        double qv = -stau * nj;
        qv = fma(-hm[0], vm[0][1], qv);
        qv = fma(-hm[1], vm[1][0], qv);
        qv = fma(-hm[2], vm[1][1], qv);
        qv = fma(-hp[0], vp[0][1], qv);
        qv = fma(-hp[1], vp[1][0], qv);
        qv = fma(-hp[2], vp[1][1], qv);
        double qm[4], qp[4];
        qm[0] = qv;
        qp[0] = -qv;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          qm[1 + k] = nj * hm[k];
          qp[1 + k] = nj * hp[k];
        }
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int nj2 = 0; nj2 < S::NJ; ++nj2) {
            if (c < 3 && nj2 >= S::NJF) continue;
            const int f = S::b2(g, c, nj2) * 32 + lane;
            dmma(ym[nj2], qm[c], Fm[f]);
            dmma(yp[nj2], qp[c], Fp[f]);
          }
      }
      }
      if (c_m >= 0) {
#pragma unroll
        for (int nj = 0; nj < S::NJ; ++nj)
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int j = 4 * (2 * nj + i) + q4;   // GEMM2 columns in the gather's lane order (capi.cu col_dof)
            if (j < N) {
              atomicAdd(a.y + ((int64_t)c_m * N + perm_m[j]) * a.nc + comp, ym[nj][i]);
              atomicAdd(a.y + ((int64_t)c_p * N + perm_p[j]) * a.nc + comp, yp[nj][i]);
            }
          }
      }
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

}  // namespace tmf
