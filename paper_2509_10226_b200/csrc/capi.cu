// C-ABI of tetmf_b200: plan creation (host-side setup of device data and
// pre-swizzled DMMA table fragments), apply, diagonal, PCG.
// See include/tetmf_b200.h for the mapping onto the reference interface.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/tetmf_b200.h"
#include "cell_block_kernel.cuh"
#include "cell_f32_kernel.cuh"
#include "cell_kernel.cuh"
#include "face_kernel.cuh"
#include "launch.h"
#include "solver_kernels.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define TMF_CUDA(call)                                                                     \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(TMF_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));          \
  } while (0)

template <typename T>
int upload(T** dst, const T* src, size_t n, size_t* total) {
  *dst = nullptr;
  if (n == 0) return TMF_OK;
  TMF_CUDA(cudaMalloc(dst, n * sizeof(T)));
  TMF_CUDA(cudaMemcpy(*dst, src, n * sizeof(T), cudaMemcpyHostToDevice));
  *total += n * sizeof(T);
  return TMF_OK;
}

// Lane-major DMMA B fragments for one table family (see cell_kernel.cuh):
//   B1[t][c][kk][lane] = E_c(8t + (lane>>2), 4kk + (lane&3))
//   B2[t][c][i][nj][lane] = w_q E_c(q = 8t + 2(lane&3) + i, 8nj + (lane>>2))
// for the T full 8-point tiles; a remainder of 1..4 points is one 4-point group
// (CellShape::GRP) with components padded to 4:
//   B1g[h][kk][lane] = E_{2h + (n&1)}(8T + (n>>1), 4kk + (lane&3)),  n = lane>>2
//   B2g[c][nj][lane] = w_q E_c(q = 8T + (lane&3), 8nj + (lane>>2))
// a remainder of 1..2 points is one pair group (CellShape::PAIR), columns (point, component):
//   B1p[kk][lane] = E_{n&3}(8T + (n>>2), 4kk + (lane&3)),  n = lane>>2
//   B2p[i][nj][lane] = w_q E_{2(k&1)+i}(q = 8T + (k>>1), 8nj + (lane>>2)),  k = lane&3
// GEMM2-type fragments (B2, B2g, B2p and the mass fragments): column n = lane>>2 of n-tile nj
// is DoF col_dof(nj, n) = 4(2nj + (n&1)) + (n>>1), so a lane's accumulators are the DoFs
// 4kk + (lane&3) it gathered (cell_kernel.cuh: the scatter reuses the gather's indices).
inline int col_dof(int nj, int n) { return 4 * (2 * nj + (n & 1)) + (n >> 1); }

template <typename F>
void build_fragments(int N, int Q, int NC, F E, const double* w, std::vector<double>& out) {
  const int KK = (N + 3) / 4, NJ = (N + 7) / 8, R = Q % 8;
  const bool pair = R >= 1 && R <= 2;
  const bool grp = R >= 3 && R <= 4;
  const int T = (grp || pair) ? Q / 8 : (Q + 7) / 8;
  for (int t = 0; t < T; ++t)
    for (int c = 0; c < NC; ++c)
      for (int kk = 0; kk < KK; ++kk)
        for (int lane = 0; lane < 32; ++lane) {
          const int q = 8 * t + (lane >> 2), j = 4 * kk + (lane & 3);
          out.push_back(q < Q && j < N ? E(c, q, j) : 0.0);
        }
  if (grp)
    for (int h = 0; h < 2; ++h)
      for (int kk = 0; kk < KK; ++kk)
        for (int lane = 0; lane < 32; ++lane) {
          const int n = lane >> 2, c = 2 * h + (n & 1), q = 8 * T + (n >> 1), j = 4 * kk + (lane & 3);
          out.push_back(q < Q && j < N && c < NC ? E(c, q, j) : 0.0);
        }
  if (pair)
    for (int kk = 0; kk < KK; ++kk)
      for (int lane = 0; lane < 32; ++lane) {
        const int n = lane >> 2, c = n & 3, q = 8 * T + (n >> 2), j = 4 * kk + (lane & 3);
        out.push_back(q < Q && j < N && c < NC ? E(c, q, j) : 0.0);
      }
  for (int t = 0; t < T; ++t)
    for (int c = 0; c < NC; ++c)
      for (int i = 0; i < 2; ++i)
        for (int nj = 0; nj < NJ; ++nj)
          for (int lane = 0; lane < 32; ++lane) {
            const int q = 8 * t + 2 * (lane & 3) + i, j = col_dof(nj, lane >> 2);
            out.push_back(q < Q && j < N ? w[q] * E(c, q, j) : 0.0);
          }
  if (grp)
    for (int c = 0; c < NC; ++c)
      for (int nj = 0; nj < NJ; ++nj)
        for (int lane = 0; lane < 32; ++lane) {
          const int q = 8 * T + (lane & 3), j = col_dof(nj, lane >> 2);
          out.push_back(q < Q && j < N ? w[q] * E(c, q, j) : 0.0);
        }
  if (pair)
    for (int i = 0; i < 2; ++i)
      for (int nj = 0; nj < NJ; ++nj)
        for (int lane = 0; lane < 32; ++lane) {
          const int k = lane & 3, c = 2 * (k & 1) + i, q = 8 * T + (k >> 1), j = col_dof(nj, lane >> 2);
          out.push_back(q < Q && j < N && c < NC ? w[q] * E(c, q, j) : 0.0);
        }
}

// Reference-tensor fragments (cell_tensor_kernel.cuh): the quadrature sum of the
// reference's cell loop taken once, in extended precision, from the same tables:
//   S_0..5 (packed kl = 00,01,02,11,12,22)
//     S_kl(i, j) = sum_q w_q (G_k(q,i) G_l(q,j) + [k != l] G_l(q,i) G_k(q,j)),
//   S_6(i, j) = sum_q w_q V(q,i) V(q,j) (mass),  S_7 = 0;
//   B[ib][p][kk][lane] = S_{2p + (n&1)}(4ib + (n>>1), 4kk + (lane&3)),  n = lane>>2
template <typename FG, typename FV>
void build_tensor_fragments(int N, int Q, bool mass, FG Eg, FV Ev, const double* w, std::vector<double>& out) {
  static const int KL[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
  const int KK = (N + 3) / 4, NP = mass ? 4 : 3, NM = mass ? 7 : 6;
  std::vector<double> S((size_t)NM * N * N);
  for (int m = 0; m < NM; ++m)
    for (int i = 0; i < N; ++i)
      for (int j = 0; j < N; ++j) {
        long double s = 0.0L;
        for (int q = 0; q < Q; ++q) {
          long double t;
          if (m == 6) {
            t = (long double)Ev(q, i) * Ev(q, j);
          } else {
            const int k = KL[m][0], l = KL[m][1];
            t = (long double)Eg(k, q, i) * Eg(l, q, j);
            if (k != l) t += (long double)Eg(l, q, i) * Eg(k, q, j);
          }
          s += (long double)w[q] * t;
        }
        S[((size_t)m * N + i) * N + j] = (double)s;
      }
  for (int ib = 0; ib < KK; ++ib)
    for (int p = 0; p < NP; ++p)
      for (int kk = 0; kk < KK; ++kk)
        for (int lane = 0; lane < 32; ++lane) {
          const int n = lane >> 2, i = 4 * ib + (n >> 1), m = 2 * p + (n & 1), j = 4 * kk + (lane & 3);
          out.push_back(i < N && j < N && m < NM ? S[((size_t)m * N + i) * N + j] : 0.0);
        }
}

// Symmetric eigendecomposition by cyclic Jacobi rotations in long double (small n):
// A (n x n, row-major, destroyed) -> eigenvalues lam (descending) and eigenvectors V
// (column m of V belongs to lam[m]).
void jacobi_eigen(int n, std::vector<long double>& A, std::vector<long double>& lam, std::vector<long double>& V) {
  V.assign((size_t)n * n, 0.0L);
  for (int i = 0; i < n; ++i) V[(size_t)i * n + i] = 1.0L;
  auto a = [&](int i, int j) -> long double& { return A[(size_t)i * n + j]; };
  for (int sweep = 0; sweep < 100; ++sweep) {
    long double off = 0.0L, diag = 0.0L;
    for (int i = 0; i < n; ++i) {
      diag += a(i, i) * a(i, i);
      for (int j = i + 1; j < n; ++j) off += a(i, j) * a(i, j);
    }
    if (off <= 1e-36L * diag) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        if (a(p, q) == 0.0L) continue;
        const long double th = (a(q, q) - a(p, p)) / (2.0L * a(p, q));
        const long double t = (th >= 0 ? 1.0L : -1.0L) / (std::fabs(th) + std::sqrt(th * th + 1.0L));
        const long double c = 1.0L / std::sqrt(t * t + 1.0L), sn = t * c;
        for (int k = 0; k < n; ++k) {   // A <- A J (columns p, q)
          const long double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - sn * akq;
          a(k, q) = sn * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {   // A <- J^T A (rows p, q)
          const long double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - sn * aqk;
          a(q, k) = sn * apk + c * aqk;
        }
        for (int k = 0; k < n; ++k) {
          long double& vp = V[(size_t)k * n + p];
          long double& vq = V[(size_t)k * n + q];
          const long double x = vp, y = vq;
          vp = c * x - sn * y;
          vq = sn * x + c * y;
        }
      }
  }
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int x, int y) { return a(x, x) > a(y, y); });
  std::vector<long double> V2((size_t)n * n);
  lam.resize(n);
  for (int m = 0; m < n; ++m) {
    lam[m] = a(ord[m], ord[m]);
    for (int k = 0; k < n; ++k) V2[(size_t)k * n + m] = V[(size_t)k * n + ord[m]];
  }
  V.swap(V2);
}

// Modal cell tables.  The reference's cell term needs only the point sums
//   H[(k,i),(l,j)] = sum_q w_q d_k phi_i(q) d_l phi_j(q)          (3N x 3N)
// -- exact integrals of products of P_{p-1} polynomials, so H is positive semidefinite
// of rank M = dim P_{p-1} = p(p+1)(p+2)/6 (4 / 10 / 20 at P2 / P3 / P4) however many
// points the rule has (GM: 15 / 35 / 70).  With H = sum_m lam_m v_m v_m^T,
//   E'(k, m, i) = sqrt(lam_m) v_m[(k,i)]   satisfies   sum_m E'(k,m,i) E'(l,m,j) = H,
// i.e. E' is an M-"point" rule with unit weights that integrates the cell term exactly:
// the quadrature-point kernel (cell_kernel.cuh) runs on it unchanged, with M instead of
// n_q points.  Returns false unless the spectrum has the expected rank gap.
bool build_modal_cell_tables(int N, int Q, int M, const double* Gm, const double* w, std::vector<double>& E) {
  const int n = 3 * N;
  std::vector<long double> H((size_t)n * n, 0.0L);
  for (int a = 0; a < n; ++a)
    for (int b = a; b < n; ++b) {
      long double acc = 0.0L;
      const int k = a / N, i = a % N, l = b / N, j = b % N;
      for (int q = 0; q < Q; ++q) acc += (long double)w[q] * Gm[(3 * q + k) * N + i] * Gm[(3 * q + l) * N + j];
      H[(size_t)a * n + b] = H[(size_t)b * n + a] = acc;
    }
  std::vector<long double> lam, V;
  jacobi_eigen(n, H, lam, V);
  if (M >= n || !(lam[0] > 0) || !(lam[M - 1] > 1e-10L * lam[0]) || !(std::fabs(lam[M]) <= 1e-12L * lam[0]))
    return false;
  E.assign((size_t)3 * M * N, 0.0);   // layout of grad_matrix: row 3 m + k, column i
  for (int m = 0; m < M; ++m) {
    const long double s = std::sqrt(lam[m]);
    for (int k = 0; k < 3; ++k)
      for (int i = 0; i < N; ++i) E[(size_t)(3 * m + k) * N + i] = (double)(s * V[(size_t)(k * N + i) * n + m]);
  }
  return true;
}

// Face tables in the face frame (see face_kernel.cuh), for one (lf, code) combo.
// Components c: 0 = value, 1..3 = D_i = a_i . grad (a_0, a_1 tangent, a_2 transversal);
// columns are DoFs in the gather order perm (face DoFs first).  Point groups of 4:
//   B1[g][h=0][kk < KKF] / [h=1][kk < KK][lane] = E_{2h + (n&1)}(4g + (n>>1), 4kk + (lane&3)), n = lane>>2
//   B2[g][c<3][nj < NJF] / [c=3][nj < NJ][lane] = w_q E_c(q = 4g + (lane&3), 8nj + (lane>>2))
template <typename F>
void build_face_fragments(int N, int NF, int Q, F E, const double* w, std::vector<double>& out) {
  const int G = (Q + 3) / 4, KK = (N + 3) / 4, NJ = (N + 7) / 8, KKF = (NF + 3) / 4, NJF = (NF + 7) / 8;
  auto Ev = [&](int c, int q, int j) { return (q < Q && j < N) ? E(c, q, j) : 0.0; };
  for (int g = 0; g < G; ++g)
    for (int h = 0; h < 2; ++h)
      for (int kk = 0; kk < (h == 0 ? KKF : KK); ++kk)
        for (int lane = 0; lane < 32; ++lane) {
          const int n = lane >> 2;
          out.push_back(Ev(2 * h + (n & 1), 4 * g + (n >> 1), 4 * kk + (lane & 3)));
        }
  for (int g = 0; g < G; ++g)
    for (int c = 0; c < 4; ++c)
      for (int nj = 0; nj < (c < 3 ? NJF : NJ); ++nj)
        for (int lane = 0; lane < 32; ++lane) {
          const int q = 4 * g + (lane & 3), j = col_dof(nj, lane >> 2);   // the lane order of the gather
          out.push_back(q < Q && j < N ? w[q] * E(c, q, j) : 0.0);
        }
}

// Fragments of the split-mode modal face layout (face_kernel.cuh, HierShape): E(c, m, j) is
// the modal table (component c of mode m at gather position j), unit weights.
template <int N, class F>
void build_face_fragments_hier(F E, std::vector<double>& out) {
  using S = tmf::HierShape<N>;
  auto val = [&](int q, int s, int r, int j) {
    if (s < 0 || j >= N) return 0.0;
    const int m = S::item_mode(q, s, r);
    return m < 0 ? 0.0 : E(S::item_comp(q, s, r), m, j);
  };
  for (int t = 0; t < S::NTF; ++t)
    for (int kk = 0; kk < S::KKF; ++kk)
      for (int lane = 0; lane < 32; ++lane) {
        const int n = lane >> 2, q = n >> 1, i = n & 1;
        out.push_back(val(q, S::tf_s(t, i), S::tf_r(t, i), 4 * kk + (lane & 3)));
      }
  for (int d = 0; d < S::NTD; ++d)
    for (int kk = 0; kk < S::KK; ++kk)
      for (int lane = 0; lane < 32; ++lane) {
        const int n = lane >> 2, q = n >> 1, i = n & 1;
        out.push_back(val(q, S::td_s(d, i), S::td_r(d, i), 4 * kk + (lane & 3)));
      }
  for (int r3 = 0; r3 < 2; ++r3)          // face-only items first, then the D2 items (HierShape::b2)
    for (int s = 0; s < S::NS; ++s)
      for (int r = (r3 ? 3 : 0); r < (r3 ? 4 : 3); ++r)
        for (int nj = 0; nj < (r < 3 ? S::NJF : S::NJ); ++nj)
          for (int lane = 0; lane < 32; ++lane) out.push_back(val(lane & 3, s, r, col_dof(nj, lane >> 2)));
}

}  // namespace

struct tmf_plan {
  int dev = 0, n_sm = 0;
  int kind = 0, degree = 0, N = 0, Q = 0, QF = 0, nc = 1;
  int engine = 0;        // (desc.flags >> 13) & 3 (| 4 via bit 19): cell engine 0 = by degree,
                         // 1 = DMMA points, 3 = reference tensor, 4 = modal
  int kengine = 0;       // engine handed to the launcher (modal runs the point kernel: 1)
  int Qk = 0;            // "points" of the cell kernel (n_q, or M for the modal tables)
  int QFk = 0;           // "points" of the face kernel (n_qf, or NF for the modal face tables)
  cudaEvent_t ev_stage = nullptr;   // end of the last staged (host-buffer) apply
  int* dbg_flag = nullptr;          // TMF_DEBUG_CHECKS builds: device check flags (common.cuh)
  bool dg = false, mass = false, faces = false;
  int64_t n_cells = 0, n_verts = 0, n_scalar = 0, n_global = 0;
  double mass_scale = 0.0, stiff_scale = 1.0;
  size_t dev_bytes = 0;
  // device data
  double* verts = nullptr;
  double* kappa = nullptr;
  double* cell_frags = nullptr;
  double* cell_geo = nullptr;
  double* face_frags = nullptr;
  double* face_frags_h = nullptr;  // interior faces, split-mode modal layout (face engine 3)
  int face_engine = 0;             // (desc.flags >> 17) & 3: 0 by degree, 1 quadrature points,
                                   // 2 modal in the flat layout, 3 modal in the split-mode layout
  int* face_perm = nullptr;
  std::vector<int> face_perm_h;   // host copy (FaceArgs::permc)
  int* cells = nullptr;
  int* dofs = nullptr;
  int* fix_list = nullptr;
  int64_t n_fix = 0;
  // CG traversal order (flags bits 22-23: 0 auto, 1 input, 2 Morton): the tile kernels walk the
  // plan's per-cell arrays in this order; u / y keep the caller's numbering
  bool cell_perm = false;
  // CG block assembly (cell_block_kernel.cuh; flags bits 15-16: 0 auto, 1 off, 2 on)
  int blocks_mode = 0;
  int blk_B = 0;                   // cells per block (0: off)
  int64_t blk_n = 0;               // blocks
  int blk_numax = 0, blk_nvmax = 0;
  std::vector<double> blk_tab;     // modal table E'(k, m, j) at [(3 m + k) N + j] (kernel parameter)
  int* blk_off = nullptr;
  int* blk_nv = nullptr;
  int* blk_uniq = nullptr;
  uint16_t* blk_loc = nullptr;
  uint16_t* blk_inc = nullptr;
  uint16_t* blk_ioff = nullptr;
  double* blk_kappa = nullptr;
  // multi-GPU peer-memory ghost access (tmf_plan_set_peers)
  tmf::PeerArgs peer{};
  const double** peer_u_tab = nullptr;   // device arrays of device pointers
  double** peer_y_tab = nullptr;
  int* ghost_rank = nullptr;
  int* ghost_index = nullptr;
  const double* peer_self_u = nullptr;   // this rank's registered buffers
  double* peer_self_y = nullptr;
  int64_t n_peer_free = 0;               // CG: cells [0, n) touch no ghost DoF (plain kernel)
  int4* if_chunks = nullptr;
  int* if_cm = nullptr;
  int* if_cp = nullptr;
  double* if_tau = nullptr;
  double* if_geo = nullptr;
  int64_t n_if_batches = 0, n_if_chunks = 0;
  int face_run = 0;   // chunk-run length of the interior-face CTA walk (face_kernel.cuh ChunkWalk)
  int4* bf_chunks = nullptr;
  int* bf_cm = nullptr;
  double* bf_tau = nullptr;
  double* bf_geo = nullptr;
  int64_t n_bf_batches = 0, n_bf_chunks = 0;
  // staging for host applies / solver scratch
  // fp32 mirror for the mixed-precision multigrid (flags bit 20, CG Laplace): modal rows
  // E'[m][k][0..NP) as float4 and per-cell G as 8 floats (cell_f32_kernel.cuh)
  float4* f32_rows = nullptr;
  float* f32_geo = nullptr;
  int f32_M = 0;
  double* stage_u = nullptr;
  double* stage_y = nullptr;
  double* pcg_buf = nullptr;
  double* diag = nullptr;
  double* diag_S = nullptr;
  tmf_plan_info info{};
  // cell range [c0, c1): per-cell arrays are offset; CG u/y are global, DG u/y
  // are cell-contiguous and offset with the cells
  tmf::CellArgs cell_args(const double* u, double* y, int64_t c0 = 0, int64_t c1 = -1, bool with_peer = true) const {
    if (c1 < 0) c1 = n_cells;
    tmf::CellArgs a{};
    const int64_t off = dg ? c0 * N * nc : 0;
    a.u = u + off;
    a.y = y + off;
    a.dofs = dg ? nullptr : dofs + c0 * N;
    a.cgeo = cell_geo + 8 * c0;
    a.frags = cell_frags;
    a.n_cells = c1 - c0;
    a.nc = nc;
    if (!dg && with_peer) a.peer = peer;   // CG ghost DoFs over peer memory (DG: the face kernel's ghost cells)
#ifdef TMF_DEBUG_CHECKS
    a.dbg_n_dofs = dg ? (c1 - c0) * N * nc : n_global;
    a.dbg_n_cells = c1 - c0;
    a.dbg_flag = dbg_flag;
#endif
    return a;
  }
  tmf::BlockArgs block_args(const double* u, double* y, double* energy) const {
    tmf::BlockArgs a{};
    a.u = u;
    a.y = y;
    a.verts = verts;
    a.kappa = blk_kappa;
    a.boff = blk_off;
    a.bnv = blk_nv;
    a.uniq = blk_uniq;
    a.loc = blk_loc;
    a.inc = blk_inc;
    a.ioff = blk_ioff;
    a.n_cells = n_cells;
    a.n_blocks = blk_n;
    a.numax = blk_numax;
    a.nvmax = blk_nvmax;
    a.scale = stiff_scale;
    a.energy = energy;
#ifdef TMF_DEBUG_CHECKS
    a.dbg_n_dofs = n_global;
    a.dbg_n_cells = n_cells;
    a.dbg_flag = dbg_flag;
#endif
    return a;
  }
  tmf::FaceArgs face_args(const double* u, double* y, bool boundary) const {
    tmf::FaceArgs a{};
    a.u = u;
    a.y = y;
    a.frags = (!boundary && face_frags_h) ? face_frags_h : face_frags;
    a.hier = (!boundary && face_frags_h) ? 1 : 0;
    a.run = boundary ? 0 : face_run;
    a.chunks = boundary ? bf_chunks : if_chunks;
    a.cm = boundary ? bf_cm : if_cm;
    a.cp = boundary ? nullptr : if_cp;
    a.geo = boundary ? bf_geo : if_geo;
    a.perm = face_perm;
    for (size_t i = 0; i < face_perm_h.size() && i < sizeof(a.permc) / sizeof(int); ++i) a.permc[i] = face_perm_h[i];
    a.n_chunks = boundary ? n_bf_chunks : n_if_chunks;
    a.n_dpc = N;
    a.nc = nc;
    a.peer = peer;
#ifdef TMF_DEBUG_CHECKS
    a.dbg_n_dofs = n_global;
    a.dbg_n_cells = n_cells;
    a.dbg_flag = dbg_flag;
#endif
    return a;
  }
  tmf::FaceGeoArgs face_geo_args(bool boundary) const {
    tmf::FaceGeoArgs a{};
    a.cells = cells;
    a.verts = verts;
    a.kappa = kappa;
    a.chunks = boundary ? bf_chunks : if_chunks;
    a.cm = boundary ? bf_cm : if_cm;
    a.cp = boundary ? nullptr : if_cp;
    a.tau = boundary ? bf_tau : if_tau;
    a.geo = boundary ? bf_geo : if_geo;
    a.n_chunks = boundary ? n_bf_chunks : n_if_chunks;
    a.scale = stiff_scale;
    return a;
  }
  ~tmf_plan() {
    if (ev_stage) cudaEventDestroy(ev_stage);
    for (void* p : {(void*)verts, (void*)kappa, (void*)cell_frags, (void*)face_frags, (void*)face_frags_h, (void*)cells,
                    (void*)dofs, (void*)fix_list, (void*)if_chunks, (void*)if_cm, (void*)if_cp,
                    (void*)if_tau, (void*)bf_chunks, (void*)bf_cm, (void*)bf_tau, (void*)stage_u,
                    (void*)stage_y, (void*)pcg_buf, (void*)diag, (void*)diag_S, (void*)if_geo, (void*)bf_geo, (void*)cell_geo, (void*)face_perm,
                    (void*)f32_rows, (void*)f32_geo, (void*)blk_off, (void*)blk_nv, (void*)blk_uniq,
                    (void*)blk_loc, (void*)blk_inc, (void*)blk_ioff, (void*)blk_kappa, (void*)dbg_flag,
                    (void*)peer_u_tab, (void*)peer_y_tab, (void*)ghost_rank, (void*)ghost_index})
      if (p) cudaFree(p);
  }
};

namespace {

int n_dofs_per_cell(int p) { return (p + 1) * (p + 2) * (p + 3) / 6; }

// measured (profiles/r01/face_window_sweep.json): 512 / 2048 / 8192 / 32768 / 131072 minus
// cells per window -> DG P3 64^3 faces 1.224 / 1.045 / 0.930 / 0.889 / 0.888 ms, Helmholtz
// P2 96^3 1.576 / 1.459 / 1.406 / 1.392 / 1.412 ms (longer signature runs, fewer chunks)
constexpr int64_t kFaceWindow = 32768;

// Split [first, first+count) batches of one signature into CTA chunks.
void push_chunks(std::vector<int4>& out, int cm, int cp, int64_t first, int64_t count, int chunk) {
  for (int64_t b = 0; b < count; b += chunk)
    out.push_back(make_int4(cm, cp, (int)(first + b), (int)std::min<int64_t>(chunk, count - b)));
}

int build_face_batches(tmf_plan* P, const tmf_plan_desc* d, int chunk, size_t* total) {
  const int64_t nif = d->n_interior_faces, nbf = d->n_boundary_faces;
  // interior: stable sort by signature (lf-, lf+, code); faces keep their
  // owning-cell order inside a signature (mesh.py:117)
  std::vector<int64_t> order(nif);
  std::iota(order.begin(), order.end(), 0);
  // faces are grouped by signature inside windows of kFaceWindow consecutive minus
  // cells, so the GPU sweeps the cell range once (u/y stay L2-resident) instead of
  // once per signature
  auto sig = [&](int64_t f) {
    const int32_t* r = d->interior_faces + 5 * f;
    return (int64_t)(r[0] / kFaceWindow) * 96 + r[1] * 24 + r[3] * 6 + r[4];
  };
  for (int64_t f = 0; f < nif; ++f) {
    const int32_t* r = d->interior_faces + 5 * f;
    if (r[0] < 0 || r[0] >= d->n_cells || r[2] < 0 || r[2] >= d->n_cells || r[1] < 0 || r[1] > 3 ||
        r[3] < 0 || r[3] > 3 || r[4] < 0 || r[4] > 5)
      return fail(TMF_EINVAL, "interior face " + std::to_string(f) + " out of range");
  }
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return sig(a) < sig(b); });
  std::vector<int4> chunks;
  std::vector<int> cm, cp;
  std::vector<double> tau;
  int64_t nb = 0;
  for (int64_t s = 0; s < nif;) {
    const int64_t key = sig(order[s]);
    int64_t e = s;
    while (e < nif && sig(order[e]) == key) ++e;
    const int32_t* r0 = d->interior_faces + 5 * order[s];
    const int64_t nbatch = (e - s + 7) / 8;
    push_chunks(chunks, r0[1] * 6, r0[3] * 6 + r0[4], nb, nbatch, chunk);
    for (int64_t k = 0; k < nbatch * 8; ++k) {
      if (s + k < e) {
        const int64_t f = order[s + k];
        const int32_t* r = d->interior_faces + 5 * f;
        cm.push_back(r[0]);
        cp.push_back(r[2]);
        tau.push_back(d->tau_interior[f]);
      } else {
        cm.push_back(-1);
        cp.push_back(-1);
        tau.push_back(0.0);
      }
    }
    nb += nbatch;
    s = e;
  }
  P->n_if_batches = nb;
  P->n_if_chunks = (int64_t)chunks.size();
  // CTA walk of the interior faces (face_kernel.cuh ChunkWalk).  P3: short chunk runs dealt
  // round-robin, so the CTAs sweep the windows together and the faces of a cell find its
  // u / y rows in L2 -- runs of 2 when the numbering has locality (consecutive chunks share
  // their tables), single chunks when it has not.  Measured with the 128-thread CTAs
  // (profiles/r02/face_runs.jsonl), DG P3 64^3 faces, run 0 (one contiguous run per CTA, round
  // 1) / 1 / 2 / 3: reordered 0.84 (256-thread CTAs) / 0.642 / 0.631 / 0.640 ms, unordered
  // 0.93 / 0.664 / 0.685 / 0.752 ms.  P4's 3-stage ring kernel is slower with any run length
  // (larger tables to restage: 40^3 0.424 -> 0.459 ms); P2's register-table kernel deals chunks
  // round-robin.  TMF_FACE_RUN (environment, experiments) overrides.
  {
    int64_t near = 0;
    for (int64_t f = 0; f < nif; ++f) {
      const int32_t* r = d->interior_faces + 5 * f;
      if (r[0] / kFaceWindow == r[2] / kFaceWindow) ++near;
    }
    const bool local = nif > 0 && 2 * near >= nif;
    P->face_run = P->N == 20 ? (local ? 2 : 1) : 0;
    if (const char* e = std::getenv("TMF_FACE_RUN")) P->face_run = std::atoi(e);
  }
  int rc;
  if ((rc = upload(&P->if_chunks, chunks.data(), chunks.size(), total))) return rc;
  if ((rc = upload(&P->if_cm, cm.data(), cm.size(), total))) return rc;
  if ((rc = upload(&P->if_cp, cp.data(), cp.size(), total))) return rc;
  if ((rc = upload(&P->if_tau, tau.data(), tau.size(), total))) return rc;

  // Dirichlet boundary faces grouped by local face (operator.py:365-366, 378-385)
  std::vector<int4> bchunks;
  std::vector<int> bcm;
  std::vector<double> btau;
  nb = 0;
  std::vector<std::vector<int64_t>> groups;
  {
    std::vector<int64_t> bord;
    for (int64_t f = 0; f < nbf; ++f)
      if (d->boundary_dirichlet && d->boundary_dirichlet[f]) bord.push_back(f);
    auto bsig = [&](int64_t f) {
      const int32_t* r = d->boundary_faces + 3 * f;
      return (int64_t)(r[0] / kFaceWindow) * 4 + r[1];
    };
    std::stable_sort(bord.begin(), bord.end(), [&](int64_t a, int64_t b) { return bsig(a) < bsig(b); });
    for (size_t s = 0; s < bord.size();) {
      size_t e = s;
      while (e < bord.size() && bsig(bord[e]) == bsig(bord[s])) ++e;
      groups.emplace_back(bord.begin() + s, bord.begin() + e);
      s = e;
    }
  }
  for (const auto& sel : groups) {
    const int lf = d->boundary_faces[3 * sel[0] + 1];
    const int64_t nbatch = ((int64_t)sel.size() + 7) / 8;
    push_chunks(bchunks, lf * 6, -1, nb, nbatch, chunk);
    for (int64_t k = 0; k < nbatch * 8; ++k) {
      if (k < (int64_t)sel.size()) {
        const int64_t f = sel[k];
        const int32_t c = d->boundary_faces[3 * f];
        if (c < 0 || c >= d->n_cells) return fail(TMF_EINVAL, "boundary face cell out of range");
        bcm.push_back(c);
        btau.push_back(d->tau_boundary ? d->tau_boundary[f] : 0.0);
      } else {
        bcm.push_back(-1);
        btau.push_back(0.0);
      }
    }
    nb += nbatch;
  }
  P->n_bf_batches = nb;
  P->n_bf_chunks = (int64_t)bchunks.size();
  if ((rc = upload(&P->bf_chunks, bchunks.data(), bchunks.size(), total))) return rc;
  if ((rc = upload(&P->bf_cm, bcm.data(), bcm.size(), total))) return rc;
  if ((rc = upload(&P->bf_tau, btau.data(), btau.size(), total))) return rc;
  return TMF_OK;
}

// Cells in Morton order of their centroids (21 bits per axis in the vertices' bounding box),
// ties by cell id: the plans' locality traversal order (a permutation of 0..n-1).
std::vector<int64_t> morton_order(const tmf_plan_desc* d) {
  const int64_t n = d->n_cells;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t v = 0; v < d->n_vertices; ++v)
    for (int k = 0; k < 3; ++k) {
      lo[k] = std::min(lo[k], d->vertices[3 * v + k]);
      hi[k] = std::max(hi[k], d->vertices[3 * v + k]);
    }
  auto spread = [](uint64_t x) {
    x &= 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffULL;
    x = (x | x << 16) & 0x1f0000ff0000ffULL;
    x = (x | x << 8) & 0x100f00f00f00f00fULL;
    x = (x | x << 4) & 0x10c30c30c30c30c3ULL;
    x = (x | x << 2) & 0x1249249249249249ULL;
    return x;
  };
  std::vector<std::pair<uint64_t, int64_t>> key(n);
  for (int64_t c = 0; c < n; ++c) {
    uint64_t code = 0;
    for (int k = 0; k < 3; ++k) {
      double x = 0.0;
      for (int i = 0; i < 4; ++i) x += d->vertices[3 * (int64_t)d->cells[c * 4 + i] + k];
      const double t = hi[k] > lo[k] ? (0.25 * x - lo[k]) / (hi[k] - lo[k]) : 0.0;
      code |= spread((uint64_t)std::min(2097151.0, std::max(0.0, t * 2097152.0))) << k;
    }
    key[c] = {code, c};
  }
  std::sort(key.begin(), key.end());
  std::vector<int64_t> order(n);
  for (int64_t i = 0; i < n; ++i) order[i] = key[i].second;
  return order;
}

// Mean distance between the centroids of consecutive cells of an order (a locality measure).
double consecutive_distance(const tmf_plan_desc* d, const int64_t* order) {
  const int64_t n = d->n_cells;
  if (n < 2) return 0.0;
  double acc = 0.0, prev[3] = {0, 0, 0};
  for (int64_t i = 0; i < n; ++i) {
    const int64_t c = order ? order[i] : i;
    double x[3] = {0, 0, 0};
    for (int k = 0; k < 3; ++k)
      for (int j = 0; j < 4; ++j) x[k] += 0.25 * d->vertices[3 * (int64_t)d->cells[c * 4 + j] + k];
    if (i) acc += std::sqrt((x[0] - prev[0]) * (x[0] - prev[0]) + (x[1] - prev[1]) * (x[1] - prev[1]) +
                            (x[2] - prev[2]) * (x[2] - prev[2]));
    for (int k = 0; k < 3; ++k) prev[k] = x[k];
  }
  return acc / (double)(n - 1);
}

// CG block assembly tables (cell_block_kernel.cuh).  Cells are taken in Morton order of
// their centroids (a locality order of the plan's own; the input numbering of cells and
// DoFs is unchanged, the sum over cells does not depend on the order) and cut into blocks
// of B.  Per block: its unique global DoFs sorted ascending (so the vertex DoFs, ids <
// n_vertices in the reference numbering, come first), each slot's local index (u16), and
// the slots of every unique DoF (u16 j*B + cl, in slot order) with their offsets.
// Returns TMF_OK with P->blk_B = 0 when the plan does not qualify (vertex DoFs are not the
// vertex ids, or a block does not fit in shared memory).
int build_blocks(tmf_plan* P, const tmf_plan_desc* d, int B, size_t* total) {
  const int N = P->N, NP = (N + 3) & ~3;
  const int64_t n = P->n_cells;
  for (int64_t c = 0; c < n; ++c)
    for (int j = 0; j < 4; ++j)
      if (d->cell_dofs[c * N + j] != d->cells[c * 4 + j]) return TMF_OK;   // not the reference numbering
  const std::vector<int64_t> order = morton_order(d);
  const int64_t nb = (n + B - 1) / B;
  std::vector<std::vector<int>> uq(nb);
  std::vector<std::vector<uint16_t>> io(nb);
  std::vector<int> nvb(nb);
  std::vector<uint16_t> loc((size_t)n * NP, 0), inc((size_t)nb * B * N + 8, 0);
  const int nth = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (int t = 0; t < nth; ++t)
    pool.emplace_back([&, t]() {
      std::vector<std::pair<int, int>> pr;   // (global DoF, slot)
      for (int64_t b = t; b < nb; b += nth) {
        const int64_t c0 = b * B;
        const int ncb = (int)std::min<int64_t>(B, n - c0);
        pr.clear();
        for (int cl = 0; cl < ncb; ++cl) {
          const int64_t c = order[c0 + cl];
          for (int j = 0; j < N; ++j) pr.emplace_back(d->cell_dofs[c * N + j], j * B + cl);
        }
        std::sort(pr.begin(), pr.end());
        std::vector<int>& U = uq[b];
        std::vector<uint16_t>& O = io[b];
        uint16_t* I = inc.data() + (size_t)b * B * N;
        int nv = 0;
        for (size_t k = 0; k < pr.size(); ++k) {
          if (k == 0 || pr[k].first != pr[k - 1].first) {
            const int g = pr[k].first;
            U.push_back(d->dirichlet_mask && d->dirichlet_mask[g] ? ~g : g);
            O.push_back((uint16_t)k);
            if (g < d->n_vertices) ++nv;
          }
          I[k] = (uint16_t)pr[k].second;
          const int slot = pr[k].second, j = slot / B, cl = slot % B;
          loc[(size_t)(c0 + cl) * NP + j] = (uint16_t)(U.size() - 1);
        }
        O.push_back((uint16_t)pr.size());
        nvb[b] = nv;
      }
    });
  for (auto& th : pool) th.join();
  std::vector<int> off(nb + 1, 0), uniq;
  std::vector<uint16_t> ioff;
  int numax = 0, nvmax = 0;
  for (int64_t b = 0; b < nb; ++b) {
    off[b + 1] = off[b] + (int)uq[b].size();
    numax = std::max(numax, (int)uq[b].size());
    nvmax = std::max(nvmax, nvb[b]);
  }
  if (numax > 65535 || tmf::block_smem_bytes(N, B, numax, nvmax) > 227 * 1024) return TMF_OK;
  uniq.reserve(off[nb]);
  ioff.reserve(off[nb] + nb);
  for (int64_t b = 0; b < nb; ++b) {
    uniq.insert(uniq.end(), uq[b].begin(), uq[b].end());
    ioff.insert(ioff.end(), io[b].begin(), io[b].end());
  }
  int rc;
  if ((rc = upload(&P->blk_off, off.data(), off.size(), total))) return rc;
  if ((rc = upload(&P->blk_nv, nvb.data(), nvb.size(), total))) return rc;
  if ((rc = upload(&P->blk_uniq, uniq.data(), uniq.size(), total))) return rc;
  if ((rc = upload(&P->blk_loc, loc.data(), loc.size(), total))) return rc;
  if ((rc = upload(&P->blk_inc, inc.data(), inc.size(), total))) return rc;
  if ((rc = upload(&P->blk_ioff, ioff.data(), ioff.size(), total))) return rc;
  if (d->kappa) {
    std::vector<double> kp(n);
    for (int64_t i = 0; i < n; ++i) kp[i] = d->kappa[order[i]];
    if ((rc = upload(&P->blk_kappa, kp.data(), kp.size(), total))) return rc;
  }
  P->blk_B = B;
  P->blk_n = nb;
  P->blk_numax = numax;
  P->blk_nvmax = nvmax;
  P->info.block_cells = B;
  P->info.block_ratio = (double)off[nb] / ((double)n * N);
  return TMF_OK;
}

#ifdef TMF_DEBUG_CHECKS
// Debug build: wait for the apply and report any index the kernels found out of range.
int debug_flag_check(tmf_plan* P, cudaStream_t st) {
  TMF_CUDA(cudaStreamSynchronize(st));
  int flag = 0;
  TMF_CUDA(cudaMemcpy(&flag, P->dbg_flag, sizeof(int), cudaMemcpyDeviceToHost));
  if (flag) {
    TMF_CUDA(cudaMemset(P->dbg_flag, 0, sizeof(int)));
    return fail(TMF_ECUDA, "debug bounds check failed in a kernel: flags " + std::to_string(flag) +
                               " (1 DoF index, 2 cell, 4 face position, 8 block-local index, 16 block slots)");
  }
  return TMF_OK;
}
#endif

// TMF_PDL=0 (read once): cudaMemsetAsync + a plain cell-kernel launch instead of the clear
// kernel with its programmatic dependent (launch_apply)
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TMF_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// y_zeroed: the caller already cleared y (CG); energy: += sum_e u_e^T A_e u_e + the identity
// rows' u_i^2 (= u.Au when the tensor cell engine runs; PCG's fused p.Ap)
int launch_apply(tmf_plan* P, const double* u, double* y, cudaStream_t st, cudaEvent_t* ev,
                 bool y_zeroed = false, double* energy = nullptr) {
  bool ok = true;
  if (ev) TMF_CUDA(cudaEventRecord(ev[0], st));
  // CG: y is cleared by a kernel that releases its dependents at once, and the cell kernel is
  // launched as its programmatic dependent (its launch, table staging and first gathers
  // overlap the clear; it waits before its first RED).  TMF_PDL=0: cudaMemsetAsync + plain launch.
  const bool pdl = pdl_enabled() && !P->dg && !y_zeroed && P->n_cells > 0;
  if (pdl) TMF_CUDA(tmf::launch_zero(y, P->n_global, P->n_sm, st));
  else if (!P->dg && !y_zeroed) TMF_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * P->n_global, st));
  struct PdlScope {
    explicit PdlScope(bool on) { tmf::tl_pdl = on; }
    ~PdlScope() { tmf::tl_pdl = false; }
  };
  {
    PdlScope scope(pdl);
    if (P->blk_B && !P->peer.u) {
      TMF_CUDA(tmf::launch_cell_block(P->N, P->block_args(u, y, energy), P->blk_tab.data(), st));
    } else {
      tmf::CellArgs ca = P->cell_args(u, y);
      ca.energy = energy;
      TMF_CUDA(tmf::launch_cell(P->N, P->Qk, P->mass, P->dg, ca, P->n_sm, st, nullptr, &ok, P->kengine));
    }
  }
  // stage events only between kernels that exist (an event record between two empty
  // stages still costs ~3 us of GPU time, which would inflate the measured apply)
  const bool fix = !P->dg && P->n_fix;
  if (ev && (P->faces || fix)) TMF_CUDA(cudaEventRecord(ev[1], st));
  if (P->faces) {
    // DG: each face kernel is the programmatic dependent of the kernel before it (its CTAs set up
    // while that one drains; they wait before touching y).  A stage event in between (timed
    // applies) makes the first one an ordinary launch again.
    PdlScope scope(pdl_enabled() && P->n_cells > 0);
    TMF_CUDA(tmf::launch_face(P->N, P->QFk, false, P->face_args(u, y, false), P->n_sm, st, nullptr, &ok));
    TMF_CUDA(tmf::launch_face(P->N, P->QFk, true, P->face_args(u, y, true), P->n_sm, st, nullptr, &ok));
  }
  if (ev && P->faces && fix) TMF_CUDA(cudaEventRecord(ev[2], st));
  if (fix) TMF_CUDA(tmf::launch_fixup(u, y, P->fix_list, P->n_fix, P->n_sm, st, energy));
  if (ev) TMF_CUDA(cudaEventRecord(ev[3], st));
#ifdef TMF_DEBUG_CHECKS
  if (int rc = debug_flag_check(P, st)) return rc;
#endif
  return TMF_OK;
}

}  // namespace

extern "C" {

int tmf_apply_stages(tmf_plan* P, const double* u, double* y, int stages, int64_t cell_begin,
                     int64_t cell_end, void* stream) {
  if (!P || !u || !y) return fail(TMF_EINVAL, "null argument");
  if (cell_begin < 0 || cell_end > P->n_cells || cell_begin > cell_end)
    return fail(TMF_EINVAL, "bad cell range");
  if (P->cell_perm && (stages & TMF_STAGE_CELLS) && cell_end > cell_begin && (cell_begin != 0 || cell_end != P->n_cells))
    return fail(TMF_EINVAL, "the plan traverses cells in its own (Morton) order: cell ranges need the caller's "
                            "order (flags bits 22-23 = 1, OperatorConfig(cell_order='input'))");
  if (P->peer.u && (u != P->peer_self_u || (!P->dg && y != P->peer_self_y)))
    return fail(TMF_EINVAL, "with peers, u (and y for CG) must be this rank's registered buffers");
  TMF_CUDA(cudaSetDevice(P->dev));
  cudaStream_t st = (cudaStream_t)stream;
  bool ok = true;
  if ((stages & TMF_STAGE_ZERO) && !P->dg)
    TMF_CUDA(cudaMemsetAsync(y, 0, sizeof(double) * P->n_global, st));
  if ((stages & TMF_STAGE_CELLS) && cell_end > cell_begin) {
    if (P->peer.u && !P->dg) {
      // cells touching no ghost DoF run the plain kernel, the rest the peer-memory one
      const int64_t m = std::min(std::max(P->n_peer_free, cell_begin), cell_end);
      if (m > cell_begin)
        TMF_CUDA(tmf::launch_cell(P->N, P->Qk, P->mass, P->dg, P->cell_args(u, y, cell_begin, m, false), P->n_sm,
                                  st, nullptr, &ok, P->kengine));
      if (cell_end > m)
        TMF_CUDA(tmf::launch_cell(P->N, P->Qk, P->mass, P->dg, P->cell_args(u, y, m, cell_end), P->n_sm, st,
                                  nullptr, &ok, P->kengine));
    } else {
      TMF_CUDA(tmf::launch_cell(P->N, P->Qk, P->mass, P->dg, P->cell_args(u, y, cell_begin, cell_end), P->n_sm,
                                st, nullptr, &ok, P->kengine));
    }
  }
  if ((stages & TMF_STAGE_FACES) && P->faces) {
    TMF_CUDA(tmf::launch_face(P->N, P->QFk, false, P->face_args(u, y, false), P->n_sm, st, nullptr, &ok));
    TMF_CUDA(tmf::launch_face(P->N, P->QFk, true, P->face_args(u, y, true), P->n_sm, st, nullptr, &ok));
  }
  if ((stages & TMF_STAGE_FIXUP) && !P->dg && P->n_fix)
    TMF_CUDA(tmf::launch_fixup(u, y, P->fix_list, P->n_fix, P->n_sm, st));
  return TMF_OK;
}

const char* tmf_last_error(void) { return g_err.c_str(); }

// error reporting for the other C-ABI translation units (multigrid.cu); not in the header
int tmf_internal_set_error(int code, const char* msg) { return fail(code, msg); }
#ifdef TMF_DEBUG_CHECKS
const char* tmf_version(void) { return "tetmf_b200 0.2 (sm_100a, fp64 DMMA) DEBUG-CHECKS"; }
#else
const char* tmf_version(void) { return "tetmf_b200 0.2 (sm_100a, fp64 DMMA)"; }
#endif

int tmf_plan_create(const tmf_plan_desc* d, tmf_plan** out) {
  if (!d || !out) return fail(TMF_EINVAL, "null descriptor/output");
  *out = nullptr;
  if (d->operator_kind < TMF_CG_LAPLACE || d->operator_kind > TMF_DG_HELMHOLTZ)
    return fail(TMF_EINVAL, "unknown operator kind " + std::to_string(d->operator_kind));
  if (d->degree < 1 || d->degree > 4)
    return fail(TMF_EINVAL, "unsupported polynomial degree " + std::to_string(d->degree));
  if (d->n_dofs_per_cell != n_dofs_per_cell(d->degree))
    return fail(TMF_EINVAL, "n_dofs_per_cell does not match the degree");
  if (d->n_components != 1 && d->n_components != 3)
    return fail(TMF_EINVAL, "n_components must be 1 or 3");
  if (d->n_cells <= 0 || d->n_vertices <= 0 || !d->vertices || !d->cells)
    return fail(TMF_EINVAL, "empty mesh");
  if (!d->grad_matrix || !d->cell_weights || d->n_q <= 0) return fail(TMF_EINVAL, "missing cell tables");
  const bool dg = d->operator_kind != TMF_CG_LAPLACE;
  if (!dg && !d->cell_dofs) return fail(TMF_EINVAL, "CG operator needs a CG dof map");
  if (dg && d->n_scalar_dofs != d->n_cells * d->n_dofs_per_cell)
    return fail(TMF_EINVAL, "DG operator needs a DG dof map");
  if (d->n_scalar_dofs >= ((int64_t)1 << 31)) return fail(TMF_EINVAL, "too many dofs for int32 indexing");
  if (d->operator_kind == TMF_DG_HELMHOLTZ && !d->value_matrix)
    return fail(TMF_EINVAL, "Helmholtz needs the value table");
  const bool faces = dg && !(d->operator_kind == TMF_DG_HELMHOLTZ && d->diffusivity == 0.0);
  if (faces && (!d->face_values || !d->face_grads || !d->face_weights || d->n_qf <= 0))
    return fail(TMF_EINVAL, "geometry was built without face data");
  if (faces && d->n_interior_faces > 0 && (!d->interior_faces || !d->tau_interior))
    return fail(TMF_EINVAL, "missing interior faces / penalty");
  for (int64_t f = 0; faces && f < d->n_interior_faces; ++f)
    if (!(d->tau_interior[f] > 0)) return fail(TMF_EINVAL, "non-positive interior penalty");

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(TMF_ECUDA, "no CUDA device available (tetmf_b200 has no CPU path)");
  if (d->device < 0 || d->device >= ndev) return fail(TMF_EINVAL, "bad device ordinal");
  TMF_CUDA(cudaSetDevice(d->device));

  auto P = new tmf_plan();
  auto bail = [&](int rc) {
    delete P;
    return rc;
  };
#ifdef TMF_DEBUG_CHECKS
  TMF_CUDA(cudaMalloc(&P->dbg_flag, sizeof(int)));
  TMF_CUDA(cudaMemset(P->dbg_flag, 0, sizeof(int)));
#endif
  P->dev = d->device;
  {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->device);
    P->n_sm = sms;
  }
  P->kind = d->operator_kind;
  P->engine = ((d->flags >> 13) & 3) | (((d->flags >> 19) & 1) << 2);
  if (P->engine == 2) return bail(fail(TMF_EINVAL, "cell engine 2 (DFMA) was removed: use auto, dmma, tensor or modal"));
  P->face_engine = (d->flags >> 17) & 3;
  P->degree = d->degree;
  P->N = d->n_dofs_per_cell;
  P->Q = d->n_q;
  P->QF = d->n_qf;
  P->nc = d->n_components;
  P->dg = dg;
  P->mass = d->operator_kind == TMF_DG_HELMHOLTZ;
  P->faces = faces;
  P->n_cells = d->n_cells;
  P->n_verts = d->n_vertices;
  P->n_scalar = d->n_scalar_dofs;
  P->n_global = d->n_scalar_dofs * d->n_components;
  P->mass_scale = P->mass ? d->mass_scale : 0.0;
  P->stiff_scale = d->operator_kind == TMF_CG_LAPLACE ? 1.0 : d->diffusivity;

  // validate mesh connectivity
  for (int64_t i = 0; i < 4 * d->n_cells; ++i)
    if (d->cells[i] < 0 || d->cells[i] >= d->n_vertices)
      return bail(fail(TMF_EINVAL, "cell vertex id out of range"));

  size_t total = 0;
  int rc;
  if ((rc = upload(&P->verts, d->vertices, 3 * d->n_vertices, &total))) return bail(rc);
  // CG traversal order: auto takes the Morton order of the centroids when the caller's cell
  // order has no locality (mean centroid distance of consecutive cells > 2x the Morton order's:
  // a randomly permuted mesh), keeps the caller's order otherwise (a locality-ordered mesh is
  // as fast or faster, its DoF numbering following it; profiles/r02/cell_order.jsonl)
  std::vector<int64_t> order;
  {
    const int mode = (d->flags >> 22) & 3;
    if (!dg && mode != 1) {
      order = morton_order(d);
      if (mode == 0 && !(consecutive_distance(d, nullptr) > 2.0 * consecutive_distance(d, order.data())))
        order.clear();
    }
    P->cell_perm = !order.empty();
    P->info.cell_order = dg ? 0 : (P->cell_perm ? 2 : 1);
  }
  std::vector<int32_t> cells_p;
  std::vector<double> kappa_p;
  const int32_t* cells_in = d->cells;
  const double* kappa_in = d->kappa;
  if (P->cell_perm) {
    cells_p.resize((size_t)4 * d->n_cells);
    for (int64_t i = 0; i < d->n_cells; ++i)
      for (int k = 0; k < 4; ++k) cells_p[4 * i + k] = d->cells[4 * order[i] + k];
    cells_in = cells_p.data();
    if (d->kappa) {
      kappa_p.resize(d->n_cells);
      for (int64_t i = 0; i < d->n_cells; ++i) kappa_p[i] = d->kappa[order[i]];
      kappa_in = kappa_p.data();
    }
  }
  if ((rc = upload(&P->cells, cells_in, 4 * d->n_cells, &total))) return bail(rc);
  if (kappa_in && (rc = upload(&P->kappa, kappa_in, d->n_cells, &total))) return bail(rc);

  // cell tables -> fragments
  {
    const int N = P->N;
    const double* V = d->value_matrix;
    const double* Gm = d->grad_matrix;
    const double* W = d->cell_weights;
    int Q = P->Q;
    // engine by default: modal tables on the point kernel for Laplace cell terms at P2-P4
    // (DMMAs per 8-cell tile 12 / 52 / 147 against 27 / 75 / 243 for the reference tensor
    // and 42 / 151 / 513 for the n_q-point loop), the reference tensor otherwise (P1, mass)
    std::vector<double> modal, ones;
    int eng = P->engine;
    if (eng == 0) eng = N >= 10 ? 4 : 3;
    const bool modal_mass = eng == 4 && P->mass;   // mass term as a separate GEMM (MM kernels)
    if (eng == 4) {
      const int p = P->degree, M = p * (p + 1) * (p + 2) / 6;
      if (P->mass && (!P->dg || N < 10))
        return bail(fail(TMF_EINVAL, "the modal cell engine with a mass term is built for DG at P2-P4"));
      if (!build_modal_cell_tables(N, Q, M, Gm, W, modal))
        return bail(fail(TMF_EINVAL, "modal cell engine: gradient tables without the P_{p-1} rank structure"));
      Gm = modal.data();
      ones.assign(M, 1.0);
      W = ones.data();
      Q = M;
    }
    P->engine = eng;
    P->kengine = eng == 4 ? 1 : eng;
    P->Qk = Q;
    tmf::CellLaunchInfo ci;
    bool ok = true;
    tmf::CellArgs dummy{};
    dummy.n_cells = P->n_cells;
    dummy.nc = P->nc;
    TMF_CUDA(tmf::launch_cell(N, Q, P->mass, P->dg, dummy, P->n_sm, 0, &ci, &ok, P->kengine));
    if (!ok) return bail(fail(TMF_EINVAL, "unsupported (n_dofs_per_cell, n_q) = (" +
                                              std::to_string(N) + ", " + std::to_string(Q) + ")"));
    const int NC = (P->mass && !modal_mass) ? 4 : 3;
    auto E = [&](int c, int q, int j) {
      if (NC == 4) return c == 0 ? V[q * N + j] : Gm[(3 * q + c - 1) * N + j];
      return Gm[(3 * q + c) * N + j];
    };
    std::vector<double> fr;
    if (ci.table == 2)
      build_tensor_fragments(
          N, Q, P->mass, [&](int k, int q, int j) { return Gm[(3 * q + k) * N + j]; },
          [&](int q, int j) { return V[q * N + j]; }, W, fr);
    else
      build_fragments(N, Q, NC, E, W, fr);
    if (modal_mass) {
      // B3[kk][nj][lane] = M(4kk + (lane&3), 8nj + (lane>>2)), M = sum_q w_q phi_i phi_j over the
      // plan's n_q-point rule (the reference's mass_action, numpy_backend.py:79-88), long double
      const int KK = (N + 3) / 4, NJ = (N + 7) / 8;
      for (int kk = 0; kk < KK; ++kk)
        for (int nj = 0; nj < NJ; ++nj)
          for (int lane = 0; lane < 32; ++lane) {
            const int i = 4 * kk + (lane & 3), j = col_dof(nj, lane >> 2);
            long double acc = 0.0L;
            if (i < N && j < N)
              for (int q = 0; q < P->Q; ++q)
                acc += (long double)d->cell_weights[q] * (long double)V[q * N + i] * (long double)V[q * N + j];
            fr.push_back((double)acc);
          }
    }
    if ((int)fr.size() != ci.frag_doubles) return bail(fail(TMF_EINVAL, "internal: fragment size"));
    if ((rc = upload(&P->cell_frags, fr.data(), fr.size(), &total))) return bail(rc);
    P->info.flops_issued = ci.flops_issued;
    P->info.cell_engine = eng == 4 ? 4 : ci.table == 2 ? 3 : 1;
  }

  // per-cell geometry (G, mass factor), computed once on the device
  {
    TMF_CUDA(cudaMalloc(&P->cell_geo, sizeof(double) * 8 * P->n_cells));
    total += sizeof(double) * 8 * P->n_cells;
    tmf::CellGeoArgs g{P->cells, P->verts, P->kappa, P->cell_geo, P->n_cells, P->stiff_scale, P->mass_scale};
    TMF_CUDA(tmf::launch_cell_geometry(g, P->n_sm, 0));
  }

  // CG dof map (masked = ~idx) and the Dirichlet fix-up list
  if (!dg) {
    std::vector<int> enc((size_t)d->n_cells * P->N);
    for (int64_t i = 0; i < (int64_t)enc.size(); ++i) {
      const int64_t c = P->cell_perm ? order[i / P->N] : i / P->N;
      const int g = d->cell_dofs[c * P->N + i % P->N];
      if (g < 0 || g >= d->n_scalar_dofs) return bail(fail(TMF_EINVAL, "cell dof out of range"));
      enc[i] = (d->dirichlet_mask && d->dirichlet_mask[g]) ? ~g : g;
    }
    if ((rc = upload(&P->dofs, enc.data(), enc.size(), &total))) return bail(rc);
    // block assembly for the scalar Laplace at P1-P3 (flags bits 15-16: 0 auto = on, 1 off, 2 on);
    // the tile kernels stay built for the multi-GPU stages (peer ghosts, cell ranges)
    P->blocks_mode = (d->flags >> 15) & 3;
    const int Bc = tmf::block_cells_for(P->N);
    const int req_engine = ((d->flags >> 13) & 3) | (((d->flags >> 19) & 1) << 2);
    // auto: P1 only (48^3: 28 vs 31-33 us per apply for the tensor tile kernel; at P2 the modal
    // tile kernel is as fast or faster, 54-63 vs 59-67 us; profiles/r02/block_assembly.jsonl)
    const bool want = P->blocks_mode == 2 || (P->blocks_mode == 0 && req_engine == 0 && P->N == 4);
    if (want && Bc > 0 && P->nc == 1 && !P->mass && (req_engine == 0 || req_engine == 4)) {
      const int p = P->degree, M = p * (p + 1) * (p + 2) / 6;
      if (build_modal_cell_tables(P->N, P->Q, M, d->grad_matrix, d->cell_weights, P->blk_tab)) {
        if ((rc = build_blocks(P, d, Bc, &total))) return bail(rc);
        if (P->blk_B) P->info.cell_engine = 5;
      }
    }
    if (P->blocks_mode == 2 && !P->blk_B)
      return bail(fail(TMF_EINVAL, "block assembly requested but the plan does not qualify (scalar CG "
                                   "Laplace at P1-P3 with the reference DoF numbering, modal or auto engine)"));
    std::vector<int> fix;
    if (d->dirichlet_mask)
      for (int64_t g = 0; g < d->n_scalar_dofs; ++g)
        if (d->dirichlet_mask[g])
          for (int c = 0; c < P->nc; ++c) fix.push_back((int)(g * P->nc + c));
    P->n_fix = (int64_t)fix.size();
    if ((rc = upload(&P->fix_list, fix.data(), fix.size(), &total))) return bail(rc);
    // S_kl[j] = sum_q w_q E_k(q,j) E_l(q,j) for the matrix-free diagonal
    const int N = P->N, Q = P->Q;
    std::vector<double> S(6 * N, 0.0);
    const int kl[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};
    for (int m = 0; m < 6; ++m)
      for (int j = 0; j < N; ++j)
        for (int q = 0; q < Q; ++q)
          S[m * N + j] += d->cell_weights[q] * d->grad_matrix[(3 * q + kl[m][0]) * N + j] *
                          d->grad_matrix[(3 * q + kl[m][1]) * N + j];
    if ((rc = upload(&P->diag_S, S.data(), S.size(), &total))) return bail(rc);
  }

  // fp32 mirror (flags bit 20): the modal rows of the reference tables and G in fp32
  if ((d->flags >> 20) & 1) {
    if (dg || P->mass || P->nc != 1 || P->kind != TMF_CG_LAPLACE)
      return bail(fail(TMF_EINVAL, "the fp32 mirror is for scalar CG Laplace plans only"));
    const int N = P->N, p = P->degree, M = p * (p + 1) * (p + 2) / 6, NP = (N + 3) & ~3;
    std::vector<double> E;
    if (!build_modal_cell_tables(N, P->Q, M, d->grad_matrix, d->cell_weights, E))
      return bail(fail(TMF_EINVAL, "fp32 mirror: gradient tables without the P_{p-1} rank structure"));
    std::vector<float> rows((size_t)M * 3 * NP, 0.0f);
    for (int m = 0; m < M; ++m)
      for (int k = 0; k < 3; ++k)
        for (int j = 0; j < N; ++j) rows[((size_t)m * 3 + k) * NP + j] = (float)E[(size_t)(3 * m + k) * N + j];
    TMF_CUDA(cudaMalloc(&P->f32_rows, rows.size() * sizeof(float)));
    TMF_CUDA(cudaMemcpy(P->f32_rows, rows.data(), rows.size() * sizeof(float), cudaMemcpyHostToDevice));
    TMF_CUDA(cudaMalloc(&P->f32_geo, sizeof(float) * 8 * P->n_cells));
    total += rows.size() * sizeof(float) + sizeof(float) * 8 * P->n_cells;
    tmf::geo_to_f32_kernel<<<P->n_sm * 8, 256>>>(P->cell_geo, P->f32_geo, 8 * P->n_cells);
    TMF_CUDA(cudaGetLastError());
    P->f32_M = M;
  }

  // face tables -> fragments per (lf, code) in the face frame, face batches
  if (faces) {
    const int N = P->N, QF = P->QF;
    const int NF = (P->degree + 1) * (P->degree + 2) / 2;
    // gather order per local face: the DoFs whose basis function does not vanish
    // on the face (nodal basis: exactly the face's NF nodes), then the rest
    std::vector<int> perm(4 * N);
    for (int lf = 0; lf < 4; ++lf) {
      const double* Fv = d->face_values + (size_t)(lf * 6) * QF * N;
      std::vector<int> on, off;
      for (int j = 0; j < N; ++j) {
        double mx = 0.0;
        for (int q = 0; q < QF; ++q) mx = std::max(mx, std::fabs(Fv[q * N + j]));
        (mx > 1e-10 ? on : off).push_back(j);
      }
      if ((int)on.size() != NF) return bail(fail(TMF_EINVAL, "face tables are not those of a nodal basis"));
      on.insert(on.end(), off.begin(), off.end());
      std::copy(on.begin(), on.end(), perm.begin() + lf * N);
    }
    if ((rc = upload(&P->face_perm, perm.data(), perm.size(), &total))) return bail(rc);
    P->face_perm_h.assign(perm.begin(), perm.end());
    // face engine by default: modal at P2-P4, the point loop at P1 (decided by measurement)
    int fe = P->face_engine;
    if (fe == 0) fe = N >= 10 ? 3 : 1;
    P->face_engine = fe;
    // modal face tables (face engines 2 / 3): every face integrand is a product of two P_p
    // polynomials on the face (values in P_p, derivatives in P_{p-1}), so NF = dim P_p
    // orthonormal modes integrate it exactly:  E'(c, m, j) = sum_q w_q psi_m(q) E(c, q, j), unit
    // weights.  The modes are degree-ordered: psi_0..psi_{MD-1} span P_{p-1} (MD = dim P_{p-1}),
    // the rest complete P_p.  They come from the tables alone (lf 0, code 0; every (lf, code)
    // table is indexed by the same reference-triangle points): pivoted Gram-Schmidt in the
    // w-inner product, first over the tangential derivatives of the face traces (their span is
    // P_{p-1} at the points), then over the traces themselves.  Derivative components then
    // have no coefficient on the modes >= MD, which the split-mode layout (engine 3) leaves out.
    std::vector<double> proj;   // (NF, QF): w_q psi_m(q)
    int QK = QF;
    const int MD = P->degree * (P->degree + 1) / 2;
    if (fe == 3 || fe == 2) {
      const double* Fv0 = d->face_values;
      const double* Fg0 = d->face_grads;
      const double fr0[2][3] = {{-1.0, 1.0, 0.0}, {-1.0, 0.0, 1.0}};   // lf 0 frame tangents (R2-R1, R3-R1)
      std::vector<std::vector<long double>> cand;
      for (int t = 0; t < 2; ++t)
        for (int a = 0; a < NF; ++a) {
          std::vector<long double> v(QF);
          for (int q = 0; q < QF; ++q) {
            long double acc = 0.0L;
            for (int k = 0; k < 3; ++k) acc += (long double)fr0[t][k] * Fg0[(size_t)(3 * q + k) * N + perm[a]];
            v[q] = acc;
          }
          cand.push_back(std::move(v));
        }
      const size_t n_der = cand.size();
      for (int a = 0; a < NF; ++a) {
        std::vector<long double> v(QF);
        for (int q = 0; q < QF; ++q) v[q] = Fv0[(size_t)q * N + perm[a]];
        cand.push_back(std::move(v));
      }
      auto dot = [&](const std::vector<long double>& x, const std::vector<long double>& y) {
        long double acc = 0.0L;
        for (int q = 0; q < QF; ++q) acc += (long double)d->face_weights[q] * x[q] * y[q];
        return acc;
      };
      std::vector<std::vector<long double>> psi;
      auto sweep = [&](size_t c0, size_t c1, int want) {   // greedy: largest residual first
        long double scale0 = 0.0L;
        for (size_t c = c0; c < c1; ++c) scale0 = std::max(scale0, dot(cand[c], cand[c]));
        for (int it = 0; it < want; ++it) {
          size_t best = c0;
          long double nb = -1.0L;
          for (size_t c = c0; c < c1; ++c) {
            const long double nn = dot(cand[c], cand[c]);
            if (nn > nb) nb = nn, best = c;
          }
          if (!(nb > 1e-20L * scale0) || !(nb > 0.0L)) return false;
          std::vector<long double> v = cand[best];
          for (int rep = 0; rep < 2; ++rep)                 // re-orthogonalise against all modes
            for (const auto& ps : psi) {
              const long double c = dot(v, ps);
              for (int q = 0; q < QF; ++q) v[q] -= c * ps[q];
            }
          const long double nv = std::sqrt(dot(v, v));
          for (int q = 0; q < QF; ++q) v[q] /= nv;
          psi.push_back(v);
          for (size_t c = c0; c < cand.size(); ++c) {       // deflate the remaining candidates
            const long double cc = dot(cand[c], v);
            for (int q = 0; q < QF; ++q) cand[c][q] -= cc * v[q];
          }
        }
        long double rest = 0.0L;                            // the span must be exhausted
        for (size_t c = c0; c < c1; ++c) rest = std::max(rest, dot(cand[c], cand[c]));
        return rest <= 1e-22L * std::max(scale0, 1.0L);
      };
      if (!sweep(0, n_der, MD) || !sweep(n_der, cand.size(), NF - MD))
        return bail(fail(TMF_EINVAL, "modal face engine: face traces are not a nodal basis of P_p"));
      proj.assign((size_t)NF * QF, 0.0);
      for (int m = 0; m < NF; ++m)
        for (int q = 0; q < QF; ++q) proj[(size_t)m * QF + q] = (double)((long double)d->face_weights[q] * psi[m][q]);
      QK = NF;
    }
    P->QFk = QK;
    std::vector<double> ones(QK, 1.0);
    std::vector<double> fr, frh;
    double lost = 0.0, kept = 0.0;   // derivative coefficients on the value-only modes (must vanish)
    for (int lf = 0; lf < 4; ++lf) {
      const double R[4][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
      const int fvv[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
      double a[3][3];  // a[i] = frame vector i
      for (int k = 0; k < 3; ++k) {
        a[0][k] = R[fvv[lf][1]][k] - R[fvv[lf][0]][k];
        a[1][k] = R[fvv[lf][2]][k] - R[fvv[lf][0]][k];
        a[2][k] = R[lf][k] - R[fvv[lf][0]][k];
      }
      const int* pm = perm.data() + lf * N;
      for (int code = 0; code < 6; ++code) {
        const double* Fv = d->face_values + (size_t)(lf * 6 + code) * QF * N;
        const double* Fg = d->face_grads + (size_t)(lf * 6 + code) * 3 * QF * N;
        auto Ept = [&](int c, int q, int j) {   // component c at face point q, gather position j
          const int jj = pm[j];
          if (c == 0) return Fv[q * N + jj];
          const double* av = a[c - 1];
          return av[0] * Fg[(3 * q) * N + jj] + av[1] * Fg[(3 * q + 1) * N + jj] + av[2] * Fg[(3 * q + 2) * N + jj];
        };
        if (fe == 3 || fe == 2) {
          std::vector<double> Em((size_t)4 * NF * N);   // modal table (c, m, j)
          for (int c = 0; c < 4; ++c)
            for (int m = 0; m < NF; ++m)
              for (int j = 0; j < N; ++j) {
                long double acc = 0.0L;
                for (int q = 0; q < QF; ++q) acc += (long double)proj[(size_t)m * QF + q] * Ept(c, q, j);
                Em[((size_t)c * NF + m) * N + j] = (double)acc;
                if (c > 0) (m >= MD ? lost : kept) = std::max(m >= MD ? lost : kept, std::fabs((double)acc));
              }
          auto Emod = [&](int c, int m, int j) { return Em[((size_t)c * NF + m) * N + j]; };
          build_face_fragments(N, NF, QK, Emod, ones.data(), fr);
          if (fe == 3) {
            if (N == 4) build_face_fragments_hier<4>(Emod, frh);
            else if (N == 10) build_face_fragments_hier<10>(Emod, frh);
            else if (N == 20) build_face_fragments_hier<20>(Emod, frh);
            else if (N == 35) build_face_fragments_hier<35>(Emod, frh);
            else return bail(fail(TMF_EINVAL, "modal face engine: unsupported n_dofs_per_cell"));
          }
        } else {
          build_face_fragments(N, NF, QF, Ept, d->face_weights, fr);
        }
      }
    }
    if (fe == 3 && !(lost <= 1e-11 * std::max(kept, 1.0)))
      return bail(fail(TMF_EINVAL, "modal face engine: derivative tables are not of degree p-1 on the face"));
    tmf::FaceLaunchInfo fi;
    bool ok = true;
    tmf::FaceArgs dummy{};
    dummy.nc = P->nc;
    TMF_CUDA(tmf::launch_face(N, QK, false, dummy, P->n_sm, 0, &fi, &ok));
    if (!ok) return bail(fail(TMF_EINVAL, "unsupported (n_dofs_per_cell, n_qf) = (" +
                                              std::to_string(N) + ", " + std::to_string(QF) + ")"));
    if ((int64_t)fr.size() != 24LL * fi.nfrag * 32) return bail(fail(TMF_EINVAL, "internal: face fragments"));
    if ((rc = upload(&P->face_frags, fr.data(), fr.size(), &total))) return bail(rc);
    const int dmma_boundary = fi.dmma_per_batch / 2;
    if (fe == 3) {   // interior faces: the split-mode layout (the boundary kernel keeps the flat one)
      dummy.hier = 1;
      TMF_CUDA(tmf::launch_face(N, QK, false, dummy, P->n_sm, 0, &fi, &ok));
      if (!ok || (int64_t)frh.size() != 24LL * fi.nfrag * 32)
        return bail(fail(TMF_EINVAL, "internal: split-mode face fragments"));
      if ((rc = upload(&P->face_frags_h, frh.data(), frh.size(), &total))) return bail(rc);
    }
    const int chunk = ((d->flags >> 8) & 0xF) ? 8 * ((d->flags >> 8) & 0xF) : fi.chunk;
    if ((rc = build_face_batches(P, d, chunk, &total))) return bail(rc);
    // per-face geometry, computed once on the device (64 B per face slot)
    for (int bnd = 0; bnd < 2; ++bnd) {
      const int64_t slots = (bnd ? P->n_bf_batches : P->n_if_batches) * 8;
      if (!slots) continue;
      double** g = bnd ? &P->bf_geo : &P->if_geo;
      TMF_CUDA(cudaMalloc(g, sizeof(double) * 8 * slots));
      total += sizeof(double) * 8 * slots;
      TMF_CUDA(tmf::launch_face_geometry(bnd != 0, P->face_geo_args(bnd != 0), P->n_sm, 0));
    }
    P->info.n_face_batches = (int32_t)(P->n_if_batches + P->n_bf_batches);
    P->info.face_engine = P->face_engine;
    P->info.flops_issued += (double)P->nc * (P->n_if_batches * (double)fi.dmma_per_batch +
                                             P->n_bf_batches * (double)dmma_boundary) * 512.0;
  }

  // algorithmic flops / bytes (reference counters)
  {
    const double nd = P->N, nq = P->Q, nqf = P->QF, nce = (double)P->n_cells;
    double n_scatter = nce * nd;
    if (!dg && d->dirichlet_mask) {
      int64_t masked = 0;
      for (int64_t i = 0; i < (int64_t)d->n_cells * P->N; ++i) masked += d->dirichlet_mask[d->cell_dofs[i]] ? 1 : 0;
      n_scatter -= (double)masked;
    }
    double f = nce * (12.0 * nq * nd + 33.0 * nq) + n_scatter;
    if (P->mass) f += nce * (4.0 * nq * nd + 5.0 * nq + nd);
    int64_t nbf_dir = 0;
    if (faces) {
      for (int64_t i = 0; i < d->n_boundary_faces; ++i) nbf_dir += (d->boundary_dirichlet && d->boundary_dirichlet[i]) ? 1 : 0;
      f += (double)d->n_interior_faces * (32.0 * nqf * nd + 26.0 * nqf) +
           (double)nbf_dir * (16.0 * nqf * nd + 13.0 * nqf);
    }
    P->info.flops_alg = f * P->nc;
    // the same apply's useful flops in the algorithms the engines run: the reference tensor
    // form replaces the cell term's 12 n_q N + 33 n_q by 12 N^2 + 12 N (+ 2 N^2 + 2 N mass)
    double fe = f;
    if (P->info.cell_engine == 3) {
      fe -= nce * (12.0 * nq * nd + 33.0 * nq);
      fe += nce * (12.0 * nd * nd + 12.0 * nd);
      if (P->mass) fe += nce * (2.0 * nd * nd + 2.0 * nd) - nce * (4.0 * nq * nd + 5.0 * nq + nd);
    } else if (P->info.cell_engine == 4 || P->info.cell_engine == 5) {
      // the point loop on M unit-weight modes: 12 M N (both GEMMs) + 18 M (G action)
      const double M = P->degree * (P->degree + 1) * (P->degree + 2) / 6;
      fe -= nce * (12.0 * nq * nd + 33.0 * nq);
      fe += nce * (12.0 * M * nd + 18.0 * M);
      // the mass term as one N x N GEMM and a row scaling
      if (P->mass) fe += nce * (2.0 * nd * nd + 2.0 * nd) - nce * (4.0 * nq * nd + 5.0 * nq + nd);
    }
    if (faces && (P->face_engine == 3 || P->face_engine == 2)) {
      // modal face tables: the point loop on NF unit-weight modes instead of n_qf points
      const double NFm = P->QFk;
      fe -= (double)d->n_interior_faces * (32.0 * nqf * nd + 26.0 * nqf) + (double)nbf_dir * (16.0 * nqf * nd + 13.0 * nqf);
      double fi_face = 32.0 * NFm * nd + 26.0 * NFm;
      if (P->face_engine == 3) {
        // split-mode layout: values and tangential derivatives on the NF face DoFs only, the
        // derivatives on MD = dim P_{p-1} modes, the transversal one on all DoFs; two GEMMs on
        // two sides (x 8 flops per table entry), 26 flops per full mode, 6 per value-only mode
        const double MDm = P->degree * (P->degree + 1) / 2;
        fi_face = 8.0 * (NFm * NFm + 2.0 * MDm * NFm + MDm * nd) + 26.0 * MDm + 6.0 * (NFm - MDm);
      }
      fe += (double)d->n_interior_faces * fi_face + (double)nbf_dir * (16.0 * NFm * nd + 13.0 * NFm);
    }
    P->info.flops_engine = fe * P->nc;
    double b = 16.0 * (double)P->n_global + 24.0 * (double)P->n_verts;
    if (!dg)
      b += 4.0 * nd * nce;
    else
      b += 16.0 * nce + 8.0 * (double)d->n_interior_faces + 4.0 * (double)d->n_boundary_faces;
    if (d->kappa) b += 8.0 * nce;
    P->info.bytes_alg = b;
  }
  P->info.n_global_dofs = P->n_global;
  P->info.kernels_per_apply = 1 + (faces ? ((P->n_if_batches ? 1 : 0) + (P->n_bf_batches ? 1 : 0)) : 0) +
                              ((!dg && P->n_fix) ? 1 : 0) + ((!dg && pdl_enabled()) ? 1 : 0);   // + the y clear kernel
  P->dev_bytes = total;
  P->info.device_bytes = (int64_t)total;
  TMF_CUDA(cudaDeviceSynchronize());
  *out = P;
  return TMF_OK;
}

int tmf_plan_set_peers(tmf_plan* P, int32_t n_ranks, const uint64_t* peer_u, const uint64_t* peer_y,
                       int32_t self_rank, int64_t n_own, int64_t n_ghost, const int32_t* ghost_rank,
                       const int32_t* ghost_index, int64_t n_peer_free_cells) {
  if (!P) return fail(TMF_EINVAL, "null plan");
  if (P->cell_perm)
    return fail(TMF_EINVAL, "peers need the caller's cell order (OperatorConfig(cell_order='input'))");
  TMF_CUDA(cudaSetDevice(P->dev));
  for (void* q : {(void*)P->peer_u_tab, (void*)P->peer_y_tab, (void*)P->ghost_rank, (void*)P->ghost_index})
    if (q) cudaFree(q);
  P->peer_u_tab = nullptr;
  P->peer_y_tab = nullptr;
  P->ghost_rank = nullptr;
  P->ghost_index = nullptr;
  P->peer = tmf::PeerArgs{};
  P->peer_self_u = nullptr;
  P->peer_self_y = nullptr;
  P->n_peer_free = 0;
  if (n_ranks == 0) return TMF_OK;
  if (n_ranks < 0 || !peer_u || self_rank < 0 || self_rank >= n_ranks || n_own < 0 || n_ghost < 0 ||
      (n_ghost && (!ghost_rank || !ghost_index)) || n_peer_free_cells < 0 || n_peer_free_cells > P->n_cells)
    return fail(TMF_EINVAL, "bad peer description");
  if (!P->dg && !peer_y) return fail(TMF_EINVAL, "a CG plan needs the peers' y buffers (ghost RED)");
  const int64_t n_entries = P->dg ? P->n_cells : P->n_scalar;
  if (n_own + n_ghost != n_entries)
    return fail(TMF_EINVAL, "n_own + n_ghost must equal the plan's local " +
                                std::string(P->dg ? "cells" : "DoFs"));
  for (int64_t i = 0; i < n_ghost; ++i)
    if (ghost_rank[i] < 0 || ghost_rank[i] >= n_ranks || ghost_rank[i] == self_rank || ghost_index[i] < 0)
      return fail(TMF_EINVAL, "ghost owner rank / index out of range");
  size_t total = 0;
  int rc;
  if ((rc = upload(reinterpret_cast<uint64_t**>(&P->peer_u_tab), peer_u, (size_t)n_ranks, &total))) return rc;
  if (peer_y && (rc = upload(reinterpret_cast<uint64_t**>(&P->peer_y_tab), peer_y, (size_t)n_ranks, &total)))
    return rc;
  if (n_ghost) {
    if ((rc = upload(&P->ghost_rank, ghost_rank, (size_t)n_ghost, &total))) return rc;
    if ((rc = upload(&P->ghost_index, ghost_index, (size_t)n_ghost, &total))) return rc;
  }
  P->peer.u = P->peer_u_tab;
  P->peer.y = peer_y ? P->peer_y_tab : nullptr;
  P->peer.rank = P->ghost_rank;
  P->peer.idx = P->ghost_index;
  P->peer.n_own = n_own;
  P->peer_self_u = reinterpret_cast<const double*>(peer_u[self_rank]);
  P->peer_self_y = peer_y ? reinterpret_cast<double*>(peer_y[self_rank]) : nullptr;
  P->n_peer_free = P->dg ? 0 : n_peer_free_cells;
  if (n_ghost == 0) {   // nothing lives elsewhere: the plain kernels (buffers stay registered)
    P->peer.u = nullptr;
    P->peer.y = nullptr;
  }
  return TMF_OK;
}

int tmf_alloc(int64_t bytes, int32_t device, void** out) {
  if (!out || bytes < 0) return fail(TMF_EINVAL, "bad argument");
  *out = nullptr;
  TMF_CUDA(cudaSetDevice(device));
  TMF_CUDA(cudaMalloc(out, bytes > 0 ? (size_t)bytes : 1));
  return TMF_OK;
}

int tmf_free(void* p) {
  if (p) TMF_CUDA(cudaFree(p));
  return TMF_OK;
}

int tmf_ipc_get_handle(const void* dev_ptr, uint8_t handle[64]) {
  if (!dev_ptr || !handle) return fail(TMF_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  TMF_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(handle, &h, 64);
  return TMF_OK;
}

int tmf_ipc_open_handle(const uint8_t handle[64], int32_t device, void** dev_ptr) {
  if (!handle || !dev_ptr) return fail(TMF_EINVAL, "null argument");
  *dev_ptr = nullptr;
  TMF_CUDA(cudaSetDevice(device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, 64);
  TMF_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return TMF_OK;
}

int tmf_ipc_close_handle(void* dev_ptr) {
  if (dev_ptr) TMF_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return TMF_OK;
}

int tmf_plan_destroy(tmf_plan* plan) {
  if (!plan) return TMF_OK;
  cudaSetDevice(plan->dev);
  delete plan;
  return TMF_OK;
}

int tmf_debug_chunk_walk(int64_t n_work, int64_t grid, int64_t block, int blocked, int run, int64_t* out,
                         int64_t cap, int64_t* n_out) {
  if (n_work < 0 || grid < 1 || block < 0 || block >= grid || !out || !n_out) return fail(TMF_EINVAL, "bad argument");
  const tmf::ChunkWalk walk(n_work, blocked != 0, run, grid, block);
  int64_t n = 0;
  for (int64_t i = 0; i < walk.nit; ++i) {
    const int64_t w = walk.at(i);
    if (w >= n_work) continue;
    if (n >= cap) return fail(TMF_EINVAL, "output capacity");
    out[n++] = w;
  }
  *n_out = n;
  return TMF_OK;
}

int tmf_debug_poke_dof(tmf_plan* P, int64_t slot, int32_t value) {
#ifdef TMF_DEBUG_CHECKS
  if (!P || P->dg || slot < 0 || slot >= P->n_cells * P->N) return fail(TMF_EINVAL, "bad poke");
  TMF_CUDA(cudaSetDevice(P->dev));
  TMF_CUDA(cudaMemcpy(P->dofs + slot, &value, sizeof(int32_t), cudaMemcpyHostToDevice));
  // the block-assembly tables are derived at plan creation: take the tile kernel from now on
  P->blk_B = 0;
  return TMF_OK;
#else
  (void)P;
  (void)slot;
  (void)value;
  return fail(TMF_EINVAL, "tmf_debug_poke_dof needs the TMF_DEBUG_CHECKS build (libtetmf_b200_debug.so)");
#endif
}

int tmf_plan_get_info(const tmf_plan* plan, tmf_plan_info* info) {
  if (!plan || !info) return fail(TMF_EINVAL, "null plan/info");
  *info = plan->info;
  return TMF_OK;
}

int tmf_apply(tmf_plan* P, const double* u, double* y, void* stream) {
  if (!P || !u || !y) return fail(TMF_EINVAL, "null argument");
  if (u == y) return fail(TMF_EINVAL, "u and y must not alias");
  if (P->peer.u && !P->dg)
    return fail(TMF_EINVAL, "a CG plan with peers needs tmf_apply_stages with cross-rank barriers "
                            "(ZERO | barrier | CELLS | FIXUP | barrier)");
  if (P->peer.u && u != P->peer_self_u) return fail(TMF_EINVAL, "u must be this rank's registered buffer");
  TMF_CUDA(cudaSetDevice(P->dev));
  return launch_apply(P, u, y, (cudaStream_t)stream, nullptr);
}

int tmf_apply_f32(tmf_plan* P, const float* u, float* y, void* stream) {
  if (!P || !u || !y) return fail(TMF_EINVAL, "null argument");
  if (u == y) return fail(TMF_EINVAL, "u and y must not alias");
  if (!P->f32_rows) return fail(TMF_EINVAL, "plan was created without the fp32 mirror (flags bit 20)");
  TMF_CUDA(cudaSetDevice(P->dev));
  const cudaStream_t st = (cudaStream_t)stream;
  TMF_CUDA(cudaMemsetAsync(y, 0, sizeof(float) * P->n_global, st));
  const int block = 256;
  int64_t grid = (P->n_cells + block - 1) / block;
  if (grid > (int64_t)P->n_sm * 8) grid = (int64_t)P->n_sm * 8;
  const float4* g4 = reinterpret_cast<const float4*>(P->f32_geo);
  switch (P->N) {
    case 4: tmf::cell_f32_kernel<4, 1, block><<<(unsigned)grid, block, 0, st>>>(u, y, P->dofs, g4, P->f32_rows, P->n_cells); break;
    case 10: tmf::cell_f32_kernel<10, 4, block><<<(unsigned)grid, block, 0, st>>>(u, y, P->dofs, g4, P->f32_rows, P->n_cells); break;
    case 20: tmf::cell_f32_kernel<20, 10, block><<<(unsigned)grid, block, 0, st>>>(u, y, P->dofs, g4, P->f32_rows, P->n_cells); break;
    case 35: tmf::cell_f32_kernel<35, 20, block><<<(unsigned)grid, block, 0, st>>>(u, y, P->dofs, g4, P->f32_rows, P->n_cells); break;
    default: return fail(TMF_EINVAL, "fp32 mirror: unsupported degree");
  }
  TMF_CUDA(cudaGetLastError());
  if (P->n_fix) {
    tmf::fixup_f32_kernel<<<P->n_sm * 4, 256, 0, st>>>(u, y, P->fix_list, P->n_fix);
    TMF_CUDA(cudaGetLastError());
  }
  return TMF_OK;
}

// Host-buffer applies stage u / y in per-plan device buffers.  ev_stage marks the end of the
// plan's last staged apply (its download): every staged apply waits for it before it uploads
// into stage_u (an earlier kernel may still read it) and records it after its download, so two
// staged applies of one plan on any streams (or twice in one pipeline call) are ordered.
static int ensure_staging(tmf_plan* P) {
  if (P->peer.u)
    return fail(TMF_EINVAL, "a plan with peers applies on its registered buffers (tmf_apply / "
                            "tmf_apply_stages), not through host staging");
  if (!P->stage_u) {
    const size_t bytes = sizeof(double) * P->n_global;
    TMF_CUDA(cudaMalloc(&P->stage_u, bytes));
    TMF_CUDA(cudaMalloc(&P->stage_y, bytes));
    TMF_CUDA(cudaEventCreateWithFlags(&P->ev_stage, cudaEventDisableTiming));
  }
  return TMF_OK;
}

int tmf_apply_host(tmf_plan* P, const double* u_host, double* y_host) {
  if (!P || !u_host || !y_host) return fail(TMF_EINVAL, "null argument");
  TMF_CUDA(cudaSetDevice(P->dev));
  if (int rc = ensure_staging(P)) return rc;
  const size_t bytes = sizeof(double) * P->n_global;
  TMF_CUDA(cudaStreamWaitEvent(0, P->ev_stage, 0));
  TMF_CUDA(cudaMemcpyAsync(P->stage_u, u_host, bytes, cudaMemcpyHostToDevice, 0));
  int rc = launch_apply(P, P->stage_u, P->stage_y, 0, nullptr);
  if (rc) return rc;
  TMF_CUDA(cudaMemcpyAsync(y_host, P->stage_y, bytes, cudaMemcpyDeviceToHost, 0));
  TMF_CUDA(cudaEventRecord(P->ev_stage, 0));
  TMF_CUDA(cudaStreamSynchronize(0));
  return TMF_OK;
}

int tmf_apply_host_async(tmf_plan* P, const double* u_host, double* y_host, void* stream) {
  if (!P || !u_host || !y_host) return fail(TMF_EINVAL, "null argument");
  TMF_CUDA(cudaSetDevice(P->dev));
  if (int rc = ensure_staging(P)) return rc;
  const size_t bytes = sizeof(double) * P->n_global;
  cudaStream_t st = (cudaStream_t)stream;
  TMF_CUDA(cudaStreamWaitEvent(st, P->ev_stage, 0));
  TMF_CUDA(cudaMemcpyAsync(P->stage_u, u_host, bytes, cudaMemcpyHostToDevice, st));
  int rc = launch_apply(P, P->stage_u, P->stage_y, st, nullptr);
  if (rc) return rc;
  TMF_CUDA(cudaMemcpyAsync(y_host, P->stage_y, bytes, cudaMemcpyDeviceToHost, st));
  TMF_CUDA(cudaEventRecord(P->ev_stage, st));
  return TMF_OK;
}

// Several plans' host applies as one three-stage pipeline: every upload on one copy stream
// in the caller's order, the kernels on one compute stream (each waits for its own upload),
// every download on a second copy stream (each waits for its own kernels).  Per-plan
// streams would let the copy engine interleave all uploads, so the first kernel (and the
// first download) would wait for most of the uploads instead of one.  The pipeline streams
// are shared per device, so concurrent callers are serialised for the (short) enqueue.
namespace {
struct HostPipe {
  cudaStream_t up = nullptr, comp = nullptr, down = nullptr;
};
HostPipe g_pipe[64];
std::mutex g_pipe_mu;
}  // namespace

int tmf_apply_host_multi(tmf_plan* const* plans, const double* const* u_hosts, double* const* y_hosts, int n,
                         void* stream) {
  if (n < 0 || (n > 0 && (!plans || !u_hosts || !y_hosts))) return fail(TMF_EINVAL, "null argument");
  if (n == 0) return TMF_OK;
  for (int i = 0; i < n; ++i) {
    if (!plans[i] || !u_hosts[i] || !y_hosts[i]) return fail(TMF_EINVAL, "null plan or host buffer");
    if (plans[i]->dev != plans[0]->dev) return fail(TMF_EINVAL, "plans on different devices");
    if (plans[i]->peer.u) return fail(TMF_EINVAL, "a plan with peers cannot take host buffers");
  }
  const int dev = plans[0]->dev;
  if (dev < 0 || dev >= 64) return fail(TMF_EINVAL, "device index out of range");
  TMF_CUDA(cudaSetDevice(dev));
  std::lock_guard<std::mutex> lk(g_pipe_mu);
  HostPipe& pp = g_pipe[dev];
  if (!pp.up) {
    TMF_CUDA(cudaStreamCreateWithFlags(&pp.up, cudaStreamNonBlocking));
    TMF_CUDA(cudaStreamCreateWithFlags(&pp.comp, cudaStreamNonBlocking));
    TMF_CUDA(cudaStreamCreateWithFlags(&pp.down, cudaStreamNonBlocking));
  }
  for (int i = 0; i < n; ++i)
    if (int rc = ensure_staging(plans[i])) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  auto link = [&](cudaStream_t from, cudaStream_t to) -> int {
    cudaEvent_t ev;
    TMF_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TMF_CUDA(cudaEventRecord(ev, from));
    TMF_CUDA(cudaStreamWaitEvent(to, ev, 0));
    TMF_CUDA(cudaEventDestroy(ev));  // released once the wait has been satisfied
    return TMF_OK;
  };
  // the caller's prior work on `stream` (e.g. writes into the host buffers' sources) comes first
  int rc = 0;
  if ((rc = link(st, pp.up)) || (rc = link(st, pp.comp)) || (rc = link(st, pp.down))) return rc;
  for (int i = 0; i < n && !rc; ++i) {
    tmf_plan* P = plans[i];
    const size_t bytes = sizeof(double) * P->n_global;
    // the plan's previous staged apply (an earlier list entry, or another call) has downloaded
    if ((rc = cudaStreamWaitEvent(pp.up, P->ev_stage, 0) == cudaSuccess ? 0 : fail(TMF_ECUDA, "event wait")))
      break;
    if (cudaMemcpyAsync(P->stage_u, u_hosts[i], bytes, cudaMemcpyHostToDevice, pp.up) != cudaSuccess) {
      rc = fail(TMF_ECUDA, "upload failed");
      break;
    }
    if ((rc = link(pp.up, pp.comp))) break;
    if ((rc = launch_apply(P, P->stage_u, P->stage_y, pp.comp, nullptr))) break;
    if ((rc = link(pp.comp, pp.down))) break;
    if (cudaMemcpyAsync(y_hosts[i], P->stage_y, bytes, cudaMemcpyDeviceToHost, pp.down) != cudaSuccess ||
        cudaEventRecord(P->ev_stage, pp.down) != cudaSuccess) {
      rc = fail(TMF_ECUDA, "download failed");
      break;
    }
  }
  // `stream` reaches the end of the pipeline only when every download has landed -- also
  // after an error, so the caller can tell when the copies touching its buffers are done
  int rl = 0;
  if ((rl = link(pp.down, st)) || (rl = link(pp.comp, st)) || (rl = link(pp.up, st))) return rc ? rc : rl;
  return rc;
}

int tmf_apply_timed(tmf_plan* P, const double* u, double* y, void* stream, int reps, double* out_ms,
                    int n_out) {
  if (!P || !u || !y || !out_ms || reps < 1) return fail(TMF_EINVAL, "bad argument");
  TMF_CUDA(cudaSetDevice(P->dev));
  cudaStream_t st = (cudaStream_t)stream;
  cudaEvent_t ev[4];
  for (auto& e : ev) TMF_CUDA(cudaEventCreate(&e));
  double acc[4] = {0, 0, 0, 0};
  // which stage events launch_apply records (see there): ev[0] and ev[3] always
  const bool fix = !P->dg && P->n_fix;
  const bool e1 = P->faces || fix, e2 = P->faces && fix;
  for (int r = 0; r < reps; ++r) {
    int rc = launch_apply(P, u, y, st, ev);
    if (rc) return rc;
    TMF_CUDA(cudaEventSynchronize(ev[3]));
    float t = 0, a = 0, b = 0, c = 0;
    cudaEventElapsedTime(&t, ev[0], ev[3]);
    // cell | faces | fixup; a stage without its closing event ends at ev[3]
    const cudaEvent_t end_cell = e1 ? ev[1] : ev[3];
    cudaEventElapsedTime(&a, ev[0], end_cell);
    if (P->faces) cudaEventElapsedTime(&b, end_cell, e2 ? ev[2] : ev[3]);
    if (fix) cudaEventElapsedTime(&c, e2 ? ev[2] : end_cell, ev[3]);
    acc[0] += t;
    acc[1] += a;
    acc[2] += b;
    acc[3] += c;
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int i = 0; i < n_out && i < 4; ++i) out_ms[i] = acc[i] / reps;
  return TMF_OK;
}

int tmf_diagonal(tmf_plan* P, double* diag, void* stream) {
  if (!P || !diag) return fail(TMF_EINVAL, "null argument");
  if (P->dg) return fail(TMF_EINVAL, "matrix-free diagonal is implemented for the CG operator");
  TMF_CUDA(cudaSetDevice(P->dev));
  cudaStream_t st = (cudaStream_t)stream;
  TMF_CUDA(cudaMemsetAsync(diag, 0, sizeof(double) * P->n_global, st));
  tmf::DiagArgs a{diag, P->dofs, P->cells, P->verts, P->diag_S, P->n_cells, P->N, P->nc, P->cell_geo};
  tmf::diag_kernel<<<P->n_sm * 8, 256, 0, st>>>(a);
  TMF_CUDA(cudaGetLastError());
  if (P->n_fix) {
    tmf::set_list_kernel<<<P->n_sm * 4, 256, 0, st>>>(diag, P->fix_list, P->n_fix, 1.0);
    TMF_CUDA(cudaGetLastError());
  }
  return TMF_OK;
}

int tmf_pcg(tmf_plan* P, const double* b, double* x, int iters, double* res_norms, void* stream) {
  if (!P || !b || !x || iters < 0) return fail(TMF_EINVAL, "bad argument");
  if (P->dg) return fail(TMF_EINVAL, "PCG is implemented for the CG operator");
  if (P->peer.u)
    return fail(TMF_EINVAL, "tmf_pcg is the single-GPU solver; a plan with peers needs the multi-rank "
                            "loop (tmf_apply_stages + tmf_pcg_* with cross-rank reductions)");
  TMF_CUDA(cudaSetDevice(P->dev));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = P->n_global;
  if (!P->pcg_buf) TMF_CUDA(cudaMalloc(&P->pcg_buf, sizeof(double) * (5 * n)));
  double *r = P->pcg_buf, *z = r + n, *p = z + n, *q = p + n, *dg = q + n;
  double* sc = nullptr;  // rz[iters+1], pq[iters+1], rr[iters+1]
  TMF_CUDA(cudaMallocAsync(&sc, sizeof(double) * 3 * (iters + 1), st));
  double *rz = sc, *pq = sc + (iters + 1), *rr = sc + 2 * (iters + 1);
  TMF_CUDA(cudaMemsetAsync(sc, 0, sizeof(double) * 3 * (iters + 1), st));
  int rc = tmf_diagonal(P, dg, stream);
  if (rc) return rc;
  const int grid = P->n_sm * 4, blk = 512;
  // fused iteration when the element energies are available (tensor cell engine, plain
  // single-GPU plan): apply(+p.Ap) -> residual -> step (x, p, q = 0)
  const bool fused = P->info.cell_engine >= 3 && !P->peer.u && !P->dg;
  if (fused) {
    tmf::pcg_init_fused_kernel<<<grid, blk, 0, st>>>(b, dg, x, r, z, p, q, n, rz, rr);
    TMF_CUDA(cudaGetLastError());
    for (int k = 0; k < iters; ++k) {
      if ((rc = launch_apply(P, p, q, st, nullptr, true, pq + k))) return rc;
      tmf::pcg_residual_kernel<<<grid, blk, 0, st>>>(q, dg, r, z, n, rz + k, pq + k, rz + k + 1, rr + k + 1);
      tmf::pcg_step_kernel<<<grid, blk, 0, st>>>(z, p, x, q, n, rz + k, pq + k, rz + k + 1);
    }
  } else {
  tmf::pcg_init_kernel<<<grid, blk, 0, st>>>(b, dg, x, r, z, p, n, rz, rr);
  TMF_CUDA(cudaGetLastError());
  for (int k = 0; k < iters; ++k) {
    if ((rc = launch_apply(P, p, q, st, nullptr))) return rc;
    tmf::dot_kernel<<<grid, blk, 0, st>>>(p, q, n, pq + k);
    tmf::pcg_update_kernel<<<grid, blk, 0, st>>>(p, q, dg, x, r, z, n, rz + k, pq + k, rz + k + 1, rr + k + 1);
    tmf::pcg_direction_kernel<<<grid, blk, 0, st>>>(z, p, n, rz + k, rz + k + 1);
  }
  }
  TMF_CUDA(cudaGetLastError());
  if (res_norms) {
    std::vector<double> h(iters + 1);
    TMF_CUDA(cudaMemcpyAsync(h.data(), rr, sizeof(double) * (iters + 1), cudaMemcpyDeviceToHost, st));
    TMF_CUDA(cudaStreamSynchronize(st));
    for (int k = 0; k <= iters; ++k) res_norms[k] = std::sqrt(h[k]);
  }
  TMF_CUDA(cudaFreeAsync(sc, st));
  return TMF_OK;
}

// ---- fused PCG vector kernels (device pointers; scalars are device doubles) --
int tmf_vec_dot(const double* a, const double* b, int64_t n, double* out, void* stream) {
  if (!a || !b || !out || n < 0) return fail(TMF_EINVAL, "bad argument");
  int dev = 0, sms = 0;
  TMF_CUDA(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  tmf::dot_kernel<<<sms * 4, 512, 0, (cudaStream_t)stream>>>(a, b, n, out);
  TMF_CUDA(cudaGetLastError());
  return TMF_OK;
}

int tmf_pcg_init(const double* b, const double* d, double* x, double* r, double* z, double* p, int64_t n,
                 double* rz, double* rr, void* stream) {
  if (!b || !d || !x || !r || !z || !p || !rz || !rr || n < 0) return fail(TMF_EINVAL, "bad argument");
  int dev = 0, sms = 0;
  TMF_CUDA(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  tmf::pcg_init_kernel<<<sms * 4, 512, 0, (cudaStream_t)stream>>>(b, d, x, r, z, p, n, rz, rr);
  TMF_CUDA(cudaGetLastError());
  return TMF_OK;
}

int tmf_pcg_update(const double* p, const double* q, const double* d, double* x, double* r, double* z,
                   int64_t n, const double* rz_k, const double* pq_k, double* rz_next, double* rr_next,
                   void* stream) {
  if (!p || !q || !d || !x || !r || !z || n < 0) return fail(TMF_EINVAL, "bad argument");
  int dev = 0, sms = 0;
  TMF_CUDA(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  tmf::pcg_update_kernel<<<sms * 4, 512, 0, (cudaStream_t)stream>>>(p, q, d, x, r, z, n, rz_k, pq_k, rz_next,
                                                                      rr_next);
  TMF_CUDA(cudaGetLastError());
  return TMF_OK;
}

int tmf_pcg_direction(const double* z, double* p, int64_t n, const double* rz_k, const double* rz_next,
                      void* stream) {
  if (!z || !p || n < 0) return fail(TMF_EINVAL, "bad argument");
  int dev = 0, sms = 0;
  TMF_CUDA(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  tmf::pcg_direction_kernel<<<sms * 4, 512, 0, (cudaStream_t)stream>>>(z, p, n, rz_k, rz_next);
  TMF_CUDA(cudaGetLastError());
  return TMF_OK;
}

}  // extern "C"
