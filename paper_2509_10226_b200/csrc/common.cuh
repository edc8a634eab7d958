// Shared device helpers for the tetmf_b200 kernels (sm_100a, FP64).
//
// FP64 tensor-core tile: mma.sync m8n8k4 .f64 (SASS DMMA.8x8x4), measured at
// 37.1 TFLOP/s on B200 vs 34 TFLOP/s for register DFMA (tools/microbench,
// profiles/r01_fp64_peak.json).  Fragment ownership (PTX ISA, m8n8k4 .f64):
//   A (8x4, row):  lane holds A[lane>>2][lane&3]
//   B (4x8, col):  lane holds B[lane&3][lane>>2]
//   C (8x8):       lane holds C[lane>>2][2*(lane&3) + {0,1}]
#pragma once
#include <cstdint>

namespace tmf {

// Debug build (-DTMF_DEBUG_CHECKS, libtetmf_b200_debug.so): the kernels test every global
// index they derive (gathered / scattered DoFs, cells, face DoF positions, block-local
// indices and slot lists) against the plan's sizes and OR a code into a device flag that
// the C-ABI reads after each apply -- the memcheck substitute on this pool, where
// compute-sanitizer is closed.  Release builds: the fields and checks do not exist (same
// SASS).
#ifdef TMF_DEBUG_CHECKS
#define TMF_DBG_FIELDS \
  int64_t dbg_n_dofs = 0;  /* vector entries (global / local layout) */ \
  int64_t dbg_n_cells = 0; \
  int* dbg_flag = nullptr;
#define TMF_CHECK(args, cond, code)                                       \
  do {                                                                    \
    if (!(cond) && (args).dbg_flag != nullptr) atomicOr((args).dbg_flag, (code)); \
  } while (0)
#else
#define TMF_DBG_FIELDS
#define TMF_CHECK(args, cond, code) \
  do {                              \
  } while (0)
#endif
// Programmatic dependent launch (launch_apply): the CG apply clears y with zero_y_kernel, which
// lets its dependents start at once; the cell kernel, launched with programmatic stream
// serialization, stages its tables and issues its first index / gather loads meanwhile and
// waits here -- before its first RED into y -- for the clear to complete and be visible.
// Without the launch attribute the wait returns immediately.
__device__ __forceinline__ void pdl_wait_prior_grid() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_release_dependents() { asm volatile("griddepcontrol.launch_dependents;"); }

enum : int {
  TMF_DBG_DOF = 1,        // gathered / scattered vector index out of range
  TMF_DBG_CELL = 2,       // cell index out of range
  TMF_DBG_PERM = 4,       // face gather position out of range
  TMF_DBG_LOCAL = 8,      // block-local DoF index >= the block's unique DoFs
  TMF_DBG_SLOT = 16,      // block slot list / offsets inconsistent
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Multi-GPU without a halo exchange: entries of the rank-local layout at or beyond
// n_own (ghost DoFs for CG, ghost cells for DG) live on their owner rank; ghost
// entry e is element idx[e] of owner rank[e]'s local vector, reached through the
// owner's mapped device pointers u[rank] / y[rank] (NVLink peer memory, or this
// device's own buffers when ranks are emulated on one GPU).  The gather is a peer
// load, the CG scatter a peer RED, fused into the cell / face kernels.
struct PeerArgs {
  const double* const* __restrict__ u = nullptr;   // nullptr: off
  double* const* __restrict__ y = nullptr;
  const int* __restrict__ rank = nullptr;
  const int* __restrict__ idx = nullptr;
  int64_t n_own = 0;
};

__device__ __forceinline__ const double* peer_src(const PeerArgs& p, const double* u, int64_t e, int nc,
                                                  int comp) {
  if (p.u != nullptr && e >= p.n_own) {
    const int64_t g = e - p.n_own;
    return p.u[__ldg(p.rank + g)] + (int64_t)__ldg(p.idx + g) * nc + comp;
  }
  return u + e * nc + comp;
}
__device__ __forceinline__ double* peer_dst(const PeerArgs& p, double* y, int64_t e, int nc, int comp) {
  if (p.y != nullptr && e >= p.n_own) {
    const int64_t g = e - p.n_own;
    return p.y[__ldg(p.rank + g)] + (int64_t)__ldg(p.idx + g) * nc + comp;
  }
  return y + e * nc + comp;
}

// Scatter-add into a (possibly peer-mapped) y entry.  The destination pointer comes out of
// a table, so atomicAdd compiles to the GENERIC returning atomic (ATOM.E.ADD.F64 plus the
// shared-memory CAS fallback, cuobjdump) and the warp waits for the old value; the address
// is always global memory, so issue the result-less global RED, system scope because other
// GPUs add into the same entries over NVLink.
__device__ __forceinline__ void peer_red_add(double* dst, double v) {
  asm volatile("red.relaxed.sys.global.add.f64 [%0], %1;\n" ::"l"(dst), "d"(v) : "memory");
}

struct Vec3 {
  double x, y, z;
};

__device__ __forceinline__ Vec3 load_vertex(const double* __restrict__ v, int id) {
  const double* p = v + 3 * (int64_t)id;
  return Vec3{__ldg(p), __ldg(p + 1), __ldg(p + 2)};
}

// Affine cell map x = x0 + J xi with J = [x1-x0 | x2-x0 | x3-x0] (mesh.py:64-67).
struct Affine {
  double J[3][3];
  double adj[3][3];  // adjugate: J^{-1} = adj / det
  double det;
};

__device__ __forceinline__ void affine_from_vertices(const Vec3& a, const Vec3& b, const Vec3& c,
                                                     const Vec3& d, Affine& g) {
  const double e1[3] = {b.x - a.x, b.y - a.y, b.z - a.z};
  const double e2[3] = {c.x - a.x, c.y - a.y, c.z - a.z};
  const double e3[3] = {d.x - a.x, d.y - a.y, d.z - a.z};
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    g.J[i][0] = e1[i];
    g.J[i][1] = e2[i];
    g.J[i][2] = e3[i];
  }
  const double(&J)[3][3] = g.J;
  g.adj[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
  g.adj[0][1] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
  g.adj[0][2] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
  g.adj[1][0] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
  g.adj[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
  g.adj[1][2] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
  g.adj[2][0] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
  g.adj[2][1] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
  g.adj[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
  g.det = J[0][0] * g.adj[0][0] + J[0][1] * g.adj[1][0] + J[0][2] * g.adj[2][0];
}

// Symmetric G = det * J^{-1} J^{-T} = adj adj^T / det, packed (00,01,02,11,12,22):
// the reference D action J^{-1} (jxw J^{-T} g) equals w_q * G g (numpy_backend.py:68-76).
__device__ __forceinline__ void stiffness_metric(const Affine& g, double scale, double (&G)[6]) {
  const double s = scale / g.det;
  const double(&A)[3][3] = g.adj;
  G[0] = s * (A[0][0] * A[0][0] + A[0][1] * A[0][1] + A[0][2] * A[0][2]);
  G[1] = s * (A[0][0] * A[1][0] + A[0][1] * A[1][1] + A[0][2] * A[1][2]);
  G[2] = s * (A[0][0] * A[2][0] + A[0][1] * A[2][1] + A[0][2] * A[2][2]);
  G[3] = s * (A[1][0] * A[1][0] + A[1][1] * A[1][1] + A[1][2] * A[1][2]);
  G[4] = s * (A[1][0] * A[2][0] + A[1][1] * A[2][1] + A[1][2] * A[2][2]);
  G[5] = s * (A[2][0] * A[2][0] + A[2][1] * A[2][1] + A[2][2] * A[2][2]);
}

// Reference-cell tangents of local face lf (corners FACE_VERTICES[lf], reference.py:25-26):
// ds = xi(c1) - xi(c0), dt = xi(c2) - xi(c0) with xi(v0)=0, xi(v_k)=e_{k-1}.
__device__ __forceinline__ void face_tangents_ref(int lf, double (&ds)[3], double (&dt)[3]) {
  // lf 0: (1,2,3) -> ds = e1-e0, dt = e2-e0;  lf 1: (0,2,3) -> ds = e1, dt = e2
  // lf 2: (0,1,3) -> ds = e0, dt = e2;        lf 3: (0,1,2) -> ds = e0, dt = e1
  ds[0] = (lf == 0) ? -1.0 : (lf >= 2 ? 1.0 : 0.0);
  ds[1] = (lf <= 1) ? 1.0 : 0.0;
  ds[2] = 0.0;
  dt[0] = (lf == 0) ? -1.0 : 0.0;
  dt[1] = (lf == 3) ? 1.0 : 0.0;
  dt[2] = (lf == 3) ? 0.0 : 1.0;
}

}  // namespace tmf
