/*
 * tetmf_b200 -- C ABI of the B200 matrix-free operator apply.
 *
 * This is the drop-in boundary for the reference's operator layer
 * (/root/reference/pkg/src/tetmf/operator.py).  One plan replaces one operator
 * object of the reference:
 *
 *   tmf_plan_create   <- CgPoissonOperator.__init__   operator.py:314-318
 *                        DgSipgOperator.__init__      operator.py:449-454
 *                        HelmholtzOperator.__init__   operator.py:473-479
 *                        (+ _OperatorBase.__init__ operator.py:190-223 and
 *                           _DgFaceMixin._setup_faces operator.py:337-385)
 *   tmf_apply         <- <Operator>.apply(u) -> y      operator.py:320-331,
 *                        456-466, 481-493 (device pointers, stream-ordered)
 *   tmf_apply_host    <- the same with host buffers (copies inside; the call the
 *                        Python shim makes for NumPy inputs)
 *   tmf_diagonal      <- sparse.assemble(...).diagonal()   sparse.py:237-243
 *                        (matrix-free, used by the Jacobi preconditioner)
 *   tmf_pcg           <- SPEC.md:509-517 cg_solve with point-Jacobi (absent
 *                        from the reference package; fixed iteration count)
 *   tmf_last_error    <- the ValueError / RuntimeError messages of the
 *                        reference (operator.py:305-308 etc.)
 *
 * All pointers in tmf_plan_desc are HOST pointers; the plan copies what it
 * needs to the device and the caller keeps ownership.  Status codes: 0 = ok,
 * TMF_EINVAL = invalid argument (Python: ValueError), TMF_ECUDA = CUDA
 * failure / no device (Python: RuntimeError).  The library has no CPU
 * fallback: every apply runs on the GPU or fails.
 */
#ifndef TETMF_B200_H
#define TETMF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMF_OK 0
#define TMF_EINVAL 1
#define TMF_ECUDA 2

/* operator kinds */
#define TMF_CG_LAPLACE 0     /* CgPoissonOperator                                   */
#define TMF_DG_SIPG 1        /* DgSipgOperator                                      */
#define TMF_DG_HELMHOLTZ 2   /* mass_scale*M + diffusivity*(kappa-)SIPG; n_comp 1|3  */

typedef struct tmf_plan tmf_plan;

typedef struct tmf_plan_desc {
  int32_t operator_kind;
  int32_t degree;              /* 1..4                                              */
  int32_t n_dofs_per_cell;     /* (p+1)(p+2)(p+3)/6                                 */
  int32_t n_components;        /* 1, or 3 interleaved (index = scalar*3 + c)        */
  int64_t n_vertices;
  int64_t n_cells;
  int64_t n_scalar_dofs;
  const double* vertices;      /* (n_vertices, 3)                                    */
  const int32_t* cells;        /* (n_cells, 4), positively oriented                  */
  const int32_t* cell_dofs;    /* (n_cells, n_dpc) CG numbering; NULL for DG         */
  const uint8_t* dirichlet_mask; /* (n_scalar_dofs,) CG strong Dirichlet, or NULL   */
  int32_t n_q;
  int32_t n_qf;
  const double* cell_weights;  /* (n_q,)                                             */
  const double* value_matrix;  /* (n_q, n_dpc)                                       */
  const double* grad_matrix;   /* (3 n_q, n_dpc), row 3*i + k                        */
  const double* face_weights;  /* (n_qf,)                         DG only            */
  const double* face_values;   /* (4, 6, n_qf, n_dpc)             DG only            */
  const double* face_grads;    /* (4, 6, 3 n_qf, n_dpc)           DG only            */
  int64_t n_interior_faces;
  const int32_t* interior_faces; /* (n_if, 5): c-, lf-, c+, lf+, code                */
  const double* tau_interior;  /* (n_if,)                                            */
  int64_t n_boundary_faces;
  const int32_t* boundary_faces; /* (n_bf, 3): cell, lf, boundary id                 */
  const double* tau_boundary;  /* (n_bf,)                                            */
  const uint8_t* boundary_dirichlet; /* (n_bf,) 1 = weak Dirichlet (SIPG) face       */
  const double* kappa;         /* (n_cells,) per-cell Laplace coefficient, or NULL   */
  double mass_scale;           /* Helmholtz mass coefficient                          */
  double diffusivity;          /* Laplace/SIPG scale (nu)                             */
  int32_t device;              /* CUDA device ordinal                                 */
  int32_t flags;               /* bits 8-11: face batches per CTA chunk / 8 (0 = 32);
                                  13-14 + 19 (bit 2): cell engine (0 by degree,
                                  1 DMMA quadrature points, 3 DMMA reference tensor,
                                  4 modal: the point kernel on M = dim P_{p-1}
                                  unit-weight modes); 15-16: CG block assembly (0 auto,
                                  1 off, 2 on); 17-18 face engine (0 by degree,
                                  1 quadrature points, 3 modal: the point loop on NF
                                  exact unit-weight face modes); 20: also build the
                                  fp32 mirror (tmf_apply_f32); 22-23 CG cell traversal
                                  order (0 auto: Morton when the given order has no
                                  locality, 1 the given order, 2 Morton; u / y keep the
                                  caller's numbering either way).  Other bits: reserved. */
} tmf_plan_desc;

typedef struct tmf_plan_info {
  int64_t n_global_dofs;       /* n_scalar_dofs * n_components                       */
  double flops_alg;            /* reference counter flops per apply     */
  double bytes_alg;            /* compulsory HBM bytes per apply         */
  double flops_issued;         /* FP64 FMA*2 the kernels actually issue (padding incl.) */
  int32_t kernels_per_apply;   /* kernel launches per tmf_apply                       */
  int32_t n_face_batches;      /* signature-uniform 8-face batches (DG)               */
  int64_t device_bytes;        /* device memory held by the plan                      */
  int32_t block_cells;         /* CG block assembly: cells per block (0 = off)         */
  double block_ratio;          /* unique block DoFs / cell-DoF slots (CG block assembly) */
  int32_t cell_engine;         /* cell kernel in use: 1 DMMA quadrature points,
                                  3 DMMA reference tensor (affine precontraction),
                                  4 modal (point kernel on M exact unit-weight modes) */
  double flops_engine;         /* useful flops per apply of the algorithm the engines
                                  run (= flops_alg except for the tensor engines)      */
  int32_t face_engine;         /* faces: 1 quadrature points, 3 modal (0: no faces)   */
  int32_t cell_order;          /* CG cell traversal: 1 the caller's order, 2 Morton order of the
                                  centroids (0: DG, always the caller's)              */
} tmf_plan_info;

int tmf_plan_create(const tmf_plan_desc* desc, tmf_plan** out);
int tmf_plan_destroy(tmf_plan* plan);
int tmf_plan_get_info(const tmf_plan* plan, tmf_plan_info* info);

/* Test hook of the bounds-checking build (libtetmf_b200_debug.so, -DTMF_DEBUG_CHECKS):
 * overwrite the device copy of one CG cell-DoF slot (to show the kernels' range checks
 * fire).  The release library returns TMF_EINVAL. */
int tmf_debug_poke_dof(tmf_plan* plan, int64_t slot, int32_t value);

/* Test hook (host only, no GPU): the order in which CTA `block` of a `grid`-CTA face launch
 * visits the `n_work` face chunks (face_kernel.cuh ChunkWalk: round-robin, one contiguous run
 * per CTA, or runs of `run` chunks dealt round-robin).  Writes the visited work items to
 * out[0..*n_out) (capacity `cap`); entries >= n_work are skipped as the kernel skips them. */
int tmf_debug_chunk_walk(int64_t n_work, int64_t grid, int64_t block, int blocked, int run,
                         int64_t* out, int64_t cap, int64_t* n_out);

/* y = A u on device pointers (length n_global_dofs), ordered on `stream`
 * (a cudaStream_t, NULL = legacy default stream).  y is overwritten. */
int tmf_apply(tmf_plan* plan, const double* u, double* y, void* stream);

/* The apply in stages, for callers that overlap communication with compute
 * (the multi-GPU operators): ZERO clears y (CG), CELLS runs the cell kernel on
 * cells [cell_begin, cell_end), FACES runs the face kernels (DG), FIXUP writes
 * the identity Dirichlet rows (CG).  tmf_apply == all four on every cell. */
#define TMF_STAGE_ZERO 1
#define TMF_STAGE_CELLS 2
#define TMF_STAGE_FACES 4
#define TMF_STAGE_FIXUP 8
int tmf_apply_stages(tmf_plan* plan, const double* u, double* y, int stages, int64_t cell_begin,
                     int64_t cell_end, void* stream);

/* Same with host buffers: H2D(u), apply, D2H(y), synchronous. */
int tmf_apply_host(tmf_plan* plan, const double* u_host, double* y_host);

/* Same, asynchronous on `stream`: H2D(u), apply, D2H(y) are enqueued and the
 * call returns; u_host/y_host should be pinned and must stay valid until the
 * stream reaches that point.  Lets a caller pipeline several plans' copies
 * against each other's kernels. */
int tmf_apply_host_async(tmf_plan* plan, const double* u_host, double* y_host, void* stream);

/* Several plans' host applies as one pipeline, asynchronous on `stream`: the
 * uploads of u_hosts[0..n) run back to back in that order on one copy stream,
 * the kernels on one compute stream (plan i's kernels wait only for plan i's
 * upload), the downloads on the other copy direction (plan i's download waits
 * only for plan i's kernels); `stream` is ordered before and after the whole
 * pipeline.  Same results as n tmf_apply_host_async calls (the reference has no
 * batched call; it replaces the caller's loop over operator.apply(u) calls,
 * operator.py:320-331).  All plans on one device; host buffers pinned.  A plan may
 * appear more than once (its entries run in order: each waits for the previous
 * download of that plan's staging buffers); plans with peers are rejected. */
int tmf_apply_host_multi(tmf_plan* const* plans, const double* const* u_hosts, double* const* y_hosts, int n,
                         void* stream);

/* Per-stage timing of `reps` back-to-back applies (device pointers), CUDA
 * events on `stream`: out_ms[0] = total, out_ms[1..] = per kernel class
 * (cell, face, fixup).  For the bench only. */
int tmf_apply_timed(tmf_plan* plan, const double* u, double* y, void* stream, int reps,
                    double* out_ms, int n_out);

/* diag(A) on device (identity rows on strong Dirichlet DoFs). CG only. */
int tmf_diagonal(tmf_plan* plan, double* diag, void* stream);

/* Point-Jacobi PCG, x0 = 0, exactly `iters` iterations (no early exit).
 * b, x device pointers; res_norms (host, length iters+1) receives ||r_k||_2,
 * or NULL.  All scalars stay on the device; one host sync at the end. */
int tmf_pcg(tmf_plan* plan, const double* b, double* x, int iters, double* res_norms,
            void* stream);

/* Fused point-Jacobi PCG vector kernels for callers that drive the iteration
 * themselves (the multi-GPU solver: local partial sums are all-reduced between
 * the calls).  All pointers are device pointers on the current device; the
 * scalar outputs are device doubles that are ACCUMULATED (caller zeroes them).
 *   tmf_vec_dot:       *out += a.b
 *   tmf_pcg_init:      x = 0, r = b, z = r/d, p = z;  *rz += r.z, *rr += r.r
 *   tmf_pcg_update:    alpha = *rz_k / *pq_k; x += alpha p; r -= alpha q; z = r/d;
 *                      *rz_next += r.z, *rr_next += r.r
 *   tmf_pcg_direction: p = z + (*rz_next / *rz_k) p                              */
int tmf_vec_dot(const double* a, const double* b, int64_t n, double* out, void* stream);
int tmf_pcg_init(const double* b, const double* d, double* x, double* r, double* z, double* p,
                 int64_t n, double* rz, double* rr, void* stream);
int tmf_pcg_update(const double* p, const double* q, const double* d, double* x, double* r,
                   double* z, int64_t n, const double* rz_k, const double* pq_k, double* rz_next,
                   double* rr_next, void* stream);
int tmf_pcg_direction(const double* z, double* p, int64_t n, const double* rz_k,
                      const double* rz_next, void* stream);

/* Multi-GPU without a halo exchange (SURVEY §8e "fused peer-store halo").  The
 * plan's local layout is owned entries [0, n_own) then ghosts [n_own, n_own+n_ghost)
 * (CG: DoFs, DG: cells); ghost e lives at element ghost_index[e] of rank
 * ghost_rank[e]'s local vector.  peer_u / peer_y hold every rank's registered
 * u / y device buffers as mapped on THIS device (tmf_ipc_open_handle for other
 * processes; plain pointers when ranks share a device).  The cell kernel (CG)
 * gathers ghost u with peer loads and scatters ghost y with peer REDs; the face
 * kernel (DG) gathers ghost cells' u from the owner -- compute and exchange in one
 * kernel over NVLink.  Applies must then pass the registered buffers; CG uses
 * tmf_apply_stages: ZERO, cross-rank barrier, CELLS|FIXUP, cross-rank barrier.
 * CG cells [0, n_peer_free_cells) touch no ghost DoF and run the plain kernel.
 * n_ranks = 0 switches peers off.  Needs the default DMMA cell engine. */
int tmf_plan_set_peers(tmf_plan* plan, int32_t n_ranks, const uint64_t* peer_u, const uint64_t* peer_y,
                       int32_t self_rank, int64_t n_own, int64_t n_ghost, const int32_t* ghost_rank,
                       const int32_t* ghost_index, int64_t n_peer_free_cells);
/* Dedicated device allocations (IPC-exportable at offset 0) and CUDA IPC handles
 * (64 bytes) for mapping another process's buffers. */
int tmf_alloc(int64_t bytes, int32_t device, void** dev_ptr);
int tmf_free(void* dev_ptr);
int tmf_ipc_get_handle(const void* dev_ptr, uint8_t handle[64]);
int tmf_ipc_open_handle(const uint8_t handle[64], int32_t device, void** dev_ptr);
int tmf_ipc_close_handle(void* dev_ptr);

/* Hierarchical cell reordering (host-side setup; no GPU needed).  Writes the
 * permutation new_of_old (cell e moves to position new_of_old[e]), to be
 * applied like mesh.apply_cell_permutation (mesh.py:291-293).  Replaces the
 * reorder module the reference only specifies. */
int tmf_hierarchical_reorder(int64_t n_cells, int64_t n_interior_faces,
                             const int32_t* interior_faces, int32_t group_size,
                             int64_t* new_of_old);

/* Host-side setup at scale (no GPU needed), bit-identical to the reference:
 * face pairing <- mesh._build_faces (mesh.py:84-120); interior_out needs room
 * for 2*n_cells rows of 5, boundary_out for 4*n_cells rows of 3 (boundary ids
 * are left 0 for the caller).  CG DoF numbering <- build_dof_map
 * (dofmap.py:67-123, + the P4 convention of SURVEY Appendix B6). */
int tmf_build_faces(int64_t n_cells, const int32_t* cells, int64_t n_vertices,
                    int32_t* interior_out, int64_t* n_interior, int32_t* boundary_out,
                    int64_t* n_boundary);
int tmf_build_cg_dofs(int64_t n_cells, const int32_t* cells, int64_t n_vertices, int32_t degree,
                      int32_t* cell_dofs, int64_t* n_scalar_dofs);

/* Greedy distance-1 colouring of the cells' face-adjacency graph (cells in order, smallest
 * colour unused by a coloured face neighbour; <= 5 colours).  Host-side setup; used to probe
 * the exact diagonal of DG operators (one apply per colour and local DoF). */
int tmf_color_cells(int64_t n_cells, int64_t n_interior_faces, const int32_t* interior_faces,
                    int32_t* colors, int32_t* n_colors);

/* p-multigrid building blocks (the paper's solver layer, PAPER.md:423-436,
 * SPEC.md:494-565; the reference has no implementation).  A transfer links two CG spaces of
 * degrees pf > pc on the same mesh (or a DG space over the CG space of the same degree: the
 * c-transfer, interp = identity): prolongation x_f = P x_c interpolates the coarse
 * function at the fine nodes (interp[i*n_coarse_dpc + j] = coarse basis j at fine node i,
 * row-major n_fine_dpc x n_coarse_dpc); restriction r_c = P^T r_f is its exact transpose.
 * Each fine DoF is written by one owner cell (the first cell containing it).  Dirichlet
 * masks (uint8 per DoF, or NULL): fine Dirichlet DoFs are set to 0 by an overwriting
 * prolongation (left alone when add != 0) and never restricted; coarse Dirichlet DoFs are
 * read as 0 and never written by restriction.  Device vectors, stream-ordered. */
typedef struct tmf_transfer tmf_transfer;
typedef struct tmf_transfer_desc {
  int64_t n_cells;
  int32_t n_fine_dpc, n_coarse_dpc;          /* fine >= coarse; coarse 4/10/20/35      */
  int64_t n_fine_dofs, n_coarse_dofs;
  const int32_t* fine_cell_dofs;             /* host (n_cells, n_fine_dpc)              */
  const int32_t* coarse_cell_dofs;           /* host (n_cells, n_coarse_dpc)            */
  const uint8_t* fine_dirichlet;             /* host (n_fine_dofs) or NULL              */
  const uint8_t* coarse_dirichlet;           /* host (n_coarse_dofs) or NULL            */
  const double* interp;                      /* host (n_fine_dpc, n_coarse_dpc)         */
  int32_t device;
} tmf_transfer_desc;
int tmf_transfer_create(const tmf_transfer_desc* desc, tmf_transfer** out);
/* h-coarsening onto a non-nested coarse mesh (P1 -> P1): fine DoF i takes the coarse values at
 * coarse_index[4i..4i+3] with weights[4i..4i+3] (the barycentric coordinates of the fine node in
 * the coarse cell containing it).  tmf_prolongate / tmf_restrict (and the _f32 forms) apply it. */
typedef struct tmf_point_transfer_desc {
  int64_t n_fine_dofs, n_coarse_dofs;
  int32_t entries_per_row;                   /* 4                                       */
  const int32_t* coarse_index;               /* host (n_fine_dofs, 4)                   */
  const double* weights;                     /* host (n_fine_dofs, 4)                   */
  const uint8_t* fine_dirichlet;             /* host (n_fine_dofs) or NULL              */
  const uint8_t* coarse_dirichlet;           /* host (n_coarse_dofs) or NULL            */
  int32_t device;
} tmf_point_transfer_desc;
int tmf_transfer_create_points(const tmf_point_transfer_desc* desc, tmf_transfer** out);
int tmf_transfer_destroy(tmf_transfer* t);
int tmf_prolongate(tmf_transfer* t, const double* xc, double* xf, int add, void* stream);
int tmf_restrict(tmf_transfer* t, const double* rf, double* rc, void* stream);
/* Chebyshev-Jacobi smoother step (fused):  ax == NULL (x = 0 on entry): d = c2 D^-1 b, x = d;
 * otherwise d = c1 d + c2 D^-1 (b - ax), x += d.   tmf_vec_axpby: out = alpha x + beta y. */
int tmf_chebyshev_step(int64_t n, const double* ax, const double* b, const double* dinv, double* x,
                       double* d, double c1, double c2, void* stream);
int tmf_vec_axpby(int64_t n, double alpha, const double* x, double beta, const double* y, double* out,
                  void* stream);
/* Single-precision mirrors for a mixed-precision V-cycle (the paper's fp32 multigrid with an
 * fp64 outer CG).  tmf_apply_f32: y = A u in fp32 for a scalar CG Laplace
 * plan created with flags bit 20 (modal cell form, fp32 FFMA, identity Dirichlet rows). */
int tmf_apply_f32(tmf_plan* plan, const float* u, float* y, void* stream);
int tmf_prolongate_f32(tmf_transfer* t, const float* xc, float* xf, int add, void* stream);
int tmf_restrict_f32(tmf_transfer* t, const float* rf, float* rc, void* stream);
int tmf_chebyshev_step_f32(int64_t n, const float* ax, const float* b, const float* dinv, float* x,
                           float* d, float c1, float c2, void* stream);
int tmf_vec_axpby_f32(int64_t n, float alpha, const float* x, float beta, const float* y, float* out,
                      void* stream);

const char* tmf_last_error(void);
const char* tmf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* TETMF_B200_H */
