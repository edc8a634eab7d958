/*
 * Plain-C use of the tetmf_b200 C-ABI (no Python, no torch): builds the CG
 * Laplace operator for P1 on one reference tetrahedron split off a cube corner
 * and on a 2-cell mesh, applies it on the GPU through tmf_apply_host, and
 * checks the constant nullspace (A 1 = 0) and symmetry (u.Av = v.Au).
 *
 *   gcc -O2 -I include examples/c_abi_demo.c -L paper_2509_10226_b200 -ltetmf_b200 \
 *       -Wl,-rpath,$PWD/paper_2509_10226_b200 -o examples/c_abi_demo && examples/c_abi_demo
 *
 * Exit code 0 = pass, 1 = numerical failure, 2 = C-ABI error (message printed).
 */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "tetmf_b200.h"

/* P1 Lagrange on the reference tet: constant gradients; the 1-point rule is exact. */
static const double kGrad[3 * 4] = {-1, 1, 0, 0, /* d/dx of phi_0..3 */
                                    -1, 0, 1, 0, /* d/dy */
                                    -1, 0, 0, 1}; /* d/dz */

static int check(int rc) {
  if (rc != TMF_OK) fprintf(stderr, "tetmf error %d: %s\n", rc, tmf_last_error());
  return rc;
}

int main(void) {
  /* two positively oriented tets sharing the face (1, 2, 3) */
  const double verts[5 * 3] = {0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1, 1, 1, 1};
  const int32_t cells[2 * 4] = {0, 1, 2, 3, 4, 1, 3, 2};
  const double w[5] = {1.0 / 6.0, 0, 0, 0, 0};
  double value[5 * 4], grad[15 * 4];
  int q, j, k;
  for (q = 0; q < 5; ++q)
    for (j = 0; j < 4; ++j) {
      value[q * 4 + j] = 0.25;
      for (k = 0; k < 3; ++k) grad[(3 * q + k) * 4 + j] = kGrad[k * 4 + j];
    }

  tmf_plan_desc d;
  memset(&d, 0, sizeof d);
  d.operator_kind = TMF_CG_LAPLACE;
  d.degree = 1;
  d.n_dofs_per_cell = 4;
  d.n_components = 1;
  d.n_vertices = 5;
  d.n_cells = 2;
  d.n_scalar_dofs = 5;
  d.vertices = verts;
  d.cells = cells;
  d.cell_dofs = cells;           /* P1: vertex DoF = vertex id (dofmap.py:113-114) */
  d.n_q = 5;                     /* a 5-point rule with weight only on point 0 */
  d.cell_weights = w;
  d.value_matrix = value;
  d.grad_matrix = grad;
  d.diffusivity = 1.0;
  d.device = 0;

  tmf_plan* plan = NULL;
  if (check(tmf_plan_create(&d, &plan))) return 2;
  tmf_plan_info info;
  if (check(tmf_plan_get_info(plan, &info))) return 2;

  double one[5] = {1, 1, 1, 1, 1}, y[5], u[5] = {0.3, -1.2, 0.7, 2.0, -0.4}, v[5] = {1.1, 0.2, -0.5, 0.9, 0.6};
  double Au[5], Av[5];
  if (check(tmf_apply_host(plan, one, y))) return 2;
  if (check(tmf_apply_host(plan, u, Au))) return 2;
  if (check(tmf_apply_host(plan, v, Av))) return 2;
  double n1 = 0, uAv = 0, vAu = 0, scale = 0;
  for (j = 0; j < 5; ++j) {
    n1 += y[j] * y[j];
    uAv += u[j] * Av[j];
    vAu += v[j] * Au[j];
    scale += Au[j] * Au[j];
  }
  printf("%s\nn_global_dofs %lld, flops_alg %.0f, kernels/apply %d\n", tmf_version(),
         (long long)info.n_global_dofs, info.flops_alg, info.kernels_per_apply);
  printf("|A 1| = %.3e, u.Av - v.Au = %.3e\n", sqrt(n1), uAv - vAu);
  tmf_plan_destroy(plan);
  const int ok = sqrt(n1) <= 1e-13 * sqrt(scale) && fabs(uAv - vAu) <= 1e-13 * sqrt(scale);
  printf("%s\n", ok ? "PASS" : "FAIL");
  return ok ? 0 : 1;
}
