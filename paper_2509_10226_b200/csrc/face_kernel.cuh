// SIPG face-term kernel on FP64 tensor cores (sm_100a).
//
// Restates the reference face loop (operator.py:387-437) with the
// quadrature-point arithmetic of face_qpoint / boundary_qpoint
// (numpy_backend.py:91-119):
//     jump = V- - V+,  avg = (m-.G- + m+.G+)/2,  w = |t_s x t_t| w_q scale
//     qv = w (tau jump - avg),   qg± = -w jump m± / 2
//     R- = Fv-^T qv + Fg-^T qg-,   R+ = -Fv+^T qv + Fg+^T qg+
//   boundary (Dirichlet): qv = w (tau V - m.G),  qg = -w V m
// One warp handles 8 faces that share the signature (lf-, lf+, code), so the
// face tables (lf-, 0) and (lf+, code) are common B operands, exactly the
// reference's grouping of faces by signature (operator.py:152-170); the host
// sorts faces by signature and pads each group to a multiple of 8.
// Tables are pre-swizzled DMMA fragments (4 components per point: value and 3
// reference gradients; GEMM2 tables carry w_q) read through L1 (__ldg).
// Geometry (unit normal outward from the minus cell, |t_s x t_t|,
// m = J^-1 n on each side) is recomputed from vertex coordinates
// (geometry.py:202-236).  Contributions are added to y with fp64 RED.
#pragma once
#include "common.cuh"

namespace tmf {

struct FaceArgs {
  const double* __restrict__ u;
  double* __restrict__ y;
  const int* __restrict__ cells;
  const double* __restrict__ verts;
  const double* __restrict__ kappa;
  const double* __restrict__ frags;   // per (lf, code) combo: B1 then B2 fragments
  const int2* __restrict__ batch_combo;  // (minus combo, plus combo); plus = -1 for boundary
  const int* __restrict__ cm;         // (n_batches*8) minus cell, -1 = padding
  const int* __restrict__ cp;         // (n_batches*8) plus cell (interior)
  const double* __restrict__ tau;     // (n_batches*8)
  int64_t n_batches;
  int n_dpc;
  int nc;
  double scale;
};

template <int N, int QF>
struct FaceShape {
  static constexpr int KK = (N + 3) / 4;
  static constexpr int T = (QF + 7) / 8;
  static constexpr int NJ = (N + 7) / 8;
  static constexpr int NB1 = T * 4 * KK;
  static constexpr int NB2 = T * 4 * 2 * NJ;
  static constexpr int NFRAG = NB1 + NB2;      // per (lf, code) combo
};

struct FaceGeo {
  double m[3];  // J^-1 n (times kappa)
  double s;     // |t_s x t_t| * scale
};

__device__ __forceinline__ void cell_affine(const FaceArgs& a, int c, Affine& g, Vec3& opp_base,
                                            int lf, Vec3& face_v0) {
  int vid[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) vid[i] = __ldg(a.cells + 4 * (int64_t)c + i);
  const Vec3 x0 = load_vertex(a.verts, vid[0]), x1 = load_vertex(a.verts, vid[1]),
             x2 = load_vertex(a.verts, vid[2]), x3 = load_vertex(a.verts, vid[3]);
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

template <int N, int QF, bool BOUNDARY>
__global__ void __launch_bounds__(256) face_apply_kernel(FaceArgs a) {
  using S = FaceShape<N, QF>;
  const int lane = threadIdx.x & 31;
  const int fs = lane >> 2;
  const int q4 = lane & 3;
  const int64_t nw = (int64_t)gridDim.x * 8;
  const int64_t nwork = a.n_batches * a.nc;

  for (int64_t w = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); w < nwork; w += nw) {
    const int comp = (int)(w / a.n_batches);
    const int64_t b = w - (int64_t)comp * a.n_batches;
    const int2 combo = __ldg(a.batch_combo + b);
    const int lfm = combo.x / 6;
    const int c_m = __ldg(a.cm + b * 8 + fs);
    const bool valid = c_m >= 0;
    const int c_p = BOUNDARY ? -1 : __ldg(a.cp + b * 8 + fs);

    // ---- gather both sides
    double am[S::KK], ap[S::KK];
#pragma unroll
    for (int kk = 0; kk < S::KK; ++kk) {
      const int j = 4 * kk + q4;
      am[kk] = 0.0;
      ap[kk] = 0.0;
      if (valid && j < N) {
        am[kk] = __ldg(a.u + ((int64_t)c_m * N + j) * a.nc + comp);
        if (!BOUNDARY) ap[kk] = __ldg(a.u + ((int64_t)c_p * N + j) * a.nc + comp);
      }
    }

    // ---- face geometry
    FaceGeo gm, gp;
    double tau = 0.0;
    {
      const int cmm = valid ? c_m : 0;
      Affine Jm;
      Vec3 opp, fv0;
      cell_affine(a, cmm, Jm, opp, lfm, fv0);
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
      // outward from the minus cell: away from the vertex opposite the face
      const double side = n[0] * (fv0.x - opp.x) + n[1] * (fv0.y - opp.y) + n[2] * (fv0.z - opp.z);
      const double inv = (side < 0 ? -1.0 : 1.0) / area2;
#pragma unroll
      for (int i = 0; i < 3; ++i) n[i] *= inv;
      apply_inv(Jm, n, gm.m);
      gm.s = area2 * a.scale;
      tau = valid ? __ldg(a.tau + b * 8 + fs) : 0.0;
      double km = 1.0;
      if (a.kappa) km = __ldg(a.kappa + cmm);
      if (!BOUNDARY) {
        const int cpp = valid ? c_p : 0;
        Affine Jp;
        Vec3 o2, f2;
        cell_affine(a, cpp, Jp, o2, 0, f2);
        apply_inv(Jp, n, gp.m);
        double kp = 1.0;
        if (a.kappa) kp = __ldg(a.kappa + cpp);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          gm.m[i] *= km;
          gp.m[i] *= kp;
        }
        tau *= fmax(km, kp);
      } else {
#pragma unroll
        for (int i = 0; i < 3; ++i) gm.m[i] *= km;
        tau *= km;
      }
    }

    const double* Fm = a.frags + (int64_t)combo.x * S::NFRAG * 32;
    const double* Fp = a.frags + (int64_t)(BOUNDARY ? 0 : combo.y) * S::NFRAG * 32;
    double ym[S::NJ][2], yp[S::NJ][2];
#pragma unroll
    for (int nj = 0; nj < S::NJ; ++nj) ym[nj][0] = ym[nj][1] = yp[nj][0] = yp[nj][1] = 0.0;

#pragma unroll
    for (int t = 0; t < S::T; ++t) {
      double vm[4][2], vp[4][2];
#pragma unroll
      for (int c = 0; c < 4; ++c) vm[c][0] = vm[c][1] = vp[c][0] = vp[c][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < S::KK; ++kk)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int f = ((t * 4 + c) * S::KK + kk) * 32 + lane;
          dmma(vm[c], am[kk], __ldg(Fm + f));
          if (!BOUNDARY) dmma(vp[c], ap[kk], __ldg(Fp + f));
        }
      double qm[4][2], qp[4][2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double dnm = gm.m[0] * vm[1][i] + gm.m[1] * vm[2][i] + gm.m[2] * vm[3][i];
        if (BOUNDARY) {
          qm[0][i] = gm.s * (tau * vm[0][i] - dnm);
          const double wj = -gm.s * vm[0][i];
#pragma unroll
          for (int k = 0; k < 3; ++k) qm[1 + k][i] = wj * gm.m[k];
        } else {
          const double dnp = gp.m[0] * vp[1][i] + gp.m[1] * vp[2][i] + gp.m[2] * vp[3][i];
          const double jump = vm[0][i] - vp[0][i];
          const double qv = gm.s * (tau * jump - 0.5 * (dnm + dnp));
          const double hw = -0.5 * gm.s * jump;
          qm[0][i] = qv;
          qp[0][i] = -qv;
#pragma unroll
          for (int k = 0; k < 3; ++k) {
            qm[1 + k][i] = hw * gm.m[k];
            qp[1 + k][i] = hw * gp.m[k];
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int nj = 0; nj < S::NJ; ++nj) {
            const int f = (S::NB1 + (((t * 4 + c) * 2 + i) * S::NJ + nj)) * 32 + lane;
            dmma(ym[nj], qm[c][i], __ldg(Fm + f));
            if (!BOUNDARY) dmma(yp[nj], qp[c][i], __ldg(Fp + f));
          }
    }

    if (valid) {
#pragma unroll
      for (int nj = 0; nj < S::NJ; ++nj)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int j = 8 * nj + 2 * q4 + i;
          if (j < N) {
            atomicAdd(a.y + ((int64_t)c_m * N + j) * a.nc + comp, ym[nj][i]);
            if (!BOUNDARY) atomicAdd(a.y + ((int64_t)c_p * N + j) * a.nc + comp, yp[nj][i]);
          }
        }
    }
  }
}

}  // namespace tmf
