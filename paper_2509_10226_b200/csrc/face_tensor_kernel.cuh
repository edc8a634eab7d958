// SIPG interior-face kernel, reference-tensor form (affine faces), on FP64 tensor cores.
//
// The reference evaluates the face terms point by point (operator.py:387-437,
// face_qpoint numpy_backend.py:91-110); face_kernel.cuh restates that loop.  On
// an affine face every geometric factor is constant -- the surface factor s,
// the penalty and m+- = J+-^-1 n (geometry.py:202-236) -- so the face operator
// is a fixed linear combination of reference matrices that depend only on the
// face signature (lf-, lf+, code):
//     y = sum_c coef_c T^c [u-; u+],
//     coef = (s tau, s m~-/2, s m~+/2)     (7 per face: the face geometry record)
// with T^c the point sums of products of the two sides' face tables (value and
// face-frame derivative D = A_lf^T grad, face_kernel.cuh), taken once per plan
// on the host in extended precision (build_face_tensor_fragments, capi.cu).
//
// Sparsity (nodal basis, DoFs gathered face-DoFs-first): the value and the two
// tangential derivatives vanish off the face's NF DoFs, so with inputs and
// outputs ordered [-F | +F | -I | +I] (F = face DoFs, I = the others) every
// coefficient couples F to F, only the transversal ones (m~-_2, m~+_2) couple
// F to I, and nothing couples I to I.  One warp = 8 faces of one signature:
//     out F:  pairs (s tau, hm0) (hm1, hp0) (hp1, 0) over K = F,
//             pair (hm2, hp2) over K = F + I
//     out I:  pair (hm2, hp2) over K = F
// KF (4 KF + KI) + KI KF DMMAs per 8 faces: 48 at P2 and 150 at P3 against
// 60 / 170 for the point loop, and the 6-term contraction per output DoF
// replaces the jump/average/penalty arithmetic at every face point.
// Column order as in cell_tensor_kernel.cuh: lane (face fs, q4) gets the
// coefficient pair of output 4 ib + q4, which is also the input it gathered
// for k-step ib, so the scatter reuses the gather's addresses.
#pragma once
#include "face_kernel.cuh"

namespace tmf {

template <int N>
struct FaceTensorShape {
  static constexpr int NF = N == 4 ? 3 : N == 10 ? 6 : N == 20 ? 10 : 15;
  static constexpr int NI = N - NF;
  static constexpr int KF = (2 * NF + 3) / 4;   // k-steps (= output i-blocks) over [-F | +F]
  static constexpr int KI = (2 * NI + 3) / 4;   // over [-I | +I]
  static constexpr int RF = 4 * KF + KI;         // fragments per out-F block
  static constexpr int NFRAG = KF * RF + KI * KF;
  static constexpr int SMEM = NFRAG * 32 * 8 + 4 * N * 4;   // tables + the 4 gather orders
  static constexpr int DMMA_PER_BATCH = NFRAG;
};

// PF: prefetch the next batch's record, geometry and gathered u (as face_apply_kernel PF 2)
template <int N, int BLOCK, int MINB, bool PF>
__global__ void __launch_bounds__(BLOCK, MINB) face_tensor_kernel(FaceArgs a) {
  using S = FaceTensorShape<N>;
  constexpr int NF = S::NF, NI = S::NI, KF = S::KF, KI = S::KI, RF = S::RF;
  extern __shared__ __align__(16) double smem[];
  int* sperm = reinterpret_cast<int*>(smem + S::NFRAG * 32);   // (4, N) gather orders
  for (int i = threadIdx.x; i < 4 * N; i += BLOCK) sperm[i] = __ldg(a.perm + i);
  const int lane = threadIdx.x & 31;
  const int fs = lane >> 2;
  const int q4 = lane & 3;
  const int warp = threadIdx.x >> 5;
  constexpr int nwb = BLOCK / 32;

  // contiguous run of chunks per CTA: consecutive chunks of one (window, signature)
  // group share their table, which is restaged only when the signature changes
  const int64_t nwork = a.n_chunks * a.nc;
  const int64_t per = (nwork + gridDim.x - 1) / gridDim.x;
  const int64_t w0 = blockIdx.x * per;
  const int64_t w1 = w0 + per < nwork ? w0 + per : nwork;
  int cur_sig = -1;
  auto chunk_at = [&](int64_t w) {
    const int comp = a.nc == 1 ? 0 : (int)(w / a.n_chunks);
    return __ldg(a.chunks + (w - (int64_t)comp * a.n_chunks));
  };
  int4 nch = w0 < w1 ? chunk_at(w0) : make_int4(0, 0, 0, 0);
  for (int64_t w = w0; w < w1; ++w) {
    const int comp = a.nc == 1 ? 0 : (int)(w / a.n_chunks);
    const int4 ch = nch;
    if (w + 1 < w1) nch = chunk_at(w + 1);   // the next chunk's record, one chunk ahead
    const int lfm = ch.x / 6, lfp = ch.y / 6;
    const int sig = lfm * 24 + ch.y;
    if (sig != cur_sig || cur_sig < 0) {
      __syncthreads();   // the previous chunk's warps are done with the staged table (and sperm is set)
      const double2* src = reinterpret_cast<const double2*>(a.tfrags + (int64_t)sig * S::NFRAG * 32);
      double2* dst = reinterpret_cast<double2*>(smem);
      for (int i = threadIdx.x; i < S::NFRAG * 16; i += BLOCK) dst[i] = __ldg(src + i);
      __syncthreads();
      cur_sig = sig;
    }
    // the lane's input (= output) DoFs: region index x = 4 k + q4 -> (side, DoF in cell)
    int offF[KF], offI[KI];
    unsigned sideF = 0, sideI = 0;   // bit k: plus side
#pragma unroll
    for (int k = 0; k < KF; ++k) {
      const int x = 4 * k + q4;
      offF[k] = -1;
      if (x < NF) {
        offF[k] = sperm[lfm * N + x];
      } else if (x < 2 * NF) {
        offF[k] = sperm[lfp * N + x - NF];
        sideF |= 1u << k;
      }
    }
#pragma unroll
    for (int k = 0; k < KI; ++k) {
      const int x = 4 * k + q4;
      offI[k] = -1;
      if (x < NI) {
        offI[k] = sperm[lfm * N + NF + x];
      } else if (x < 2 * NI) {
        offI[k] = sperm[lfp * N + NF + x - NI];
        sideI |= 1u << k;
      }
    }

    int n_cm = -1, n_cp = -1;
    double naF[KF], naI[KI], ng[8];
    auto fetch = [&](int bi) {
      n_cm = -1;
      n_cp = -1;
      if (bi < ch.w) {
        const int64_t slot = ((int64_t)ch.z + bi) * 8 + fs;
        n_cm = __ldg(a.cm + slot);
        n_cp = __ldg(a.cp + slot);
        const double2* gp = reinterpret_cast<const double2*>(a.geo + slot * 8);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const double2 v = __ldg(gp + i);
          ng[2 * i] = v.x;
          ng[2 * i + 1] = v.y;
        }
      }
#pragma unroll
      for (int k = 0; k < KF; ++k) {
        const int c = (sideF >> k) & 1 ? n_cp : n_cm;
        naF[k] = (n_cm >= 0 && offF[k] >= 0) ? __ldg(a.u + ((int64_t)c * N + offF[k]) * a.nc + comp) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < KI; ++k) {
        const int c = (sideI >> k) & 1 ? n_cp : n_cm;
        naI[k] = (n_cm >= 0 && offI[k] >= 0) ? __ldg(a.u + ((int64_t)c * N + offI[k]) * a.nc + comp) : 0.0;
      }
    };
    if (PF) fetch(warp);

    for (int bi = warp; bi < ch.w; bi += nwb) {
      if (!PF) fetch(bi);
      const int c_m = n_cm, c_p = n_cp;
      double aF[KF], aI[KI];
#pragma unroll
      for (int k = 0; k < KF; ++k) aF[k] = naF[k];
#pragma unroll
      for (int k = 0; k < KI; ++k) aI[k] = naI[k];
      // coefficient slots: 0 s tau, 1 hm0, 2 hm1, 3 hp0, 4 hp1, 5 -, 6 hm2, 7 hp2
      const double cf[8] = {ng[6], ng[0], ng[1], ng[3], ng[4], 0.0, ng[2], ng[5]};
      if (PF) fetch(bi + nwb);

#pragma unroll
      for (int ib = 0; ib < KF; ++ib) {
        double wv[4][2];
#pragma unroll
        for (int p = 0; p < 4; ++p) wv[p][0] = wv[p][1] = 0.0;
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int kk = 0; kk < KF; ++kk) dmma(wv[p], aF[kk], smem[((ib * RF) + p * KF + kk) * 32 + lane]);
#pragma unroll
        for (int kk = 0; kk < KI; ++kk) dmma(wv[3], aI[kk], smem[((ib * RF) + 4 * KF + kk) * 32 + lane]);
        double yv = cf[0] * wv[0][0];
        yv = fma(cf[1], wv[0][1], yv);
        yv = fma(cf[2], wv[1][0], yv);
        yv = fma(cf[3], wv[1][1], yv);
        yv = fma(cf[4], wv[2][0], yv);
        yv = fma(cf[6], wv[3][0], yv);
        yv = fma(cf[7], wv[3][1], yv);
        if (c_m >= 0 && offF[ib] >= 0) {
          const int c = (sideF >> ib) & 1 ? c_p : c_m;
          atomicAdd(a.y + ((int64_t)c * N + offF[ib]) * a.nc + comp, yv);
        }
      }
#pragma unroll
      for (int ib = 0; ib < KI; ++ib) {
        double wv[2] = {0.0, 0.0};
#pragma unroll
        for (int kk = 0; kk < KF; ++kk) dmma(wv, aF[kk], smem[(KF * RF + ib * KF + kk) * 32 + lane]);
        const double yv = fma(cf[6], wv[0], cf[7] * wv[1]);
        if (c_m >= 0 && offI[ib] >= 0) {
          const int c = (sideI >> ib) & 1 ? c_p : c_m;
          atomicAdd(a.y + ((int64_t)c * N + offI[ib]) * a.nc + comp, yv);
        }
      }
    }
  }
}

}  // namespace tmf
