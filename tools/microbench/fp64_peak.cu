// FP64 peak microbenchmarks for the B200 roofline denominator.
//
// The matrix-free apply is FP64-bound, and MEASURED_PEAKS.json
// holds no FP64 number, so this measures it:
//   dfma_reg   : register-only DFMA chains            (vector FP64 pipe peak)
//   dmma_reg   : mma.sync m8n8k4 f64 chains           (FP64 tensor-core peak)
//   dfma_const : DFMA whose multiplicand is a __constant__ operand at a
//                compile-time offset, streamed over 4096 distinct constants
//                (the E-table-in-constant-bank design of the cell kernel)
//   dfma_smem  : DFMA with a broadcast shared-memory multiplicand
// Each kernel is timed with CUDA events; the SM clock is sampled with
// clock64()/globaltimer inside the kernel so the FMA/clk/SM figure is exact.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ unsigned long long g_clk[2];

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

template <int CHAINS>
__global__ void dfma_reg(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  uint64_t c0 = clock64(), t0 = gtimer();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  uint64_t c1 = clock64(), t1 = gtimer();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 1234.5678) out[threadIdx.x] = s;  // keeps the chains live
  if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[0] = c1 - c0; g_clk[1] = t1 - t0; }
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int CHAINS>
__global__ void dmma_reg(double* out, int iters, double a, double b) {
  double acc[CHAINS][2];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { acc[c][0] = c; acc[c][1] = -c; }
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  uint64_t c0 = clock64(), t0 = gtimer();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int c = 0; c < CHAINS; ++c) dmma(acc[c], av, bv);
  }
  uint64_t c1 = clock64(), t1 = gtimer();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1234.5678) out[threadIdx.x] = s;  // keeps the chains live
  if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[0] = c1 - c0; g_clk[1] = t1 - t0; }
}

constexpr int NCONST = 4096;
__constant__ double c_tab[NCONST];

// 8 chains x 512 constants per pass; each DFMA reads a distinct constant.
__global__ void dfma_const(double* out, int iters) {
  double acc[8], x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { acc[c] = threadIdx.x * 1e-3 + c; x[c] = 1e-3 * (c + 1); }
  uint64_t c0 = clock64(), t0 = gtimer();
  // single pass (no outer loop: a loop would let ptxas hoist the constants)
#pragma unroll
  for (int k = 0; k < NCONST / 8; ++k)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma(c_tab[k * 8 + c], x[c], acc[c]);
  uint64_t c1 = clock64(), t1 = gtimer();
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  if (s == 1234.5678) out[threadIdx.x] = s;  // keeps the chains live
  if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[0] = c1 - c0; g_clk[1] = t1 - t0; }
}

__global__ void dfma_smem(double* out, int iters) {
  __shared__ double tab[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) tab[i] = 1.0 + 1e-6 * i;
  __syncthreads();
  double acc[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  uint64_t c0 = clock64(), t0 = gtimer();
  for (int i = 0; i < iters; ++i) {
#pragma unroll 4
    for (int k = 0; k < 1024; k += 2) {
      double2 e = *reinterpret_cast<const double2*>(&tab[k]);
#pragma unroll
      for (int c = 0; c < 8; c += 2) { acc[c] = fma(acc[c], e.x, 0.5); acc[c + 1] = fma(acc[c + 1], e.y, 0.5); }
    }
  }
  uint64_t c1 = clock64(), t1 = gtimer();
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c];
  if (s == 1234.5678) out[threadIdx.x] = s;  // keeps the chains live
  if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[0] = c1 - c0; g_clk[1] = t1 - t0; }
}

// DMMA and DFMA issued together: are the tensor FP64 pipe and the vector FP64
// pipe independent?  RATIO DFMA per DMMA per warp.
template <int RATIO>
__global__ void mix_kernel(double* out, int iters, double a, double b) {
  double acc[8][2];
  double f[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { acc[c][0] = c; acc[c][1] = -c; f[c] = threadIdx.x * 1e-3 + c; }
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  uint64_t c0 = clock64(), t0 = gtimer();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      dmma(acc[c], av, bv);
#pragma unroll
      for (int r = 0; r < RATIO; ++r) f[(c + r) & 7] = fma(f[(c + r) & 7], a, b);
    }
  }
  uint64_t c1 = clock64(), t1 = gtimer();
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1] + f[c];
  if (s == 1234.5678) out[threadIdx.x] = s;  // keeps the chains live
  if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[0] = c1 - c0; g_clk[1] = t1 - t0; }
}

// DMMA dependent-chain latency: one warp per SMSP, CH independent chains.
template <int CH>
__global__ void dmma_chain(double* out, int iters, double a, double b) {
  double acc[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) { acc[c][0] = c; acc[c][1] = -c; }
  double av = a + threadIdx.x * 1e-9, bv = b - threadIdx.x * 1e-9;
  uint64_t c0 = clock64(), t0 = gtimer();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(acc[c], av, bv);
  }
  uint64_t c1 = clock64(), t1 = gtimer();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1];
  if (s == 1234.5678) out[threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[0] = c1 - c0; g_clk[1] = t1 - t0; }
}

template <typename F>
static int timeit(const char* name, F launch, double fma_per_launch, int n_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  launch(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0); launch(); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  unsigned long long clk[2];
  cudaMemcpyFromSymbol(clk, g_clk, sizeof(clk));
  double mhz = clk[1] ? 1e3 * (double)clk[0] / (double)clk[1] : 0;
  double tflops = 2.0 * fma_per_launch / (best * 1e-3) / 1e12;
  double fma_clk_sm = fma_per_launch / (best * 1e-3) / (mhz * 1e6) / n_sm;
  printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"tflops\": %.3f, \"sm_mhz_in_kernel\": %.0f, "
         "\"fma_per_clk_per_sm\": %.2f}\n", name, best, tflops, mhz, fma_clk_sm);
  return 0;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int n_sm = p.multiProcessorCount;
  printf("{\"device\": \"%s\", \"sm\": %d, \"cc\": \"%d.%d\"}\n", p.name, n_sm, p.major, p.minor);
  double* out; CK(cudaMalloc(&out, sizeof(double) * n_sm * 64 * 1024));
  double h[NCONST]; for (int i = 0; i < NCONST; ++i) h[i] = 1.0 + 1e-7 * i;
  CK(cudaMemcpyToSymbol(c_tab, h, sizeof(h)));
  const int threads = 256;
  for (int bps : {4, 8}) {
    int blocks = n_sm * bps; int iters = 4096;
    char nm[64]; snprintf(nm, 64, "dfma_reg_8ch_%dblk", bps);
    timeit(nm, [&] { dfma_reg<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); },
           (double)blocks * threads * iters * 16 * 8, n_sm);
  }
  {
    int blocks = n_sm * 4; int iters = 4096;
    timeit("dfma_reg_4ch", [&] { dfma_reg<4><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); },
           (double)blocks * threads * iters * 16 * 4, n_sm);
  }
  for (int bps : {2, 4, 8}) {
    int blocks = n_sm * bps; int iters = 2048;
    char nm[64]; snprintf(nm, 64, "dmma_m8n8k4_8ch_%dblk", bps);
    // each mma: 8*8*4 = 256 FMA per warp
    timeit(nm, [&] { dmma_reg<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); },
           (double)blocks * (threads / 32) * iters * 4 * 8 * 256, n_sm);
  }
  for (int bps : {2, 4, 8}) {
    int blocks = n_sm * bps * 64; int iters = 1;
    char nm[64]; snprintf(nm, 64, "dfma_const_%dblk", bps);
    timeit(nm, [&] { dfma_const<<<blocks, threads>>>(out, iters); },
           (double)blocks * threads * NCONST, n_sm);
  }
  {
    int blocks = n_sm * 4; int iters = 1024;
    // FMA counted: DMMA 256 per warp-instr; DFMA 32 per warp-instr
    timeit("mix_dmma_only(ratio0)", [&] { mix_kernel<0><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); },
           (double)blocks * (threads / 32) * iters * 8 * 256, n_sm);
    timeit("mix_ratio2_dmma_fma_only", [&] { mix_kernel<2><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); },
           (double)blocks * (threads / 32) * iters * 8 * 256, n_sm);
    timeit("mix_ratio4_dmma_fma_only", [&] { mix_kernel<4><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); },
           (double)blocks * (threads / 32) * iters * 8 * 256, n_sm);
    timeit("mix_ratio8_dmma_fma_only", [&] { mix_kernel<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); },
           (double)blocks * (threads / 32) * iters * 8 * 256, n_sm);
  }
  {
    // 1 block of 128 threads (one warp per SMSP) per SM; cycles per DMMA per warp = latency / CH
    int blocks = n_sm; int iters = 4096;
    auto run = [&](const char* nm, auto kern, int ch) {
      timeit(nm, [&] { kern<<<blocks, 128>>>(out, iters, 1.0000001, 1e-9); },
             (double)blocks * 4 * iters * ch * 256, n_sm);
      unsigned long long clk[2];
      cudaMemcpyFromSymbol(clk, g_clk, sizeof(clk));
      printf("{\"kernel\": \"%s_cycles_per_dmma_per_warp\", \"value\": %.2f}\n", nm, (double)clk[0] / (iters * ch));
    };
    run("chain1", dmma_chain<1>, 1);
    run("chain2", dmma_chain<2>, 2);
    run("chain3", dmma_chain<3>, 3);
    run("chain4", dmma_chain<4>, 4);
    run("chain8", dmma_chain<8>, 8);
  }
  for (int bps : {4, 8}) {
    int blocks = n_sm * bps; int iters = 64;
    char nm[64]; snprintf(nm, 64, "dfma_smem_%dblk", bps);
    timeit(nm, [&] { dfma_smem<<<blocks, threads>>>(out, iters); },
           (double)blocks * threads * iters * 1024 * 4, n_sm);
  }
  return 0;
}
