// FP64 MMA shape throughput on B200: mma.sync m8n8k4 (sm_80+) vs m16n8k4 / m16n8k8 / m16n8k16
// (sm_90+ f64 shapes).  Register-only accumulation chains, CHAINS independent accumulators per
// warp, grid = 148 x 4 CTAs of 4..16 warps.  Reports TFLOP/s (2 flops per multiply-add).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_shapes dmma_shapes.cu
// Finding (cuobjdump -sass): ptxas lowers every f64 shape to SASS DMMA.8x8x4 on sm_100a
// (m16n8k16 = 8 of them), so the larger shapes cannot raise the FP64 tensor rate.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__device__ __forceinline__ void mma1684(double (&d)[4], double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3]) : "d"(a0), "d"(a1), "d"(b));
}
__device__ __forceinline__ void mma1688(double (&d)[4], const double (&a)[4], const double (&b)[2]) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
}
__device__ __forceinline__ void mma16816(double (&d)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
               : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

template <int SHAPE, int CHAINS>
__global__ void bench(double* out, int iters, double x) {
  double acc[CHAINS][4];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c][0] = acc[c][1] = acc[c][2] = acc[c][3] = c;
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = x + i * 1e-3 + threadIdx.x * 1e-9;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = x - i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (SHAPE == 0) { double d2[2] = {acc[c][0], acc[c][1]}; mma884(d2, a[c & 7], b[c & 3]); acc[c][0] = d2[0]; acc[c][1] = d2[1]; }
      if (SHAPE == 1) mma1684(acc[c], a[0], a[1], b[0]);
      if (SHAPE == 2) { const double aa[4] = {a[0], a[1], a[2], a[3]}; const double bb[2] = {b[0], b[1]}; mma1688(acc[c], aa, bb); }
      if (SHAPE == 3) mma16816(acc[c], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 1234.5) out[threadIdx.x] = s;
}

template <int SHAPE, int CHAINS>
void run(const char* name, double macs_per_mma, int warps) {
  double* out;
  cudaMalloc(&out, 4096 * sizeof(double));
  const int iters = 4096, blocks = 148 * 4;
  bench<SHAPE, CHAINS><<<blocks, 32 * warps>>>(out, 16, 1.0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<SHAPE, CHAINS><<<blocks, 32 * warps>>>(out, iters, 1.0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double mmas = (double)blocks * warps * iters * CHAINS;
  printf("{\"shape\": \"%s\", \"chains\": %d, \"warps_per_cta\": %d, \"tflops\": %.2f, \"err\": \"%s\"}\n", name, CHAINS,
         warps, mmas * macs_per_mma * 2 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0, 4>("m8n8k4", 8 * 8 * 4, w);
    run<1, 4>("m16n8k4", 16 * 8 * 4, w);
    run<2, 4>("m16n8k8", 16 * 8 * 8, w);
    run<3, 4>("m16n8k16", 16 * 8 * 16, w);
  }
  return 0;
}
