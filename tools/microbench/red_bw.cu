// fp64 scatter-add throughput on B200: how many doubles per second the L2 can reduce for
// the access patterns of the apply kernels.
//   scatter   : every lane RED.ADD.F64 to an independent pseudo-random double (CG gather/scatter)
//   group4    : 4 consecutive lanes hit one 32 B sector (4 doubles), sector random
//   cell10    : lanes 0..9 / 16..25 hit the 10 contiguous doubles of a random DG cell (P2 side)
//   bulk10    : the same 80 B per cell reduced by ONE cp.reduce.async.bulk.add.f64 from shared
//   bulk20    : 160 B per cell (DG P3 side) by one bulk reduce
//   store10   : plain stores of the cell10 pattern (bandwidth reference)
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o red_bw red_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// ops = doubles reduced in total
__global__ void k_scatter(double* y, uint32_t n, int iters) {
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
        uint32_t a = hash32(t * 977u + i) % n;
        atomicAdd(y + a, 1.0);
    }
}

__global__ void k_group4(double* y, uint32_t n, int iters) {
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t g = t >> 2, l = t & 3;
    for (int i = 0; i < iters; ++i) {
        uint32_t s = hash32(g * 977u + i) % (n / 4);
        atomicAdd(y + 4 * s + l, 1.0);
    }
}

template <int W>
__global__ void k_cell(double* y, uint32_t ncell, int iters, int store) {
    // each half-warp handles one cell of W doubles (W <= 16)
    uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t g = t >> 4, l = t & 15;
    for (int i = 0; i < iters; ++i) {
        uint32_t c = hash32(g * 977u + i) % ncell;
        if (l < W) {
            if (store) y[(size_t)c * W + l] = 1.0;
            else atomicAdd(y + (size_t)c * W + l, 1.0);
        }
    }
}

template <int W>
__global__ void k_bulk(double* y, uint32_t ncell, int iters) {
    // one warp = 2 cells per iteration; the W-double rows are staged in shared memory and reduced
    // into global memory with one cp.reduce.async.bulk per cell
    __shared__ __align__(128) double buf[8][4][2][W];  // [warp][ring][cell][W]
    int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int i = 0; i < iters; ++i) {
        int r = i & 3;
        if (i >= 3 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
        __syncwarp();
        for (int k = lane; k < 2 * W; k += 32) (&buf[w][r][0][0])[k] = 1.0;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane < 2) {
            uint32_t c = hash32((2 * gw + lane) * 977u + i) % ncell;
            double* dst = y + (size_t)c * W;
            uint32_t src = (uint32_t)__cvta_generic_to_shared(&buf[w][r][lane][0]);
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;"
                         :: "l"(dst), "r"(src), "r"(W * 8) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
    }
    if (lane < 2) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const uint32_t n = 16u << 20;  // 16 Mi doubles = 128 MB (about L2 size); also test 1 Mi
    double* y;
    cudaMalloc(&y, (size_t)64 << 20 << 3);
    cudaMemset(y, 0, (size_t)64 << 20 << 3);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = 148 * 8, threads = 256, iters = 64;
    const double threads_total = (double)blocks * threads;
    uint32_t sizes[3] = {1u << 20, n, 64u << 20};
    for (uint32_t sz : sizes) {
        auto run = [&](const char* name, double ops, auto launch) {
            for (int w = 0; w < 3; ++w) launch();
            cudaEventRecord(e0);
            const int reps = 10;
            for (int r = 0; r < reps; ++r) launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double s = ms * 1e-3 / reps;
            printf("{\"pattern\": \"%s\", \"vector_mb\": %.1f, \"us\": %.2f, \"gdoubles_per_s\": %.1f, \"err\": \"%s\"}\n",
                   name, sz * 8.0 / 1e6, s * 1e6, ops / s * 1e-9, cudaGetErrorString(cudaGetLastError()));
        };
        run("scatter", threads_total * iters, [&] { k_scatter<<<blocks, threads>>>(y, sz, iters); });
        run("group4", threads_total * iters, [&] { k_group4<<<blocks, threads>>>(y, sz, iters); });
        run("cell10_red", threads_total / 16 * 10 * iters, [&] { k_cell<10><<<blocks, threads>>>(y, sz / 10, iters, 0); });
        run("cell10_store", threads_total / 16 * 10 * iters, [&] { k_cell<10><<<blocks, threads>>>(y, sz / 10, iters, 1); });
        run("cell16_red", threads_total / 16 * 16 * iters, [&] { k_cell<16><<<blocks, threads>>>(y, sz / 16, iters, 0); });
        run("bulk10", threads_total / 16 * 10 * iters, [&] { k_bulk<10><<<blocks, threads>>>(y, sz / 10, iters); });
        run("bulk20", threads_total / 16 * 20 * iters, [&] { k_bulk<20><<<blocks, threads>>>(y, sz / 20, iters); });
        run("bulk16", threads_total / 16 * 16 * iters, [&] { k_bulk<16><<<blocks, threads>>>(y, sz / 16, iters); });
    }
    return 0;
}
