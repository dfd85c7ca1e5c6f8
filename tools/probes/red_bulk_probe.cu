// Probe (diagnostics): FP64 reduction throughput into L2/HBM, per element (REDG.F64, one warp
// instruction per 26-double run) vs bulk (cp.reduce.async.bulk .add.f64 of 208 B from shared
// memory), runs at random 16-B aligned positions of a 2 GB array.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

__global__ void k_red(double *out, int64_t nruns_space, int iters)
{
    const int lane = threadIdx.x & 31;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int i = 0; i < iters; ++i) {
        const int64_t r = hash(w * 7919 + i * 104729) % nruns_space;
        double *p = out + r * 26;
        if (lane < 26)
            asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p + lane), "d"(1.0) : "memory");
    }
}

__global__ void k_bulk(double *out, int64_t nruns_space, int iters)
{
    __shared__ __align__(128) double buf[8][32];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (lane < 26)
        buf[wl][lane] = 1.0;
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    for (int i = 0; i < iters; ++i) {
        const int64_t r = hash(w * 7919 + i * 104729) % nruns_space;
        double *p = out + r * 26;
        if (lane == 0)
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 208;" ::"l"(p),
                         "r"((uint32_t)__cvta_generic_to_shared(&buf[wl][0]))
                         : "memory");
    }
    if (lane == 0) {
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
}

int main()
{
    const int64_t n = (int64_t)256 << 20;  // 2 GB of doubles
    double *out;
    cudaMalloc(&out, n * 8);
    cudaMemset(out, 0, n * 8);
    const int64_t runs = n / 26;
    const int blocks = 148 * 8, threads = 256, iters = 64;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
        for (int mode = 0; mode < 2; ++mode) {
            cudaEventRecord(a);
            if (mode == 0)
                k_red<<<blocks, threads>>>(out, runs, iters);
            else
                k_bulk<<<blocks, threads>>>(out, runs, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double elems = (double)blocks * (threads / 32) * iters * 26;
            printf("%s: %.3f ms, %.1f G element-adds/s (%s)\n", mode ? "bulk 208B" : "REDG.F64 x26", ms,
                   elems / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
