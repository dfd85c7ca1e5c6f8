// Microbenchmarks that set the roofline denominators this build reports
// (DESIGN.md §Roofline): FP64 DMMA 8x8x4 and DFMA peaks, global FP64 RED
// throughput for the deposit pattern, HBM copy.  Not part of the hot path;
// built as libmm_probe.so.  Each entry point returns the kernel time in ms
// measured with CUDA events (<0 on error).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

template <int CH>
__global__ void k_dmma(int iters, double *sink, double seed)
{
    double acc[CH][2];
#pragma unroll
    for (int c = 0; c < CH; ++c)
        acc[c][0] = acc[c][1] = 0.0;
    double a = seed * (threadIdx.x + 1), b = seed + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            dmma(acc[c][0], acc[c][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c)
        s += acc[c][0] + acc[c][1];
    if (s == 12345.678)
        sink[threadIdx.x] = s;
}

template <int CH>
__global__ void k_dfma(int iters, double *sink, double seed)
{
    double acc[CH];
    double a = seed * (threadIdx.x + 1), b = seed + threadIdx.x;
#pragma unroll
    for (int c = 0; c < CH; ++c)
        acc[c] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            acc[c] = fma(acc[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c)
        s += acc[c];
    if (s == 12345.678)
        sink[threadIdx.x] = s;
}

// DMMA with interleaved DFMAs (ratio per DMMA) — do they share a pipe?
template <int CH, int NF>
__global__ void k_mixed(int iters, double *sink, double seed)
{
    double acc[CH][2], f[NF];
#pragma unroll
    for (int c = 0; c < CH; ++c)
        acc[c][0] = acc[c][1] = 0.0;
#pragma unroll
    for (int c = 0; c < NF; ++c)
        f[c] = c;
    double a = seed * (threadIdx.x + 1), b = seed + threadIdx.x;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c)
            dmma(acc[c][0], acc[c][1], a, b);
#pragma unroll
        for (int c = 0; c < NF; ++c)
            f[c] = fma(f[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c)
        s += acc[c][0] + acc[c][1];
#pragma unroll
    for (int c = 0; c < NF; ++c)
        s += f[c];
    if (s == 12345.678)
        sink[threadIdx.x] = s;
}

// Global FP64 reductions: each warp issues `per_warp` rounds; round r of warp w
// targets a pseudo-random 256-B aligned line (contig=1: 32 lanes -> 32
// consecutive doubles, i.e. 8 sectors) or a random double per lane (contig=0).
__global__ void k_red(double *buf, int64_t nelem, int per_warp, int contig, uint32_t seed)
{
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    uint32_t x = (uint32_t)(warp * 2654435761u) ^ seed;
    for (int r = 0; r < per_warp; ++r) {
        x = x * 1664525u + 1013904223u;
        uint32_t y = contig ? x : (x ^ (lane * 0x9E3779B9u)) * 2246822519u;
        int64_t base = contig ? ((int64_t)(y % (uint32_t)(nelem / 32)) * 32 + lane)
                              : (int64_t)(y % (uint32_t)nelem);
        atomicAdd(buf + base, 1.0);
    }
}

// The order-1 assembly's batch loop in isolation: per batch one LDS of w, the 9 s values
// (LDS.128 pairs), 9 DMUL (A = s w) and 9 DMMA; no prep, no deposit.  Shows what DMMA
// utilisation the DMUL -> DMMA interleave itself allows.
__global__ void k_batch(int iters, double *sink)
{
    __shared__ __align__(16) double sw[8][8 * 36];
    __shared__ __align__(16) double ss[8][32 * 10];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = lane; i < 8 * 36; i += 32)
        sw[warp][i] = 1.0 + 1e-3 * i;
    for (int i = lane; i < 32 * 10; i += 32)
        ss[warp][i] = 0.5 + 1e-3 * i;
    __syncwarp();
    double acc[9][2];
#pragma unroll
    for (int c = 0; c < 9; ++c)
        acc[c][0] = acc[c][1] = 0.0;
    const double *wrow = sw[warp] + (lane >> 2) * 36 + (lane & 3);
    const double *srow = ss[warp] + (lane & 3) * 10;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int kb = 0; kb < 32; kb += 4) {
            const double w = wrow[kb];
            const double *sp = srow + kb * 10;
#pragma unroll
            for (int c = 0; c < 8; c += 2) {
                const double2 sv = *reinterpret_cast<const double2 *>(sp + c);
                dmma(acc[c][0], acc[c][1], sv.x * w, w);
                dmma(acc[c + 1][0], acc[c + 1][1], sv.y * w, w);
            }
            dmma(acc[8][0], acc[8][1], sp[8] * w, w);
        }
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < 9; ++c)
        s += acc[c][0] + acc[c][1];
    if (s == 12345.678)
        sink[threadIdx.x] = s;
}

// tcgen05 TF32 peak: one thread per CTA issues back-to-back tcgen05.mma kind::tf32 (M = 128,
// N = 256, K = 8) from two 128-B-swizzled K-major smem tiles (contents irrelevant) into TMEM,
// `iters` x 4 K-steps, then one commit; the CTA waits on the mbarrier.  FLOPs per MMA =
// 2 x 128 x 256 x 8.  (The TF32 roofline denominator the north_star asks for.)
__device__ __forceinline__ uint32_t p_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) k_tf32_mma(int iters, double *sink)
{
    extern __shared__ __align__(1024) unsigned char psm[];
    unsigned char *A = psm, *B = psm + 128 * 128;  // A: 128 rows x 128 B, B: 256 rows x 128 B
    __shared__ uint64_t bar;
    __shared__ uint32_t taddr;
    const int tid = threadIdx.x;
    for (int i = tid; i < (128 + 256) * 128 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(psm)[i] = 0x3f800000u ^ (uint32_t)(i & 0xff);
    if (tid == 0)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(p_smem_u32(&bar)) : "memory");
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(p_smem_u32(&taddr))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = taddr;
    if (tid == 0) {
        auto desc = [](uint32_t a) {
            return ((uint64_t)(a >> 4) & 0x3FFFull) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
                   (1ull << 46) | (2ull << 61);
        };
        const uint64_t dA = desc(p_smem_u32(A)), dB = desc(p_smem_u32(B));
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(256 >> 3) << 17) |
                               ((uint32_t)(128 >> 4) << 24);
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint32_t acc = (it > 0 || ks > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                    "l"(dA + 2 * ks), "l"(dB + 2 * ks), "r"(idesc), "r"(acc)
                    : "memory");
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         p_smem_u32(&bar))
                     : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred p;\n\tW_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(p_smem_u32(&bar))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((32u * (tid >> 5)) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (v == 0x12345678u)
        sink[tid] = (double)v;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

__global__ void k_copy(const double4 *__restrict__ a, double4 *__restrict__ b, int64_t n)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        b[i] = a[i];
}

template <typename F>
float timed(F f)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    f();  // warm-up
    cudaEventRecord(e0);
    f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = -1.f;
    if (cudaGetLastError() == cudaSuccess)
        cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return ms;
}

}  // namespace

extern "C" {

// FP64 flops = blocks * threads/32 * iters * 8 chains * 512
float probe_dmma(int blocks, int threads, int iters, double *sink)
{
    return timed([&] { k_dmma<8><<<blocks, threads>>>(iters, sink, 1.0000001); });
}

// FP64 flops = blocks * threads * iters * 8 chains * 2
float probe_dfma(int blocks, int threads, int iters, double *sink)
{
    return timed([&] { k_dfma<8><<<blocks, threads>>>(iters, sink, 1.0000001); });
}

// 8 DMMA + 8 DFMA (per lane) per iteration
float probe_mixed(int blocks, int threads, int iters, double *sink)
{
    return timed([&] { k_mixed<8, 8><<<blocks, threads>>>(iters, sink, 1.0000001); });
}

// REDs = blocks * threads * per_warp
float probe_red(double *buf, int64_t nelem, int blocks, int threads, int per_warp, int contig)
{
    return timed([&] { k_red<<<blocks, threads>>>(buf, nelem, per_warp, contig, 12345u); });
}

// DMMA flops = blocks * 8 warps * iters * 8 batches * 9 * 512  (blockDim = 256)
float probe_batch(int blocks, int iters, double *sink)
{
    return timed([&] { k_batch<<<blocks, 256>>>(iters, sink); });
}

// TF32 flops = blocks * iters * 4 * 2 * 128 * 256 * 8  (one CTA per SM)
float probe_tf32(int blocks, int iters, double *sink)
{
    const int smem = (128 + 256) * 128;
    if (cudaFuncSetAttribute(k_tf32_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return -1.f;
    return timed([&] { k_tf32_mma<<<blocks, 128, smem>>>(iters, sink); });
}

// bytes = 2 * n4 * 32
float probe_copy(const double *a, double *b, int64_t n4)
{
    return timed([&] {
        k_copy<<<148 * 8, 256>>>(reinterpret_cast<const double4 *>(a), reinterpret_cast<double4 *>(b), n4);
    });
}

}  // extern "C"
