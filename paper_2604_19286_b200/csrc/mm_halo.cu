// Slab decomposition support:
//  * ghost-plane reduction: received ghost node rows are added into the owned rows they
//    belong to (HBM-bound streaming add, 24 B per element);
//  * particle migration (NEXT-1, the "sort & communicate" stage): a stable
//    3-way partition of a rank's particles into [stay | to previous slab | to next slab] by
//    their cell along x, so that only the leavers are exchanged before the next sort.
#include "mm_internal.cuh"

namespace mm {

namespace {

__global__ void k_ghost_add(double *__restrict__ out, const double *__restrict__ recv, int64_t n)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] += __ldg(recv + i);
}

constexpr int PT = 512, PI = 4, PTILE = PT * PI;  // partition: threads, items per thread

// class of a particle: 0 stays (cell x in [x_begin, x_end)), 1 leaves through x_begin (to the
// previous slab), 2 through x_end (to the next slab); u = (c_x - x_begin) mod n0 splits the
// outside cells half-and-half between the two directions.  Cell by the IEEE quotient (R5).
__device__ __forceinline__ int slab_class(double x, double h, int n0, int xb, int xe)
{
    if (!isfinite(x) || x < 0.0 || !(x < n0 * h))
        return 0;  // left for mm_sort_by_cell to report (never clamped)
    const double c = floor(__ddiv_rn(x, h));
    int u = (int)c - xb;
    u = ((u % n0) + n0) % n0;
    const int w = xe - xb;
    if (u < w)
        return 0;
    return (u - w) < (n0 - w + 1) / 2 ? 2 : 1;
}

__device__ __forceinline__ int block_scan3(int v, int &total)
{
    __shared__ int ws[PT / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o)
            x += y;
    }
    if (lane == 31)
        ws[w] = x;
    __syncthreads();
    if (w == 0) {
        int t = lane < PT / 32 ? ws[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o)
                t += y;
        }
        if (lane < PT / 32)
            ws[lane] = t;
    }
    __syncthreads();
    total = ws[PT / 32 - 1];
    const int r = (w ? ws[w - 1] : 0) + x - v;
    __syncthreads();
    return r;
}

// pass 1: per tile counts of the three classes
__global__ void __launch_bounds__(PT) k_part_count(int64_t np, const double *__restrict__ pos, double h, int n0,
                                                   int xb, int xe, int32_t *__restrict__ tcount)
{
    __shared__ int sc[3];
    if (threadIdx.x < 3)
        sc[threadIdx.x] = 0;
    __syncthreads();
    int c3[3] = {0, 0, 0};
    const int64_t base = (int64_t)blockIdx.x * PTILE;
#pragma unroll
    for (int k = 0; k < PI; ++k) {
        const int64_t i = base + k * PT + threadIdx.x;
        if (i < np)
            ++c3[slab_class(__ldg(pos + 3 * i), h, n0, xb, xe)];
    }
#pragma unroll
    for (int c = 0; c < 3; ++c)
        if (c3[c])
            atomicAdd(&sc[c], c3[c]);
    __syncthreads();
    if (threadIdx.x < 3)
        tcount[3 * blockIdx.x + threadIdx.x] = sc[threadIdx.x];
}

// exclusive offsets of every (tile, class) in class-major order (one CTA, serial over tiles in
// chunks of PT); totals of the classes in tcount[3 ntiles .. 3 ntiles + 2]
__global__ void __launch_bounds__(PT) k_part_scan(int ntiles, int32_t *__restrict__ tcount)
{
    int carry = 0;
    for (int c = 0; c < 3; ++c) {
        for (int t0 = 0; t0 < ntiles; t0 += PT) {
            const int t = t0 + threadIdx.x;
            const int v = t < ntiles ? tcount[3 * t + c] : 0;
            int total;
            const int e = block_scan3(v, total);
            if (t < ntiles)
                tcount[3 * t + c] = carry + e;
            carry += total;
        }
        if (threadIdx.x == 0)
            tcount[3 * ntiles + c] = carry;  // inclusive end of class c
    }
}

// pass 2: stable placement (tile order, then element order inside the tile)
__global__ void __launch_bounds__(PT) k_part_place(int64_t np, const double *__restrict__ pos,
                                                   const double *__restrict__ q, const double *__restrict__ B,
                                                   double h, int n0, int xb, int xe,
                                                   const int32_t *__restrict__ toff, double *__restrict__ pos_o,
                                                   double *__restrict__ q_o, double *__restrict__ B_o)
{
    const int64_t base = (int64_t)blockIdx.x * PTILE;
    int run[3] = {toff[3 * blockIdx.x], toff[3 * blockIdx.x + 1], toff[3 * blockIdx.x + 2]};
    for (int k = 0; k < PI; ++k) {
        const int64_t i = base + k * PT + threadIdx.x;
        const int cls = i < np ? slab_class(__ldg(pos + 3 * i), h, n0, xb, xe) : 3;
        int slot = 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            int total;
            const int e = block_scan3(cls == c ? 1 : 0, total);
            if (cls == c)
                slot = run[c] + e;
            run[c] += total;
        }
        if (cls < 3) {
#pragma unroll
            for (int m = 0; m < 3; ++m)
                pos_o[3 * (int64_t)slot + m] = __ldg(pos + 3 * i + m);
            q_o[slot] = __ldg(q + i);
            if (B)
#pragma unroll
                for (int m = 0; m < 3; ++m)
                    B_o[3 * (int64_t)slot + m] = __ldg(B + 3 * i + m);
        }
    }
}

}  // namespace

int64_t partition_tmp_elems(int64_t np)
{
    return 3 * ((np + PTILE - 1) / PTILE) + 3;
}

cudaError_t partition_enqueue(const Geo &g, int64_t np, const double *pos, const double *q, const double *B,
                              double *pos_o, double *q_o, double *B_o, int32_t *tmp, cudaStream_t s)
{
    const int ntiles = (int)((np + PTILE - 1) / PTILE);
    if (ntiles == 0)
        return cudaMemsetAsync(tmp, 0, 3 * sizeof(int32_t), s);
    k_part_count<<<ntiles, PT, 0, s>>>(np, pos, g.h0, g.n0, g.x_begin, g.x_end, tmp);
    k_part_scan<<<1, PT, 0, s>>>(ntiles, tmp);
    k_part_place<<<ntiles, PT, 0, s>>>(np, pos, q, B, g.h0, g.n0, g.x_begin, g.x_end, tmp, pos_o, q_o, B_o);
    count_launch(3);
    return cudaGetLastError();
}

cudaError_t ghost_add_enqueue(double *out, const double *recv, int64_t n, cudaStream_t s)
{
    if (n <= 0)
        return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16)
        blocks = 148 * 16;
    k_ghost_add<<<(unsigned)blocks, 256, 0, s>>>(out, recv, n);
    count_launch();
    return cudaGetLastError();
}

}  // namespace mm
