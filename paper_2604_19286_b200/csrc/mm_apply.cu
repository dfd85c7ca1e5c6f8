// Matrix-free product of the assembled mass matrix with a nodal field,
//   y[g][i] = sum_slot sum_j M[g][slot][3i+j] E[wrap(g + d(slot))][j]
// as the implicit field equation uses it ((L + sum_s M_s) E = b, eq_field_eq,
// PAPER.md:77-83).  HBM-bound: the matrix (S x C x 8 B per node) is read once; E (24 B per
// node) is re-read by the (2R+1)^3 neighbours from L1/L2.
//
// One warp per node row, two rows in flight (grid-stride): lane l owns stencil slots l, l+32, ...;
// for its slot it reads the 9 (or 1) matrix values (the warp covers the contiguous row),
// gathers the neighbour's E (read-only path) and accumulates the 3 (or 1) row sums; a
// butterfly reduction leaves y[g] in lane 0.
#include "mm_internal.cuh"

namespace mm {

namespace {

__device__ __forceinline__ int wrapi(int i, int n)
{
    return i < 0 ? i + n : (i >= n ? i - n : i);
}

template <int R, int C, int U>
__device__ __forceinline__ void apply_rows(const Geo &g, const double *__restrict__ M, const double *__restrict__ E,
                                           double *__restrict__ y, int accumulate, const int64_t (&rows)[U], int lane)
{
    constexpr int W = 2 * R + 1, S = W * W * W, NV = C == 9 ? 3 : 1;
    double acc[U][NV];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < NV; ++i)
            acc[u][i] = 0.0;
#pragma unroll
    for (int s0 = 0; s0 < S; s0 += 32) {
        const int sl = s0 + lane;
        if (sl < S) {
            const int dx = sl / (W * W) - R, dy = (sl / W) % W - R, dz = sl % W - R;
            // all loads of the U rows first (memory-level parallelism), then the FMAs
            double mv[U][NV * NV], e[U][NV];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t row = rows[u] < 0 ? 0 : rows[u];
                const int gz = (int)(row % g.n2), gxy = (int)(row / g.n2), gy = gxy % g.n1, gx = gxy / g.n1;
                const int64_t nb = ((int64_t)wrapi(gx + dx, g.n0) * g.n1 + wrapi(gy + dy, g.n1)) * g.n2 +
                                   wrapi(gz + dz, g.n2);
                const double *m = M + row * (S * C) + sl * C;
#pragma unroll
                for (int k = 0; k < NV * NV; ++k)
                    mv[u][k] = __ldg(m + k);
#pragma unroll
                for (int j = 0; j < NV; ++j)
                    e[u][j] = __ldg(E + nb * NV + j);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int i = 0; i < NV; ++i)
#pragma unroll
                    for (int j = 0; j < NV; ++j)
                        acc[u][i] = fma(mv[u][NV * i + j], e[u][j], acc[u][i]);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int i = 0; i < NV; ++i)
                acc[u][i] += __shfl_xor_sync(0xffffffffu, acc[u][i], o);
        if (lane < NV && rows[u] >= 0) {
            const double v = lane == 0 ? acc[u][0] : (lane == 1 ? acc[u][NV > 1 ? 1 : 0] : acc[u][NV > 2 ? 2 : 0]);
            y[rows[u] * NV + lane] = accumulate ? y[rows[u] * NV + lane] + v : v;
        }
    }
}

// Warp per node row, U = 2 rows in flight per warp so that their matrix and field loads
// overlap (4 rows was slower for CIC: 0.63 vs 0.70 of HBM).
template <int R, int C>
__global__ void __launch_bounds__(256) k_apply(Geo g, const double *__restrict__ M, const double *__restrict__ E,
                                               double *__restrict__ y, int accumulate)
{
    constexpr int U = 2;
    const int lane = threadIdx.x & 31;
    const int64_t nrows = (int64_t)g.n0 * g.n1 * g.n2;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); row < nrows; row += U * nw) {
        int64_t rows[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
            rows[u] = row + u * nw < nrows ? row + u * nw : -1;
        apply_rows<R, C, U>(g, M, E, y, accumulate, rows, lane);
    }
}

template <int R, int C>
cudaError_t launch(const Geo &geo, const double *M, const double *E, double *y, int accumulate, cudaStream_t s)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nrows = (int64_t)geo.n0 * geo.n1 * geo.n2;
    int64_t want = (nrows + 7) / 8;
    const int64_t cap = (int64_t)sms * 8;
    k_apply<R, C><<<(unsigned)(want < cap ? want : cap), 256, 0, s>>>(geo, M, E, y, accumulate);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t apply_enqueue(const Geo &geo, int ncomp, const double *M, const double *E, double *y, int accumulate,
                          cudaStream_t s)
{
    if (geo.order == 1)
        return ncomp == 9 ? launch<1, 9>(geo, M, E, y, accumulate, s) : launch<1, 1>(geo, M, E, y, accumulate, s);
    return ncomp == 9 ? launch<2, 9>(geo, M, E, y, accumulate, s) : launch<2, 1>(geo, M, E, y, accumulate, s);
}

}  // namespace mm
