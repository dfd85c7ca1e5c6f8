// Particle binning for the mass-matrix assembly: locate + key, histogram,
// K-padded scan, stable placement, per-bin fix-up, record scatter.
//
// PAPER.md:228   "We assume that particles have been sorted by cell"
// PAPER.md:242   batches of K_t particles, "the last batch zero-padded"
// PAPER.md:290   eq_group_partition: particles grouped by identical support
// DESIGN.md R5   u = x/h (IEEE RN division), c = floor(u), xi = u - c
// DESIGN.md R12  bin = support-window base node, axis 0 local & unwrapped
// DESIGN.md R13  pad slots: perm = -1, record all zeros
//
// Pipeline (one stream, no host sync until the very end):
//   k_key      coalesced over particles: validate, key, rank = atomicAdd(count[key])
//   k_scan_*   padded exclusive scan of count -> seg_begin
//   k_place    perm[seg_begin[key] + rank] = p        (order inside a bin arbitrary)
//   k_fix_*    per bin: sort its perm slice ascending (=> STABLE), dest[perm[i]] = i,
//              write pad slots; warp path (<= 1024), CTA path (<= 16384), huge path
//   k_scatter  coalesced over particles: rec[dest[p]] = {xi, q, B, 0} (64-B records)
#include <climits>

#include "mm_internal.cuh"

namespace mm {

namespace {

__device__ __forceinline__ int32_t wrapi(int32_t i, int32_t n)
{
    return i < 0 ? i + n : (i >= n ? i - n : i);
}

struct Located {
    double xi[3];
    int32_t c[3];
    int err;
};

__device__ __forceinline__ Located locate(const Geo &g, double x0, double x1, double x2)
{
    Located L;
    L.err = 0;
    const double x[3] = {x0, x1, x2};
    const double h[3] = {g.h0, g.h1, g.h2};
#pragma unroll
    for (int mu = 0; mu < 3; ++mu) {
        if (!isfinite(x[mu])) {
            L.err |= ERR_NONFINITE;
            L.xi[mu] = 0.0;
            L.c[mu] = 0;
            continue;
        }
        double u = __ddiv_rn(x[mu], h[mu]);
        double c = floor(u);
        L.xi[mu] = u - c;
        double lo = mu == 0 ? (double)g.x_begin : 0.0;
        double hi = mu == 0 ? (double)g.x_end : (double)(mu == 1 ? g.n1 : g.n2);
        if (!(c >= lo && c < hi)) {
            L.err |= ERR_DOMAIN;
            L.c[mu] = 0;
        } else {
            L.c[mu] = (int32_t)c;
        }
    }
    return L;
}

__global__ void k_key(Geo g, int64_t np, const double *__restrict__ pos, const double *__restrict__ q,
                      const double *__restrict__ B, uint32_t *__restrict__ key,
                      int32_t *__restrict__ rank, int32_t *__restrict__ count,
                      int32_t *__restrict__ status)
{
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np)
        return;
    Located L = locate(g, pos[3 * p], pos[3 * p + 1], pos[3 * p + 2]);
    int err = L.err;
    if (!isfinite(q[p]))
        err |= ERR_NONFINITE;
    if (B && !(isfinite(B[3 * p]) && isfinite(B[3 * p + 1]) && isfinite(B[3 * p + 2])))
        err |= ERR_NONFINITE;
    if (err) {
        atomicOr(&status[ST_ERR], err);
        key[p] = 0xffffffffu;
        return;
    }
    int32_t b[3];
#pragma unroll
    for (int mu = 0; mu < 3; ++mu)
        b[mu] = (g.order == 1) ? 0 : (L.xi[mu] >= 0.5 ? 0 : -1);  // PAPER.md:168, R4
    int32_t bx = L.c[0] + b[0] - g.x_begin + (g.order - 1);
    int32_t by = wrapi(L.c[1] + b[1], g.n1);
    int32_t bz = wrapi(L.c[2] + b[2], g.n2);
    uint32_t k = (uint32_t)(((int64_t)bx * g.n1 + by) * g.n2 + bz);
    key[p] = k;
    rank[p] = atomicAdd(&count[k], 1);
}

// ---- K-padded exclusive scan ----------------------------------------------
constexpr int SCAN_T = 1024, SCAN_I = 4, SCAN_TILE = SCAN_T * SCAN_I;

__device__ __forceinline__ int block_excl_scan(int v, int &total)
{
    __shared__ int wsum[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o)
            x += y;
    }
    if (lane == 31)
        wsum[warp] = x;
    __syncthreads();
    if (warp == 0) {
        int w = lane < nw ? wsum[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o)
                w += y;
        }
        wsum[lane] = w;
    }
    __syncthreads();
    int pre = warp ? wsum[warp - 1] : 0;
    total = wsum[nw - 1];
    __syncthreads();
    return pre + x - v;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_local(const int32_t *__restrict__ count, int64_t nbins,
                                                       int k_pad, int32_t *__restrict__ seg_begin,
                                                       int32_t *__restrict__ bsum)
{
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE + (int64_t)threadIdx.x * SCAN_I;
    int v[SCAN_I], s = 0;
#pragma unroll
    for (int j = 0; j < SCAN_I; ++j) {
        int64_t i = base + j;
        int c = i < nbins ? count[i] : 0;
        v[j] = (c + k_pad - 1) / k_pad * k_pad;
        s += v[j];
    }
    int total;
    int pre = block_excl_scan(s, total);
#pragma unroll
    for (int j = 0; j < SCAN_I; ++j) {
        int64_t i = base + j;
        if (i < nbins)
            seg_begin[i] = pre;
        pre += v[j];
    }
    if (threadIdx.x == 0)
        bsum[blockIdx.x] = total;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_top(int32_t *__restrict__ bsum, int nblk,
                                                     int32_t *__restrict__ seg_end,
                                                     int32_t *__restrict__ status)
{
    int carry = 0;
    for (int c0 = 0; c0 < nblk; c0 += SCAN_TILE) {
        int v[SCAN_I], s = 0;
#pragma unroll
        for (int j = 0; j < SCAN_I; ++j) {
            int i = c0 + threadIdx.x * SCAN_I + j;
            v[j] = i < nblk ? bsum[i] : 0;
            s += v[j];
        }
        int total;
        int pre = block_excl_scan(s, total) + carry;
#pragma unroll
        for (int j = 0; j < SCAN_I; ++j) {
            int i = c0 + threadIdx.x * SCAN_I + j;
            if (i < nblk)
                bsum[i] = pre;
            pre += v[j];
        }
        carry += total;
    }
    if (threadIdx.x == 0) {
        *seg_end = carry;
        status[ST_NPAD] = carry;
    }
}

__global__ void __launch_bounds__(SCAN_T) k_scan_add(int32_t *__restrict__ seg_begin, int64_t nbins,
                                                     const int32_t *__restrict__ bsum)
{
    int off = bsum[blockIdx.x];
    int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
    for (int j = threadIdx.x; j < SCAN_TILE; j += SCAN_T) {
        int64_t i = base + j;
        if (i < nbins)
            seg_begin[i] += off;
    }
}

__global__ void k_place(int64_t np, const uint32_t *__restrict__ key, const int32_t *__restrict__ rank,
                        const int32_t *__restrict__ seg_begin, int32_t *__restrict__ perm)
{
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np)
        return;
    uint32_t k = key[p];
    if (k == 0xffffffffu)
        return;
    perm[seg_begin[k] + rank[p]] = (int32_t)p;
}

// ---- per-bin fix-up: ascending order of original indices == stable sort ----
constexpr int FIX_WARPS = 8;

__device__ __forceinline__ void zero_pads(int32_t *perm, double *rec, int64_t from, int64_t to, int tid,
                                          int nthr)
{
    for (int64_t i = from + tid; i < to; i += nthr) {
        perm[i] = -1;
        double2 z = make_double2(0.0, 0.0);
        double2 *r = reinterpret_cast<double2 *>(rec + 8 * i);
        r[0] = z;
        r[1] = z;
        r[2] = z;
        r[3] = z;
    }
}

__global__ void __launch_bounds__(FIX_WARPS * 32) k_fix_warp(int64_t nbins, const int32_t *__restrict__ count,
                                                             const int32_t *__restrict__ seg_begin,
                                                             int32_t *__restrict__ perm, int32_t *__restrict__ dest,
                                                             double *__restrict__ rec, int32_t *__restrict__ mid_list,
                                                             int32_t *__restrict__ huge_list,
                                                             int32_t *__restrict__ status)
{
    __shared__ int32_t buf[FIX_WARPS][WARP_BIN_MAX];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t *s = buf[w];
    const int64_t nwarps = (int64_t)gridDim.x * FIX_WARPS;
    for (int64_t bin = (int64_t)blockIdx.x * FIX_WARPS + w; bin < nbins; bin += nwarps) {
        const int n = count[bin];
        const int64_t b = seg_begin[bin], e = seg_begin[bin + 1];
        zero_pads(perm, rec, b + n, e, lane, 32);
        if (n == 0)
            continue;
        if (n > WARP_BIN_MAX) {
            if (lane == 0) {
                if (n > CTA_BIN_MAX)
                    huge_list[atomicAdd(&status[ST_NHUGE], 1)] = (int32_t)bin;
                else
                    mid_list[atomicAdd(&status[ST_NMID], 1)] = (int32_t)bin;
            }
            continue;
        }
        if (n == 1) {
            if (lane == 0)
                dest[perm[b]] = (int32_t)b;
            continue;
        }
        int N = 32;
        while (N < n)
            N <<= 1;
        for (int i = lane; i < N; i += 32)
            s[i] = i < n ? perm[b + i] : INT_MAX;
        __syncwarp();
        for (int k = 2; k <= N; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = lane; i < N; i += 32) {
                    int ixj = i ^ j;
                    if (ixj > i) {
                        int32_t x = s[i], y = s[ixj];
                        bool up = (i & k) == 0;
                        if ((x > y) == up) {
                            s[i] = y;
                            s[ixj] = x;
                        }
                    }
                }
                __syncwarp();
            }
        }
        for (int i = lane; i < n; i += 32) {
            int32_t v = s[i];
            perm[b + i] = v;
            dest[v] = (int32_t)(b + i);
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(1024) k_fix_cta(const int32_t *__restrict__ count,
                                                  const int32_t *__restrict__ seg_begin,
                                                  int32_t *__restrict__ perm, int32_t *__restrict__ dest,
                                                  const int32_t *__restrict__ mid_list,
                                                  const int32_t *__restrict__ status)
{
    extern __shared__ int32_t s[];
    const int nmid = status[ST_NMID];
    for (int it = blockIdx.x; it < nmid; it += gridDim.x) {
        const int32_t bin = mid_list[it];
        const int n = count[bin];
        const int64_t b = seg_begin[bin];
        int N = 1024;
        while (N < n)
            N <<= 1;
        for (int i = threadIdx.x; i < N; i += blockDim.x)
            s[i] = i < n ? perm[b + i] : INT_MAX;
        __syncthreads();
        for (int k = 2; k <= N; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < N; i += blockDim.x) {
                    int ixj = i ^ j;
                    if (ixj > i) {
                        int32_t x = s[i], y = s[ixj];
                        bool up = (i & k) == 0;
                        if ((x > y) == up) {
                            s[i] = y;
                            s[ixj] = x;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            int32_t v = s[i];
            perm[b + i] = v;
            dest[v] = (int32_t)(b + i);
        }
        __syncthreads();
    }
}

// Bins with more than CTA_BIN_MAX particles: a stable compaction of the
// particle list (O(np) per such bin; only degenerate inputs reach it).
__global__ void __launch_bounds__(1024) k_fix_huge(int64_t np, const uint32_t *__restrict__ key,
                                                   const int32_t *__restrict__ seg_begin,
                                                   int32_t *__restrict__ perm, int32_t *__restrict__ dest,
                                                   const int32_t *__restrict__ huge_list,
                                                   const int32_t *__restrict__ status)
{
    const int nhuge = status[ST_NHUGE];
    for (int it = blockIdx.x; it < nhuge; it += gridDim.x) {
        const uint32_t bin = (uint32_t)huge_list[it];
        int64_t out = seg_begin[bin];
        for (int64_t c0 = 0; c0 < np; c0 += blockDim.x) {
            int64_t p = c0 + threadIdx.x;
            int f = (p < np && key[p] == bin) ? 1 : 0;
            int total;
            int pre = block_excl_scan(f, total);
            if (f) {
                perm[out + pre] = (int32_t)p;
                dest[p] = (int32_t)(out + pre);
            }
            out += total;
        }
    }
}

__global__ void k_scatter(Geo g, int64_t np, const double *__restrict__ pos, const double *__restrict__ q,
                          const double *__restrict__ B, const uint32_t *__restrict__ key,
                          const int32_t *__restrict__ dest, double *__restrict__ rec)
{
    int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np || key[p] == 0xffffffffu)
        return;
    Located L = locate(g, pos[3 * p], pos[3 * p + 1], pos[3 * p + 2]);
    double2 *r = reinterpret_cast<double2 *>(rec + 8 * (int64_t)dest[p]);
    r[0] = make_double2(L.xi[0], L.xi[1]);
    if (B) {
        r[1] = make_double2(L.xi[2], q[p]);
        r[2] = make_double2(B[3 * p], B[3 * p + 1]);
        r[3] = make_double2(B[3 * p + 2], 0.0);
    } else {
        r[1] = make_double2(L.xi[2], q[p]);
        r[2] = make_double2(0.0, 0.0);
        r[3] = make_double2(0.0, 0.0);
    }
}

inline unsigned blocks_for(int64_t n, int t)
{
    return (unsigned)((n + t - 1) / t);
}

}  // namespace

int64_t scan_tmp_elems(int64_t nbins)
{
    return (nbins + SCAN_TILE - 1) / SCAN_TILE + 1;
}

cudaError_t sort_enqueue(const Geo &geo, const SortBufs &b, cudaStream_t s)
{
    cudaError_t e;
    if ((e = cudaMemsetAsync(b.count, 0, sizeof(int32_t) * (size_t)b.nbins, s)))
        return e;
    if ((e = cudaMemsetAsync(b.status, 0, sizeof(int32_t) * ST_WORDS, s)))
        return e;
    const int T = 256;
    if (b.np > 0) {
        k_key<<<blocks_for(b.np, T), T, 0, s>>>(geo, b.np, b.pos, b.q, b.B, b.key, b.rank, b.count, b.status);
        count_launch();
    }
    const int nblk = (int)((b.nbins + SCAN_TILE - 1) / SCAN_TILE);
    k_scan_local<<<nblk, SCAN_T, 0, s>>>(b.count, b.nbins, b.k_pad, b.seg_begin, b.scan_tmp);
    k_scan_top<<<1, SCAN_T, 0, s>>>(b.scan_tmp, nblk, b.seg_begin + b.nbins, b.status);
    k_scan_add<<<nblk, SCAN_T, 0, s>>>(b.seg_begin, b.nbins, b.scan_tmp);
    count_launch(3);
    if (b.np > 0) {
        k_place<<<blocks_for(b.np, T), T, 0, s>>>(b.np, b.key, b.rank, b.seg_begin, b.perm);
        count_launch();
    }
    {
        int64_t want = (b.nbins + FIX_WARPS - 1) / FIX_WARPS;
        unsigned grid = (unsigned)(want < 148 * 16 ? want : 148 * 16);
        if (grid < 1)
            grid = 1;
        k_fix_warp<<<grid, FIX_WARPS * 32, 0, s>>>(b.nbins, b.count, b.seg_begin, b.perm, b.rank, b.rec,
                                                   b.mid_list, b.huge_list, b.status);
        count_launch();
    }
    if (b.np > WARP_BIN_MAX) {
        static bool attr = false;
        if (!attr) {
            if ((e = cudaFuncSetAttribute(k_fix_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          CTA_BIN_MAX * 4)))
                return e;
            attr = true;
        }
        k_fix_cta<<<148, 1024, CTA_BIN_MAX * 4, s>>>(b.count, b.seg_begin, b.perm, b.rank, b.mid_list, b.status);
        count_launch();
    }
    if (b.np > CTA_BIN_MAX) {
        k_fix_huge<<<8, 1024, 0, s>>>(b.np, b.key, b.seg_begin, b.perm, b.rank, b.huge_list, b.status);
        count_launch();
    }
    if (b.np > 0) {
        k_scatter<<<blocks_for(b.np, T), T, 0, s>>>(geo, b.np, b.pos, b.q, b.B, b.key, b.rank, b.rec);
        count_launch();
    }
    return cudaGetLastError();
}

}  // namespace mm
