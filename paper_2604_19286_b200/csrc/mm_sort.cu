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
//   k_key      coalesced over particles: validate, key, rank = atomicAdd(count[key]) (one
//              atomic per run of equal keys in consecutive lanes)
//   k_scan_*   padded exclusive scan of count -> seg_begin
//   k_place    perm[seg_begin[key] + rank] = p        (order inside a bin arbitrary)
//   k_fix_*    per bin: sort its perm slice ascending (=> STABLE), dest[perm[i]] = i,
//              write pad slots; warp path (<= 1024), CTA path (<= 16384), huge path
//   k_scatter  coalesced over particles: rec[dest[p]] = {xi, q, B, 0} (64-B records;
//              32-B {xi, q} for a scalar-only handle sorted without B)
#include <climits>
#include <cstdio>
#include <cstdlib>

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
    const double ih[3] = {g.ih0, g.ih1, g.ih2};
#pragma unroll
    for (int mu = 0; mu < 3; ++mu) {
        if (!isfinite(x[mu])) {
            L.err |= ERR_NONFINITE;
            L.xi[mu] = 0.0;
            L.c[mu] = 0;
            continue;
        }
        // IEEE RN division (bit-exact binning); for a power-of-two spacing the product with
        // the exact reciprocal is the same correctly rounded quotient
        double u = g.h_pow2 ? x[mu] * ih[mu] : __ddiv_rn(x[mu], h[mu]);
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

__device__ __forceinline__ double4 ld256(const double *p)
{
    double4 v;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p));
    return v;
}

// Load the 3-vectors of particles p0..p0+3 ([np][3] FP64); VEC: three 256-bit loads.
template <bool VEC>
__device__ __forceinline__ void load_vec3x4(const double *__restrict__ a, int64_t p0, int64_t np, double v[12])
{
    if (VEC && p0 + 4 <= np) {
        double4 x = ld256(a + 3 * p0), y = ld256(a + 3 * p0 + 4), z = ld256(a + 3 * p0 + 8);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
        v[8] = z.x; v[9] = z.y; v[10] = z.z; v[11] = z.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int m = 0; m < 3; ++m)
                v[3 * j + m] = (p0 + j < np) ? a[3 * (p0 + j) + m] : 0.0;
    }
}

// FP32 variant (mixed-precision inputs): three 16-B loads, widened exactly.
template <bool VEC>
__device__ __forceinline__ void load_vec3x4(const float *__restrict__ a, int64_t p0, int64_t np, double v[12])
{
    if (VEC && p0 + 4 <= np) {
        const float4 *a4 = reinterpret_cast<const float4 *>(a + 3 * p0);
        const float4 x = __ldg(a4), y = __ldg(a4 + 1), z = __ldg(a4 + 2);
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
        v[4] = y.x; v[5] = y.y; v[6] = y.z; v[7] = y.w;
        v[8] = z.x; v[9] = z.y; v[10] = z.z; v[11] = z.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int m = 0; m < 3; ++m)
                v[3 * j + m] = (p0 + j < np) ? (double)a[3 * (p0 + j) + m] : 0.0;
    }
}

__device__ __forceinline__ uint32_t bin_of(const Geo &g, const Located &L)
{
    int32_t b[3];
#pragma unroll
    for (int mu = 0; mu < 3; ++mu)
        b[mu] = (g.order == 1) ? 0 : (L.xi[mu] >= 0.5 ? 0 : -1);  // PAPER.md:168, R4
    int32_t bx = L.c[0] + b[0] - g.x_begin + (g.order - 1);
    int32_t by = wrapi(L.c[1] + b[1], g.n1);
    int32_t bz = wrapi(L.c[2] + b[2], g.n2);
    return (uint32_t)(((int64_t)bx * g.n1 + by) * g.n2 + bz);
}

// Warp-strided particles (round j: particles base + 32 j + lane, coalesced 768-B position
// loads), 4 rounds per warp with all loads issued first.  Runs of equal keys in consecutive
// lanes share ONE atomicAdd (the run head adds the run length; the lanes take consecutive
// ranks): on cell-ordered input (the PIC regime) a warp's 32 particles fall into 1-3 bins, so
// this removes the same-address atomic serialisation, and the ranks follow the particle index
// inside each run (the per-bin fix-up then finds most slices already ascending).  On shuffled
// input every lane is its own run (one atomic each, as before).
constexpr int KEY_R = 4;  // rounds of 32 particles per warp (8 spills and is slower on shuffled input)

template <typename TP>
__global__ void __launch_bounds__(256, 4) k_key(Geo g, int64_t np, const TP *__restrict__ pos,
                                                uint32_t *__restrict__ key, int32_t *__restrict__ rank,
                                                int32_t *__restrict__ count, int32_t *__restrict__ status)
{
    const int lane = threadIdx.x & 31;
    const int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (32 * KEY_R);
    if (base >= np)
        return;
    double x[KEY_R][3];
#pragma unroll
    for (int j = 0; j < KEY_R; ++j) {
        const int64_t p = base + 32 * j + lane;
#pragma unroll
        for (int m = 0; m < 3; ++m)
            x[j][m] = p < np ? (double)__ldg(pos + 3 * p + m) : 0.0;
    }
    int err = 0;
    const unsigned below = (2u << lane) - 1u;  // lanes <= lane
    uint32_t k[KEY_R];
    int h[KEY_R], len[KEY_R];
#pragma unroll
    for (int j = 0; j < KEY_R; ++j) {
        const int64_t p = base + 32 * j + lane;
        k[j] = 0xffffffffu;
        if (p < np) {
            Located L = locate(g, x[j][0], x[j][1], x[j][2]);
            if (L.err)
                err |= L.err;
            else
                k[j] = bin_of(g, L);
        }
        const uint32_t kp = __shfl_up_sync(0xffffffffu, k[j], 1);
        const bool head = lane == 0 || k[j] != kp;
        const unsigned heads = __ballot_sync(0xffffffffu, head);
        h[j] = 31 - __clz(heads & below);                         // this lane's run head
        const unsigned after = heads & ~below;                    // heads past this lane
        len[j] = head ? (after ? __ffs(after) - 1 : 32) - lane : 0;  // run length (heads only)
    }
    // the rounds' atomics are independent: issue them all before using any result
    int r[KEY_R];
#pragma unroll
    for (int j = 0; j < KEY_R; ++j)
        r[j] = (len[j] > 0 && k[j] != 0xffffffffu) ? atomicAdd(&count[k[j]], len[j]) : 0;
#pragma unroll
    for (int j = 0; j < KEY_R; ++j) {
        const int64_t p = base + 32 * j + lane;
        const int rr = __shfl_sync(0xffffffffu, r[j], h[j]) + (lane - h[j]);
        if (p < np) {
            key[p] = k[j];
            rank[p] = k[j] != 0xffffffffu ? rr : -1;  // -1: no bin (the call fails), no record
        }
    }
    if (err) {
        atomicOr(&status[ST_ERR], err);
        atomicOr(&status[ST_STICKY], err);
    }
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
    const int64_t p0 = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    if (p0 >= np)
        return;
    uint32_t k[4];
    int r[4];
    if (p0 + 4 <= np) {
        uint4 kk = *reinterpret_cast<const uint4 *>(key + p0);
        int4 rr = *reinterpret_cast<const int4 *>(rank + p0);
        k[0] = kk.x; k[1] = kk.y; k[2] = kk.z; k[3] = kk.w;
        r[0] = rr.x; r[1] = rr.y; r[2] = rr.z; r[3] = rr.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            k[j] = p0 + j < np ? key[p0 + j] : 0xffffffffu;
            r[j] = p0 + j < np ? rank[p0 + j] : 0;
        }
    }
    int sb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        sb[j] = k[j] != 0xffffffffu ? __ldg(seg_begin + k[j]) : 0;
#pragma unroll
    for (int j = 0; j < 4; ++j)
        if (k[j] != 0xffffffffu)
            perm[sb[j] + r[j]] = (int32_t)(p0 + j);
}

// ---- per-bin fix-up: ascending order of original indices == stable sort ----
constexpr int FIX_WARPS = 8;
#ifndef FIX_DYN
#define FIX_DYN 16  // per-bin fix-up kernels: bins per atomic of the work counter (c4 k_fixrec_warp
                    // 3.81 -> 3.33 ms against the static grid stride; c2 unchanged); 0: static
#endif
constexpr int ST_FIXCNT = 7;  // status word: the fix-up kernels' work counter (cleared per launch)

__device__ __forceinline__ void st256(double *p, double a, double b, double c, double d)
{
    asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}


// Register bitonic network over K = 32 or 64 keys (2 per lane), fully unrolled so the
// partner distances and directions are compile-time constants.
template <int K>
__device__ __forceinline__ void bitonic_reg(int32_t &v0, int32_t &v1, int lane)
{
#pragma unroll
    for (int k = 2; k <= K; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j == 32) {
                const int32_t lo = min(v0, v1), hi = max(v0, v1);
                v0 = lo;  // k == 64: every index ascends
                v1 = hi;
            } else {
                const bool lower = (lane & j) == 0;
                const int32_t p0 = __shfl_xor_sync(0xffffffffu, v0, j);
                const bool up0 = (lane & k) == 0;
                v0 = (lower == up0) ? min(v0, p0) : max(v0, p0);
                if (K == 64) {
                    const int32_t p1 = __shfl_xor_sync(0xffffffffu, v1, j);
                    const bool up1 = ((lane + 32) & k) == 0;
                    v1 = (lower == up1) ? min(v1, p1) : max(v1, p1);
                }
            }
        }
    }
}

// pad slots: perm -1, all-zero records (rs = record stride in doubles: 8 with B, 4 without)
// Register bitonic network over K = 32 R keys, element i = lane + 32 r in v[r]: partners at
// distance j >= 32 sit in the same lane (register r ^ j/32), at j < 32 in lane ^ j (shuffle).
// Everything is unrolled: partner distances, directions and register indices are constants.
template <int R>
__device__ __forceinline__ void bitonic_regs(int32_t (&v)[R], int lane)
{
    constexpr int K = 32 * R;
#pragma unroll
    for (int k = 2; k <= K; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jr = j >> 5;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (r & jr)
                        continue;
                    const int r2 = r | jr;
                    const bool up = ((lane + 32 * r) & k) == 0;
                    const int32_t lo = min(v[r], v[r2]), hi = max(v[r], v[r2]);
                    v[r] = up ? lo : hi;
                    v[r2] = up ? hi : lo;
                }
            } else {
                const bool lower = (lane & j) == 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int32_t pv = __shfl_xor_sync(0xffffffffu, v[r], j);
                    const bool up = ((lane + 32 * r) & k) == 0;
                    v[r] = (lower == up) ? min(v[r], pv) : max(v[r], pv);
                }
            }
        }
    }
}

// A bin of 64 < n <= 32 R particles held in registers: skip the network when the slice is
// already ascending, then write perm and the inverse permutation.
template <int R>
__device__ __forceinline__ void fix_bin_regs(int32_t *__restrict__ perm, int32_t *__restrict__ dest, int64_t b, int n,
                                             int lane)
{
    int32_t v[R];
#pragma unroll
    for (int r = 0; r < R; ++r)
        v[r] = lane + 32 * r < n ? perm[b + lane + 32 * r] : INT_MAX;
    bool ok = true;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int32_t nx = __shfl_down_sync(0xffffffffu, v[r], 1);
        const int32_t first = r + 1 < R ? __shfl_sync(0xffffffffu, v[r + 1 < R ? r + 1 : r], 0) : INT_MAX;
        ok = ok && (lane < 31 ? v[r] <= nx : v[r] <= first);
    }
    if (!__all_sync(0xffffffffu, ok))
        bitonic_regs<R>(v, lane);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        if (i < n) {
            perm[b + i] = v[r];
            if (dest)
                dest[v[r]] = (int32_t)(b + i);
        }
    }
}

__device__ __forceinline__ void zero_pads(int32_t *perm, double *rec, int rs, int64_t from, int64_t to, int tid,
                                          int nthr)
{
    for (int64_t i = from + tid; i < to; i += nthr) {
        perm[i] = -1;
        st256(rec + rs * i, 0.0, 0.0, 0.0, 0.0);
        if (rs == 8)
            st256(rec + rs * i + 4, 0.0, 0.0, 0.0, 0.0);
    }
}

__global__ void __launch_bounds__(FIX_WARPS * 32) k_fix_warp(int64_t nbins, const int32_t *__restrict__ count,
                                                             const int32_t *__restrict__ seg_begin,
                                                             int32_t *__restrict__ perm, int32_t *__restrict__ dest,
                                                             double *__restrict__ rec, int32_t *__restrict__ mid_list,
                                                             int32_t *__restrict__ huge_list,
                                                             int32_t *__restrict__ status, int rs)
{
    __shared__ int32_t buf[FIX_WARPS][WARP_BIN_MAX];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int32_t *s = buf[w];
    // bins from the status word ST_FIXCNT in runs of FIX_DYN per warp (dynamic balance); FIX_DYN 0:
    // the static grid stride
    const int64_t nwarps = (int64_t)gridDim.x * FIX_WARPS;
    int64_t bin = FIX_DYN ? 0 : (int64_t)blockIdx.x * FIX_WARPS + w, bend = 0;
    for (;; bin += FIX_DYN ? 1 : nwarps) {
        if (FIX_DYN && bin == bend) {
            int t = 0;
            if (lane == 0)
                t = atomicAdd(&status[ST_FIXCNT], FIX_DYN);
            bin = __shfl_sync(0xffffffffu, t, 0);
            bend = bin + FIX_DYN;
        }
        if (bin >= nbins)
            break;
        const int n = count[bin];
        const int64_t b = seg_begin[bin], e = seg_begin[bin + 1];
        zero_pads(perm, rec, rs, b + n, e, lane, 32);
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
        if (n <= 64) {
            // bitonic sort of the bin's keys held as (v0 = elem lane, v1 = elem lane + 32)
            int32_t v0 = lane < n ? perm[b + lane] : INT_MAX;
            int32_t v1 = lane + 32 < n ? perm[b + lane + 32] : INT_MAX;
            // atomic ranks mostly follow the particle index already (CTAs run roughly in
            // order): skip the network when the slice is ascending
            const int32_t nx0 = __shfl_down_sync(0xffffffffu, v0, 1);
            const int32_t first1 = __shfl_sync(0xffffffffu, v1, 0);
            const int32_t nx1 = __shfl_down_sync(0xffffffffu, v1, 1);
            const bool ok0 = lane < 31 ? v0 <= nx0 : v0 <= first1;
            const bool ok1 = lane < 31 ? v1 <= nx1 : true;
            if (!__all_sync(0xffffffffu, ok0 && ok1)) {
                if (n <= 32)
                    bitonic_reg<32>(v0, v1, lane);
                else
                    bitonic_reg<64>(v0, v1, lane);
            }
            if (lane < n) {
                perm[b + lane] = v0;
                if (dest)
                    dest[v0] = (int32_t)(b + lane);
            }
            if (lane + 32 < n) {
                perm[b + lane + 32] = v1;
                if (dest)
                    dest[v1] = (int32_t)(b + lane + 32);
            }
            continue;
        }
        if (n <= 512) {  // register networks (the shared-memory network below is slower)
            if (n <= 128)
                fix_bin_regs<4>(perm, dest, b, n, lane);
            else if (n <= 256)
                fix_bin_regs<8>(perm, dest, b, n, lane);
            else
                fix_bin_regs<16>(perm, dest, b, n, lane);
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
            if (dest)
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
            if (dest)
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
                if (dest)
                    dest[p] = (int32_t)(out + pre);
            }
            out += total;
        }
    }
}

template <bool VEC, typename TP>
__global__ void __launch_bounds__(256, 3) k_scatter(Geo g, int64_t np, const TP *__restrict__ pos, const double *__restrict__ q,
                          const TP *__restrict__ B, const int32_t *__restrict__ dest, double *__restrict__ rec,
                          int32_t *__restrict__ status)
{
    extern __shared__ __align__(128) double sm_rec[];  // [256 threads][4 records][8]
    const int64_t p0 = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    if (p0 >= np)
        return;
    const bool full = p0 + 4 <= np;
    int d[4];  // sorted slot of each particle; -1 for a particle without a bin (failed locate)
    double qq[4], x[12], bb[12];
    if (full) {
        int4 dd = *reinterpret_cast<const int4 *>(dest + p0);
        d[0] = dd.x; d[1] = dd.y; d[2] = dd.z; d[3] = dd.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            d[j] = p0 + j < np ? dest[p0 + j] : -1;
    }
    load_vec3x4<VEC>(pos, p0, np, x);
    if (VEC && full) {
        double4 t = ld256(q + p0);
        qq[0] = t.x; qq[1] = t.y; qq[2] = t.z; qq[3] = t.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            qq[j] = p0 + j < np ? q[p0 + j] : 0.0;
    }
    if (B) {
        load_vec3x4<VEC>(B, p0, np, bb);
    } else {
#pragma unroll
        for (int j = 0; j < 12; ++j)
            bb[j] = 0.0;
    }
    int err = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (d[j] < 0)
            continue;
        Located L = locate(g, x[3 * j], x[3 * j + 1], x[3 * j + 2]);
        if (!(isfinite(qq[j]) && isfinite(bb[3 * j]) && isfinite(bb[3 * j + 1]) && isfinite(bb[3 * j + 2])))
            err |= ERR_NONFINITE;
        // The record is staged in shared memory and written with ONE bulk copy (cp.async.bulk,
        // 64 B; 32 B {xi, q} for a scalar-only handle): a single L2 request per random record
        // instead of two 32-B stores (record scatter 640 -> 503 us at c2).
        double *sr = sm_rec + 32 * threadIdx.x + 8 * j;
        sr[0] = L.xi[0];
        sr[1] = L.xi[1];
        sr[2] = L.xi[2];
        sr[3] = qq[j];
        if (B) {
            sr[4] = bb[3 * j];
            sr[5] = bb[3 * j + 1];
            sr[6] = bb[3 * j + 2];
            sr[7] = 0.0;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (B)
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 64;" ::"l"(rec + 8 * (int64_t)d[j]),
                         "r"((uint32_t)__cvta_generic_to_shared(sr))
                         : "memory");
        else
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 32;" ::"l"(rec + 4 * (int64_t)d[j]),
                         "r"((uint32_t)__cvta_generic_to_shared(sr))
                         : "memory");
    }
    // the copies read this thread's staging slots: wait before the CTA may exit
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (err) {
        atomicOr(&status[ST_ERR], err);
        atomicOr(&status[ST_STICKY], err);
    }
}

// ---- record-first path for inputs beyond L2 ----------------------------------------------
// Beyond the 126 MB L2 the classic path's two random 4-B passes (k_place: perm[seg + rank] = p;
// the fix-up's inverse permutation dest[perm[i]] = i) cost 9 of the 14 ms of a 134.7 M-particle
// sort: random stores are bound by the L2 request rate (one request per lane) whatever their
// width.  Here the only random pass is the record one:
//   k_scatter0  coalesced over particles: the 64-B record {xi, q, B, p} goes to its UNSTABLE
//               slot seg_begin[key] + rank of a scratch buffer (the particle index p in the pad
//               double), one cp.async.bulk each;
//   k_fixrec_*  per bin, coalesced: sort the (p, slot) pairs of the bin by p (= stable order),
//               write perm and the final records (pad double 0; 32-B records without B) in
//               order, zero the K-padding.
// The result is bit-identical to the classic path (tests/test_gpu_parity_sort_tf32.py runs
// both).  The inverse permutation is not produced; mm_resort_by_cell rebuilds it (k_inverse).

template <bool VEC, typename TP>
__global__ void __launch_bounds__(256, 3) k_scatter0(Geo g, int64_t np, const TP *__restrict__ pos,
                                                     const double *__restrict__ q, const TP *__restrict__ B,
                                                     const uint32_t *__restrict__ key,
                                                     const int32_t *__restrict__ rank,
                                                     const int32_t *__restrict__ seg_begin,
                                                     double *__restrict__ tmp, int32_t *__restrict__ status)
{
    extern __shared__ __align__(128) double sm_rec0[];  // [256 threads][4 records][8]
    const int64_t p0 = 4 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
    if (p0 >= np)
        return;
    const bool full = p0 + 4 <= np;
    uint32_t k[4];
    int r[4];
    if (full) {
        const uint4 kk = *reinterpret_cast<const uint4 *>(key + p0);
        const int4 rr = *reinterpret_cast<const int4 *>(rank + p0);
        k[0] = kk.x; k[1] = kk.y; k[2] = kk.z; k[3] = kk.w;
        r[0] = rr.x; r[1] = rr.y; r[2] = rr.z; r[3] = rr.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            k[j] = p0 + j < np ? key[p0 + j] : 0xffffffffu;
            r[j] = p0 + j < np ? rank[p0 + j] : 0;
        }
    }
    int d[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
        d[j] = k[j] != 0xffffffffu ? __ldg(seg_begin + k[j]) + r[j] : -1;
    double qq[4], x[12], bb[12];
    load_vec3x4<VEC>(pos, p0, np, x);
    if (VEC && full) {
        const double4 t = ld256(q + p0);
        qq[0] = t.x; qq[1] = t.y; qq[2] = t.z; qq[3] = t.w;
    } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            qq[j] = p0 + j < np ? q[p0 + j] : 0.0;
    }
    if (B) {
        load_vec3x4<VEC>(B, p0, np, bb);
    } else {
#pragma unroll
        for (int j = 0; j < 12; ++j)
            bb[j] = 0.0;
    }
    int err = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        if (d[j] < 0)
            continue;
        Located L = locate(g, x[3 * j], x[3 * j + 1], x[3 * j + 2]);
        if (!(isfinite(qq[j]) && isfinite(bb[3 * j]) && isfinite(bb[3 * j + 1]) && isfinite(bb[3 * j + 2])))
            err |= ERR_NONFINITE;
        double *sr = sm_rec0 + 32 * threadIdx.x + 8 * j;
        sr[0] = L.xi[0];
        sr[1] = L.xi[1];
        sr[2] = L.xi[2];
        sr[3] = qq[j];
        sr[4] = bb[3 * j];
        sr[5] = bb[3 * j + 1];
        sr[6] = bb[3 * j + 2];
        sr[7] = __longlong_as_double(p0 + j);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 64;" ::"l"(tmp + 8 * (int64_t)d[j]),
                     "r"((uint32_t)__cvta_generic_to_shared(sr))
                     : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (err) {
        atomicOr(&status[ST_ERR], err);
        atomicOr(&status[ST_STICKY], err);
    }
}

// Register bitonic network over K = 32 R 64-bit keys (element i = lane + 32 r in v[r]), as
// bitonic_regs; keys are (particle index << 32 | scratch slot), distinct.
template <int R>
__device__ __forceinline__ void bitonic_regs64(uint64_t (&v)[R], int lane)
{
    constexpr int K = 32 * R;
#pragma unroll
    for (int k = 2; k <= K; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jr = j >> 5;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (r & jr)
                        continue;
                    const int r2 = r | jr;
                    const bool up = ((lane + 32 * r) & k) == 0;
                    const uint64_t lo = min(v[r], v[r2]), hi = max(v[r], v[r2]);
                    v[r] = up ? lo : hi;
                    v[r2] = up ? hi : lo;
                }
            } else {
                const bool lower = (lane & j) == 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint64_t pv = __shfl_xor_sync(0xffffffffu, v[r], j);
                    const bool up = ((lane + 32 * r) & k) == 0;
                    v[r] = (lower == up) ? min(v[r], pv) : max(v[r], pv);
                }
            }
        }
    }
}

// slot j of the bin (sorted position) <- scratch record src: perm and the final record
__device__ __forceinline__ void put_rec(const double *__restrict__ tmp, double *__restrict__ rec,
                                        int32_t *__restrict__ perm, int rs, int64_t j, int64_t src, int32_t p)
{
    perm[j] = p;
    const double4 a = ld256(tmp + 8 * src);
    st256(rec + rs * j, a.x, a.y, a.z, a.w);
    if (rs == 8) {
        const double4 c = ld256(tmp + 8 * src + 4);
        st256(rec + rs * j + 4, c.x, c.y, c.z, 0.0);
    }
}

template <int R>
__device__ __forceinline__ void fixrec_regs(const double *__restrict__ tmp, double *__restrict__ rec,
                                            int32_t *__restrict__ perm, int rs, int64_t b, int n, int lane)
{
    uint64_t v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        v[r] = i < n ? ((uint64_t)(uint32_t)__double_as_longlong(tmp[8 * (b + i) + 7]) << 32) | (uint32_t)i
                     : ~0ull;
    }
    bool ok = true;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint64_t nx = __shfl_down_sync(0xffffffffu, v[r], 1);
        const uint64_t first = __shfl_sync(0xffffffffu, v[r + 1 < R ? r + 1 : r], 0);
        ok = ok && (lane < 31 ? v[r] <= nx : (r + 1 < R ? v[r] <= first : true));
    }
    if (!__all_sync(0xffffffffu, ok))
        bitonic_regs64<R>(v, lane);
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        if (i < n)
            put_rec(tmp, rec, perm, rs, b + i, b + (uint32_t)v[r], (int32_t)(v[r] >> 32));
    }
}

// Bins of 64 < n <= 32 R: the 32-bit network on the particle indices alone (half the work of the
// 64-bit one), then each element finds its sorted position by binary search in the sorted list
// (indices are distinct) and leaves its scratch slot there, so the record copies run in order.
template <int R>
__device__ __forceinline__ void fixrec_regs32(const double *__restrict__ tmp, double *__restrict__ rec,
                                              int32_t *__restrict__ perm, int rs, int64_t b, int n, int lane,
                                              int32_t *__restrict__ sp, int16_t *__restrict__ src)
{
    int32_t v[R], o[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        v[r] = o[r] = i < n ? (int32_t)__double_as_longlong(tmp[8 * (b + i) + 7]) : INT_MAX;
    }
    bool ok = true;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int32_t nx = __shfl_down_sync(0xffffffffu, v[r], 1);
        const int32_t first = __shfl_sync(0xffffffffu, v[r + 1 < R ? r + 1 : r], 0);
        ok = ok && (lane < 31 ? v[r] <= nx : (r + 1 < R ? v[r] <= first : true));
    }
    if (__all_sync(0xffffffffu, ok)) {  // already ascending: slot i stays at i
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const int i = lane + 32 * r;
            if (i < n)
                put_rec(tmp, rec, perm, rs, b + i, b + i, v[r]);
        }
        return;
    }
    bitonic_regs<R>(v, lane);
#pragma unroll
    for (int r = 0; r < R; ++r)
        sp[lane + 32 * r] = v[r];
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        if (i < n) {
            int lo = 0, hi = n;  // first position with sp[pos] >= o[r]
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sp[mid] < o[r])
                    lo = mid + 1;
                else
                    hi = mid;
            }
            src[lo] = (int16_t)i;
        }
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int j = lane + 32 * r;
        if (j < n)
            put_rec(tmp, rec, perm, rs, b + j, b + src[j], v[r]);
    }
    __syncwarp();  // sp / src are reused by the warp's next bin
}

constexpr int FIXREC_WARP_MAX = 512;

__global__ void __launch_bounds__(FIX_WARPS * 32) k_fixrec_warp(int64_t nbins, const int32_t *__restrict__ count,
                                                                const int32_t *__restrict__ seg_begin,
                                                                const double *__restrict__ tmp,
                                                                int32_t *__restrict__ perm, double *__restrict__ rec,
                                                                int32_t *__restrict__ mid_list,
                                                                int32_t *__restrict__ huge_list,
                                                                int32_t *__restrict__ status, int rs)
{
    __shared__ int32_t s_sp[FIX_WARPS][FIXREC_WARP_MAX];
    __shared__ int16_t s_src[FIX_WARPS][FIXREC_WARP_MAX];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    // bins from the status word ST_FIXCNT in runs of FIX_DYN per warp (dynamic balance); FIX_DYN 0:
    // the static grid stride
    const int64_t nwarps = (int64_t)gridDim.x * FIX_WARPS;
    int64_t bin = FIX_DYN ? 0 : (int64_t)blockIdx.x * FIX_WARPS + w, bend = 0;
    for (;; bin += FIX_DYN ? 1 : nwarps) {
        if (FIX_DYN && bin == bend) {
            int t = 0;
            if (lane == 0)
                t = atomicAdd(&status[ST_FIXCNT], FIX_DYN);
            bin = __shfl_sync(0xffffffffu, t, 0);
            bend = bin + FIX_DYN;
        }
        if (bin >= nbins)
            break;
        const int n = count[bin];
        const int64_t b = seg_begin[bin], e = seg_begin[bin + 1];
        zero_pads(perm, rec, rs, b + n, e, lane, 32);
        if (n == 0)
            continue;
        if (n > FIXREC_WARP_MAX) {
            if (lane == 0) {
                if (n > CTA_BIN_MAX)
                    huge_list[atomicAdd(&status[ST_NHUGE], 1)] = (int32_t)bin;
                else
                    mid_list[atomicAdd(&status[ST_NMID], 1)] = (int32_t)bin;
            }
            continue;
        }
        if (n <= 64)
            fixrec_regs<2>(tmp, rec, perm, rs, b, n, lane);
        else if (n <= 128)
            fixrec_regs32<4>(tmp, rec, perm, rs, b, n, lane, s_sp[w], s_src[w]);
        else if (n <= 256)
            fixrec_regs32<8>(tmp, rec, perm, rs, b, n, lane, s_sp[w], s_src[w]);
        else
            fixrec_regs32<16>(tmp, rec, perm, rs, b, n, lane, s_sp[w], s_src[w]);
    }
}

// bins of FIXREC_WARP_MAX < n <= CTA_BIN_MAX: bitonic sort of the 64-bit keys in shared memory
__global__ void __launch_bounds__(1024) k_fixrec_cta(const int32_t *__restrict__ count,
                                                     const int32_t *__restrict__ seg_begin,
                                                     const double *__restrict__ tmp, int32_t *__restrict__ perm,
                                                     double *__restrict__ rec, const int32_t *__restrict__ mid_list,
                                                     const int32_t *__restrict__ status, int rs)
{
    extern __shared__ uint64_t s64[];
    const int nmid = status[ST_NMID];
    for (int it = blockIdx.x; it < nmid; it += gridDim.x) {
        const int32_t bin = mid_list[it];
        const int n = count[bin];
        const int64_t b = seg_begin[bin];
        int N = 1024;
        while (N < n)
            N <<= 1;
        for (int i = threadIdx.x; i < N; i += blockDim.x)
            s64[i] = i < n ? ((uint64_t)(uint32_t)__double_as_longlong(tmp[8 * (b + i) + 7]) << 32) | (uint32_t)i
                           : ~0ull;
        __syncthreads();
        for (int k = 2; k <= N; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int i = threadIdx.x; i < N; i += blockDim.x) {
                    const int ixj = i ^ j;
                    if (ixj > i) {
                        const uint64_t x = s64[i], y = s64[ixj];
                        const bool up = (i & k) == 0;
                        if ((x > y) == up) {
                            s64[i] = y;
                            s64[ixj] = x;
                        }
                    }
                }
                __syncthreads();
            }
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x)
            put_rec(tmp, rec, perm, rs, b + i, b + (uint32_t)s64[i], (int32_t)(s64[i] >> 32));
        __syncthreads();
    }
}

// bins of more than CTA_BIN_MAX particles (degenerate inputs): stable compaction over the
// particles; the scratch slot of particle p is seg_begin[key] + rank[p]
__global__ void __launch_bounds__(1024) k_fixrec_huge(int64_t np, const uint32_t *__restrict__ key,
                                                      const int32_t *__restrict__ rank,
                                                      const int32_t *__restrict__ seg_begin,
                                                      const double *__restrict__ tmp, int32_t *__restrict__ perm,
                                                      double *__restrict__ rec, const int32_t *__restrict__ huge_list,
                                                      const int32_t *__restrict__ status, int rs)
{
    const int nhuge = status[ST_NHUGE];
    for (int it = blockIdx.x; it < nhuge; it += gridDim.x) {
        const uint32_t bin = (uint32_t)huge_list[it];
        const int64_t b = seg_begin[bin];
        int64_t out = b;
        for (int64_t c0 = 0; c0 < np; c0 += blockDim.x) {
            const int64_t p = c0 + threadIdx.x;
            const int f = (p < np && key[p] == bin) ? 1 : 0;
            int total;
            const int pre = block_excl_scan(f, total);
            if (f)
                put_rec(tmp, rec, perm, rs, out + pre, b + rank[p], (int32_t)p);
            out += total;
        }
    }
}

// dest[perm[i]] = i over the padded slots (mm_resort_by_cell needs the previous sort's inverse
// permutation; the record-first path does not produce it)
__global__ void k_inverse(const int32_t *__restrict__ perm, const int32_t *__restrict__ total,
                          int32_t *__restrict__ dest)
{
    const int64_t n = *total;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = perm[i];
        if (p >= 0)
            dest[p] = (int32_t)i;
    }
}

// ---- incremental re-binning (NEXT-1; the "sort & communicate" stage of a PIC
// cycle): the same particles, moved.  Every particle is re-keyed; only the
// ones whose bin changed touch the bin counters (leave the old bin, join the new one, get an
// arrival rank); each bin's member list is then its old (stable, ascending) slice minus the
// leavers plus its arrivals, and the per-bin fix-up restores ascending order - the result is
// bit-identical to a fresh sort of the new positions.
// rank[] holds the previous sort's dest (each particle's old slot) on entry: a mover marks its
// old slot in the old permutation (-3, so the member pass needs no key lookup) and rank[] then
// carries its arrival rank (-2 for a stayer, -1 for a particle outside the grid) until the
// fix-up rewrites dest
template <typename TP>
__global__ void __launch_bounds__(256) k_rekey(Geo g, int64_t np, const TP *__restrict__ pos,
                                               uint32_t *__restrict__ key, int32_t *__restrict__ rank,
                                               int32_t *__restrict__ count, int32_t *__restrict__ arr_count,
                                               int32_t *__restrict__ perm_old, int32_t *__restrict__ status)
{
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np)
        return;
    int err = 0;
    uint32_t kn = 0xffffffffu;
    const double x0 = (double)__ldg(pos + 3 * p), x1 = (double)__ldg(pos + 3 * p + 1),
                 x2 = (double)__ldg(pos + 3 * p + 2);
    const uint32_t ko = key[p];
    Located L = locate(g, x0, x1, x2);
    if (L.err)
        err = L.err;
    else
        kn = bin_of(g, L);
    int r = -2;
    if (kn != ko) {
        if (ko != 0xffffffffu) {
            atomicSub(&count[ko], 1);
            perm_old[rank[p]] = -3;  // leaver
        }
        if (kn != 0xffffffffu) {
            atomicAdd(&count[kn], 1);
            r = atomicAdd(&arr_count[kn], 1);
        }
        key[p] = kn;
    }
    rank[p] = kn == 0xffffffffu ? -1 : r;
    if (err) {
        atomicOr(&status[ST_ERR], err);
        atomicOr(&status[ST_STICKY], err);
    }
}

__global__ void __launch_bounds__(256) k_arrive(int64_t np, const uint32_t *__restrict__ key,
                                                const int32_t *__restrict__ rank, const int32_t *__restrict__ arr_begin,
                                                int32_t *__restrict__ arr)
{
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= np)
        return;
    const int r = rank[p];
    if (r >= 0)
        arr[arr_begin[key[p]] + r] = (int32_t)p;
}

// warp per bin: the old slice's stayers (still keyed to this bin) in their old ascending order,
// then the bin's arrivals; the fix-up sorts the slice
__global__ void __launch_bounds__(256) k_members(int64_t nbins, const int32_t *__restrict__ seg_old,
                                                 const int32_t *__restrict__ perm_old,
                                                 const uint32_t *__restrict__ key,
                                                 const int32_t *__restrict__ arr_begin,
                                                 const int32_t *__restrict__ arr_count,
                                                 const int32_t *__restrict__ arr,
                                                 const int32_t *__restrict__ seg_begin, int32_t *__restrict__ perm)
{
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t bin = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); bin < nbins; bin += nw) {
        const int o0 = seg_old[bin], o1 = seg_old[bin + 1];
        int out = seg_begin[bin];
        for (int i = o0; i < o1; i += 32) {
            const int pp = i + lane < o1 ? perm_old[i + lane] : -1;
            const bool stay = pp >= 0;  // leavers were marked -3 by k_rekey
            const unsigned b = __ballot_sync(0xffffffffu, stay);
            if (stay)
                perm[out + __popc(b & ((1u << lane) - 1u))] = pp;
            out += __popc(b);
            if (__ballot_sync(0xffffffffu, pp == -1 && i + lane < o1))
                break;  // the padding (-1, not a leaver's -3) ends the old members
        }
        const int a0 = arr_begin[bin], na = arr_count[bin];
        for (int j = lane; j < na; j += 32)
            perm[out + j] = arr[a0 + j];
    }
}

inline unsigned blocks_for(int64_t n, int t)
{
    return (unsigned)((n + t - 1) / t);
}

// Diagnostics (MM_SORT_TIMERS=1): CUDA events after every phase, printed to stderr.
struct PhaseTimer {
    bool on = false;
    cudaStream_t s = nullptr;
    int n = 0;
    cudaEvent_t ev[32];
    const char *tag[32];
    explicit PhaseTimer(cudaStream_t st) : s(st)
    {
        static const bool env = [] {
            const char *v = getenv("MM_SORT_TIMERS");
            return v && v[0] == '1';
        }();
        on = env;
        mark("start");
    }
    void mark(const char *t)
    {
        if (!on || n >= 32)
            return;
        cudaEventCreate(&ev[n]);
        cudaEventRecord(ev[n], s);
        tag[n++] = t;
    }
    ~PhaseTimer()
    {
        if (!on)
            return;
        cudaEventSynchronize(ev[n - 1]);
        fprintf(stderr, "[mm sort]");
        for (int i = 1; i < n; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            fprintf(stderr, " %s %.1f", tag[i], ms * 1e3f);
        }
        fprintf(stderr, " us\n");
        for (int i = 0; i < n; ++i)
            cudaEventDestroy(ev[i]);
    }
};

}  // namespace

int64_t scan_tmp_elems(int64_t nbins)
{
    return (nbins + SCAN_TILE - 1) / SCAN_TILE + 1;
}

// The per-bin fix-up (ascending original indices = stable order, dest, K padding) and the
// record scatter, shared by the full and the incremental sort.
template <typename PT>
cudaError_t fixup_scatter_enqueue(const Geo &geo, const SortBufs &b, cudaStream_t s, PT &pt)
{
    cudaError_t e;
    const int T = 256;
    const bool vec = ((uintptr_t)b.pos % 32 == 0) && ((uintptr_t)b.q % 32 == 0) && ((uintptr_t)b.B % 32 == 0);
    int32_t *dest = b.rank;
    {
        int64_t want = (b.nbins + FIX_WARPS - 1) / FIX_WARPS;
        unsigned grid = (unsigned)(want < 148 * 16 ? want : 148 * 16);
        if (grid < 1)
            grid = 1;
        if ((e = cudaMemsetAsync(b.status + ST_FIXCNT, 0, sizeof(int32_t), s)))
            return e;
        k_fix_warp<<<grid, FIX_WARPS * 32, 0, s>>>(b.nbins, b.count, b.seg_begin, b.perm, dest, b.rec,
                                                   b.mid_list, b.huge_list, b.status, b.B ? 8 : 4);
        count_launch();
        pt.mark("fix");
    }
    if (b.np > WARP_BIN_MAX) {
        // per call: the attribute is per device/context (a process may drive several GPUs)
        if ((e = cudaFuncSetAttribute(k_fix_cta, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      CTA_BIN_MAX * 4)))
            return e;
        k_fix_cta<<<148, 1024, CTA_BIN_MAX * 4, s>>>(b.count, b.seg_begin, b.perm, dest, b.mid_list, b.status);
        count_launch();
    }
    if (b.np > CTA_BIN_MAX) {
        k_fix_huge<<<8, 1024, 0, s>>>(b.np, b.key, b.seg_begin, b.perm, dest, b.huge_list, b.status);
        count_launch();
    }

    if (b.np > 0) {
        const unsigned gs = blocks_for((b.np + 3) / 4, T);
        constexpr int SCAT_SMEM = 256 * 4 * 64;
        // per call: the attribute is per device/context (a process may drive several GPUs)
        if ((e = cudaFuncSetAttribute(k_scatter<true, double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SCAT_SMEM)) ||
            (e = cudaFuncSetAttribute(k_scatter<false, double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SCAT_SMEM)) ||
            (e = cudaFuncSetAttribute(k_scatter<true, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SCAT_SMEM)) ||
            (e = cudaFuncSetAttribute(k_scatter<false, float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SCAT_SMEM)))
            return e;
        if (b.f32) {
            const float *pf = reinterpret_cast<const float *>(b.pos), *bf = reinterpret_cast<const float *>(b.B);
            const bool v16 = ((uintptr_t)pf % 16 == 0) && ((uintptr_t)bf % 16 == 0) && ((uintptr_t)b.q % 32 == 0);
            if (v16)
                k_scatter<true, float><<<gs, T, SCAT_SMEM, s>>>(geo, b.np, pf, b.q, bf, b.rank, b.rec, b.status);
            else
                k_scatter<false, float><<<gs, T, SCAT_SMEM, s>>>(geo, b.np, pf, b.q, bf, b.rank, b.rec,
                                                                 b.status);
        } else if (vec) {
            k_scatter<true, double><<<gs, T, SCAT_SMEM, s>>>(geo, b.np, b.pos, b.q, b.B, b.rank, b.rec, b.status);
        } else {
            k_scatter<false, double><<<gs, T, SCAT_SMEM, s>>>(geo, b.np, b.pos, b.q, b.B, b.rank, b.rec,
                                                              b.status);
        }
        count_launch();
        pt.mark("scatter");
    }
    return cudaGetLastError();
}

template <typename PT>
cudaError_t recfirst_enqueue(const Geo &geo, const SortBufs &b, cudaStream_t s, PT &pt)
{
    cudaError_t e;
    const int T = 256;
    const int rs = b.B ? 8 : 4;
    {
        constexpr int SMEM0 = 256 * 4 * 64;
        const unsigned gs = blocks_for((b.np + 3) / 4, T);
        auto k_d_v = k_scatter0<true, double>, k_d_n = k_scatter0<false, double>;
        auto k_f_v = k_scatter0<true, float>, k_f_n = k_scatter0<false, float>;
        if ((e = cudaFuncSetAttribute(k_d_v, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM0)) ||
            (e = cudaFuncSetAttribute(k_d_n, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM0)) ||
            (e = cudaFuncSetAttribute(k_f_v, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM0)) ||
            (e = cudaFuncSetAttribute(k_f_n, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM0)))
            return e;
        if (b.f32) {
            const float *pf = reinterpret_cast<const float *>(b.pos), *bf = reinterpret_cast<const float *>(b.B);
            const bool v16 = ((uintptr_t)pf % 16 == 0) && ((uintptr_t)bf % 16 == 0) && ((uintptr_t)b.q % 32 == 0);
            (v16 ? k_f_v : k_f_n)<<<gs, T, SMEM0, s>>>(geo, b.np, pf, b.q, bf, b.key, b.rank, b.seg_begin, b.rec_tmp,
                                                       b.status);
        } else {
            const bool vec = ((uintptr_t)b.pos % 32 == 0) && ((uintptr_t)b.q % 32 == 0) && ((uintptr_t)b.B % 32 == 0);
            (vec ? k_d_v : k_d_n)<<<gs, T, SMEM0, s>>>(geo, b.np, b.pos, b.q, b.B, b.key, b.rank, b.seg_begin,
                                                       b.rec_tmp, b.status);
        }
        count_launch();
        pt.mark("scatter0");
    }
    {
        const int64_t want = (b.nbins + FIX_WARPS - 1) / FIX_WARPS;
        const unsigned grid = (unsigned)(want < 148 * 16 ? (want < 1 ? 1 : want) : 148 * 16);
        if ((e = cudaMemsetAsync(b.status + ST_FIXCNT, 0, sizeof(int32_t), s)))
            return e;
        k_fixrec_warp<<<grid, FIX_WARPS * 32, 0, s>>>(b.nbins, b.count, b.seg_begin, b.rec_tmp, b.perm, b.rec,
                                                      b.mid_list, b.huge_list, b.status, rs);
        count_launch();
    }
    if (b.np > FIXREC_WARP_MAX) {
        if ((e = cudaFuncSetAttribute(k_fixrec_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, CTA_BIN_MAX * 8)))
            return e;
        k_fixrec_cta<<<148, 1024, CTA_BIN_MAX * 8, s>>>(b.count, b.seg_begin, b.rec_tmp, b.perm, b.rec, b.mid_list,
                                                         b.status, rs);
        count_launch();
    }
    if (b.np > CTA_BIN_MAX) {
        k_fixrec_huge<<<8, 1024, 0, s>>>(b.np, b.key, b.rank, b.seg_begin, b.rec_tmp, b.perm, b.rec, b.huge_list,
                                          b.status, rs);
        count_launch();
    }
    pt.mark("fixrec");
    return cudaGetLastError();
}

cudaError_t sort_enqueue(const Geo &geo, const SortBufs &b, cudaStream_t s)
{
    cudaError_t e;
    PhaseTimer pt(s);
    if ((e = cudaMemsetAsync(b.count, 0, sizeof(int32_t) * (size_t)b.nbins, s)))
        return e;
    if ((e = cudaMemsetAsync(b.status, 0, sizeof(int32_t) * ST_PER_SORT, s)))
        return e;
    const int T = 256;
    if (b.np > 0) {
        if (b.f32)
            k_key<float><<<blocks_for((b.np + 32 * KEY_R - 1) / (32 * KEY_R) * 32, T), T, 0, s>>>(
                geo, b.np, reinterpret_cast<const float *>(b.pos), b.key, b.rank, b.count, b.status);
        else
            k_key<double><<<blocks_for((b.np + 32 * KEY_R - 1) / (32 * KEY_R) * 32, T), T, 0, s>>>(geo, b.np, b.pos, b.key, b.rank,
                                                                              b.count, b.status);
        count_launch();
        pt.mark("key");
    }
    const int nblk = (int)((b.nbins + SCAN_TILE - 1) / SCAN_TILE);
    k_scan_local<<<nblk, SCAN_T, 0, s>>>(b.count, b.nbins, b.k_pad, b.seg_begin, b.scan_tmp);
    k_scan_top<<<1, SCAN_T, 0, s>>>(b.scan_tmp, nblk, b.seg_begin + b.nbins, b.status);
    k_scan_add<<<nblk, SCAN_T, 0, s>>>(b.seg_begin, b.nbins, b.scan_tmp);
    count_launch(3);
    pt.mark("scan");
    if (b.rec_tmp && b.np > 0)
        return recfirst_enqueue(geo, b, s, pt);
    if (b.np > 0) {
        k_place<<<blocks_for((b.np + 3) / 4, T), T, 0, s>>>(b.np, b.key, b.rank, b.seg_begin, b.perm);
        count_launch();
        pt.mark("place");
    }
    return fixup_scatter_enqueue(geo, b, s, pt);
}

cudaError_t inverse_enqueue(const int32_t *perm, const int32_t *seg_end, int64_t capacity, int32_t *dest,
                            cudaStream_t s)
{
    const int64_t want = (capacity + 255) / 256;
    k_inverse<<<(unsigned)(want < 148 * 16 ? (want < 1 ? 1 : want) : 148 * 16), 256, 0, s>>>(perm, seg_end, dest);
    count_launch();
    return cudaGetLastError();
}

cudaError_t resort_enqueue(const Geo &geo, const SortBufs &b, const IncBufs &ib, cudaStream_t s)
{
    cudaError_t e;
    PhaseTimer pt(s);
    if ((e = cudaMemsetAsync(b.status, 0, sizeof(int32_t) * ST_PER_SORT, s)))
        return e;
    if ((e = cudaMemsetAsync(ib.arr_count, 0, sizeof(int32_t) * (size_t)b.nbins, s)))
        return e;
    if ((e = cudaMemcpyAsync(ib.seg_old, b.seg_begin, sizeof(int32_t) * (size_t)(b.nbins + 1),
                             cudaMemcpyDeviceToDevice, s)))
        return e;
    const int T = 256;
    if (b.np > 0) {
        k_rekey<double><<<blocks_for(b.np, T), T, 0, s>>>(geo, b.np, b.pos, b.key, b.rank, b.count, ib.arr_count,
                                                           ib.perm_old, b.status);
        count_launch();
    }
    pt.mark("rekey");
    const int nblk = (int)((b.nbins + SCAN_TILE - 1) / SCAN_TILE);
    k_scan_local<<<nblk, SCAN_T, 0, s>>>(b.count, b.nbins, b.k_pad, b.seg_begin, b.scan_tmp);
    k_scan_top<<<1, SCAN_T, 0, s>>>(b.scan_tmp, nblk, b.seg_begin + b.nbins, b.status);
    k_scan_add<<<nblk, SCAN_T, 0, s>>>(b.seg_begin, b.nbins, b.scan_tmp);
    // arrivals: plain exclusive scan (k_pad 1); its total goes to scratch status words
    k_scan_local<<<nblk, SCAN_T, 0, s>>>(ib.arr_count, b.nbins, 1, ib.arr_begin, b.scan_tmp);
    k_scan_top<<<1, SCAN_T, 0, s>>>(b.scan_tmp, nblk, ib.arr_begin + b.nbins, b.status + ST_STICKY + 1);
    k_scan_add<<<nblk, SCAN_T, 0, s>>>(ib.arr_begin, b.nbins, b.scan_tmp);
    count_launch(6);
    pt.mark("scans");
    if (b.np > 0)
        k_arrive<<<blocks_for(b.np, T), T, 0, s>>>(b.np, b.key, b.rank, ib.arr_begin, ib.arr);
    {
        const int64_t want = (b.nbins + 7) / 8;
        const unsigned grid = (unsigned)(want < 148 * 16 ? (want < 1 ? 1 : want) : 148 * 16);
        k_members<<<grid, T, 0, s>>>(b.nbins, ib.seg_old, ib.perm_old, b.key, ib.arr_begin, ib.arr_count, ib.arr,
                                     b.seg_begin, b.perm);
    }
    count_launch(2);
    pt.mark("members");
    return fixup_scatter_enqueue(geo, b, s, pt);
}

}  // namespace mm
