// Order-1 (CIC) tensor mass matrix on FP64 DMMA tiles: the c2 headline kernel.
//
// Algorithm 1 of the paper per support-window bin (R12): the
// bin's particles are contracted in batches of K_t = 4 (eq_D_batches) on mma.sync.m8n8k4.f64
// tiles, then the finished block is deposited into the node-stencil storage.
//
// Operands (pair-product plan): the tensor-product B-spline makes W_a W_b a
// product of per-axis pair products q_mu(u_mu), u_mu = a_mu + b_mu in {0,1,2}
// (q(0) = w0 w0, q(1) = w0 w1, q(2) = w1 w1, w0 = 1 - xi, w1 = xi), so the 8 x 8 x 9 node
// block of a bin is determined by the 243 sums
//
//   D[uxy][uz][c] = sum_p X_p[uxy] q_z,p(uz) s^c_p,   X = q_x(ux) q_y(uy)  (9 values)
//
// Tile plan (5 DMMA per batch of 4 particles; lane t holds k = t&3, r = t>>2):
//   T0..T2   A[r][k] = X_k[r] (r = the 8 xy-pairs 0..7)   B[k][c] = qz_k[nt] s_k[c], c < 8
//            (qz staged per particle: 3 DMUL per lane and batch form the three B operands)
//   T3       A as above                                   B[k][n] = V_k[n]  (columns 0-2 kept)
//   T4       A'[c][k] = s_k[c] (c < 8)                    B[k][n] = V_k[n]  (columns 3-5 kept)
//            V = (qz0 s8, qz1 s8, qz2 s8, X8 qz0, X8 qz1, X8 qz2, 0, 0)
//   SIMT     (uxy = 8, uz, c = 8): three FMAs per particle in the prep, reduced per bin.
// The B values are formed in registers from compact per-particle rows (X, s, q_z, V) staged
// in shared memory once per chunk: 25 staged values per particle instead of the 36 operand
// columns of a fully staged plan, 6 LDS.128 per two batches (a shared-memory load costs
// 32 lanes x its width regardless of broadcast, so the per-lane bytes are what count), and 5
// instead of 8 DMMAs per batch (640 instead of 1024 executed FLOP per particle; F_unique = 648).
//
// Deposit: the 243 sums are staged in shared memory and added into the 8 node rows of the bin
// (576 entries) with REDs.  Both the row offset and the stage index of entry (a, b, c) are
// sums of a node-a term and a (b, c) term (slot(b - a) = 13 + sb(b) - sa(a), stage = ka(a) +
// kb(b) + c), so lane p holds the (b, c) terms of p, p + 32 and 64 + (p & 7) and the a terms
// are compile-time offsets / one shared row pointer: 18 REDs of 32 lanes per bin, ~4
// instructions each.  Bins are taken in DESCENDING order from a work counter, a warp drawing
// runs of O1T_DYN consecutive tickets with one atomic (dynamic balance across the SMs, and the
// run's z-adjacent bins share half their node rows in L2); with MM_ZERO_O1 the output is zeroed
// inside the kernel, row by row, by the first-writer scheme of mm_device.cuh (one ticket per
// bin).  Records are read with an L2 evict-first hint (streamed once), so the 126 MB L2 keeps
// node rows.
#include <cstdlib>

#include "mm_device.cuh"

#ifndef O1T_UNROLL
#define O1T_UNROLL 4  // full chunks run the 4 batch pairs unrolled (0.683 -> 0.678 ms at c2); 1: rolled loop
#endif

#ifndef O1T_DYN
#define O1T_DYN 8  // bins from the work counter in runs of 8 tickets (c2 0.680 -> 0.653 ms incl. the
                   // zero-fill against the static interleaved schedule; runs of 1: 1.47 ms, the
                   // single counter serialises; 2: 0.97, 4: 0.70, 16: 0.653, 32: 0.667); 0: static
#endif

#ifndef O1T_MINB
#define O1T_MINB 5  // resident CTAs per SM the register allocation targets (96 registers)
#endif

namespace mm {

namespace {

using namespace dev;

struct O1T {
    static constexpr int WARPS = 4;
    static constexpr int XS = 40;   // row stride (doubles), = 8 mod 16: LDS.128 fragment loads conflict-free
    static constexpr int ROWS = 26; // 0-7 X, 8-15 s[0..7], 16-18 q_z, 19-24 V, 25 zeros
    static constexpr int R_S = 8, R_Q = 16, R_V = 19, R_ZERO = 25;
    static constexpr int WD = ROWS * XS;  // the stage [9][27] aliases rows 0..6
    static constexpr size_t SMEM = (size_t)WARPS * WD * 8 + WARPS * 8 * 8;
};

template <bool ZERO, int MINB>
__global__ void __launch_bounds__(O1T::WARPS * 32, MINB)
    k_asm_o1t(Geo g, const double *__restrict__ rec, const int32_t *__restrict__ seg_begin, int nbins, double wscale,
              double sigma, double *__restrict__ out, double *__restrict__ ghost, int *__restrict__ work, ZeroPlan zp)
{
    using L = O1T;
    constexpr bool TICKET = ZERO || O1T_DYN > 0;  // bins from the work counter
    extern __shared__ __align__(16) double dsm_o1t[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *xz = dsm_o1t + warp * L::WD;
    double *stage = xz;  // [9 uxy][27 = 9 uz + c] after the last batch of a bin
    double **s_row = reinterpret_cast<double **>(dsm_o1t + L::WARPS * L::WD) + warp * 8;  // node rows - 9 sa(a)
    const int plane = g.n1 * g.n2;

    xz[L::R_ZERO * L::XS + lane] = 0.0;
    xz[L::R_ZERO * L::XS + 32 + (lane & 7)] = 0.0;

    // deposit terms of this lane's (b, c) pairs p = lane, lane + 32, 64 + (lane & 7):
    // row offset 9 (13 + sb(b)) + c, stage offset kb(b) + c (the node-a terms are added per a)
    int doff[3], dst[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const int p = j < 2 ? lane + 32 * j : 64 + (lane & 7);
        const int b = p / 9, c = p - 9 * b, bx = b >> 2, by = (b >> 1) & 1, bz = b & 1;
        doff[j] = 9 * (13 + 9 * bx + 3 * by + bz) + c;
        dst[j] = 81 * bx + 27 * by + 9 * bz + c;
    }
    const int a3 = lane >> 3;  // node a of the third group: a3 (first pass), a3 + 4 (second)
    const int ka3 = 81 * (a3 >> 2) + 27 * ((a3 >> 1) & 1) + 9 * (a3 & 1);
    const int ka3b = 81 * 1 + 27 * ((a3 >> 1) & 1) + 9 * (a3 & 1);  // a3 + 4: ax = 1

    const int kq = lane & 3, rq = lane >> 2;
    const double *fx = xz + rq * L::XS + 2 * kq;                               // X[r]
    const double *fs = xz + (L::R_S + rq) * L::XS + 2 * kq;                    // s[r]
    const double *fq = xz + L::R_Q * L::XS + 2 * kq;                           // q_z[0..2]
    // T3 and T4 share ONE B operand, V = (qz0 s8, qz1 s8, qz2 s8, X8 qz0, X8 qz1, X8 qz2, 0, 0):
    // T3 (A = X) keeps its columns 0-2, T4 (A = s) its columns 3-5; the other columns are
    // never read, so no lane needs a select
    const double *fv = xz + (rq < 6 ? L::R_V + rq : L::R_ZERO) * L::XS + 2 * kq;

    // tickets: cur (this bin) and nxt, in processing order; bin = nbins - 1 - ticket.  A
    // ticket's zero task (mm_device.cuh) runs as soon as the ticket is known: lanes lbase..+7
    // get the rows of ticket + D, lanes lbase+8..+15 the own rows of a ticket < D.
    // ZERO: one ticket per bin from the work counter (the first-writer zeroing needs them);
    // O1T_DYN > 0: runs of O1T_DYN tickets per atomic; O1T_DYN = 0: the static interleaved
    // schedule (warp w: tickets w, w + W, ...)
    const int W = gridDim.x * L::WARPS;
    int cur = blockIdx.x * L::WARPS + warp, nxt = cur + W;
    // O1T_DYN: lane 0 draws runs of O1T_DYN consecutive tickets with one atomic (tk .. tk_end)
    int tk = 0, tk_end = 0;
    auto next_ticket = [&]() {
        if (ZERO)
            return ticket(work);
        if (tk == tk_end) {
            tk = atomicAdd(work, O1T_DYN > 0 ? O1T_DYN : 1);
            tk_end = tk + (O1T_DYN > 0 ? O1T_DYN : 1);
        }
        return tk++;
    };
    if (TICKET) {
        if (lane == 0) {
            cur = next_ticket();
            nxt = next_ticket();
        }
        cur = __shfl_sync(0xffffffffu, cur, 0);
        nxt = __shfl_sync(0xffffffffu, nxt, 0);
    }
    // bin coordinates (bin plane x, y, z) of the static schedule, stepped by the mixed-radix
    // digits of W instead of two integer divisions per bin
    int cx = 0, cy = 0, cz = 0, wx = 0, wy = 0, wz = 0;
    if (!TICKET) {
        wz = W % g.n2;
        wy = (W / g.n2) % g.n1;
        wx = W / plane;
        if (cur < nbins) {
            const int bin = nbins - 1 - cur;
            cx = bin / plane;
            cy = (bin - cx * plane) / g.n2;
            cz = bin - cx * plane - cy * g.n2;
        }
    }
    int64_t rel = -1;  // flag index of a row this lane publishes before the warp's next wait
    auto zero_task = [&](int tk, int lbase) {
        if (tk + zp.lookahead < nbins)
            zero_first_rows(g, nbins - 1 - tk - zp.lookahead, out, ghost, 243, lane, lbase, rel);
        if (tk < zp.lookahead && tk < nbins)
            zero_first_rows(g, nbins - 1 - tk, out, ghost, 243, lane, lbase + 8, rel);
    };
    if (ZERO) {
        zero_task(cur, 0);
        zero_task(nxt, 16);
    }
    int b0 = 0, b1 = 0, nb0 = 0, nb1 = 0;
    if (cur < nbins) {
        b0 = __ldg(seg_begin + (nbins - 1 - cur));
        b1 = __ldg(seg_begin + (nbins - cur));
    }
    if (nxt < nbins) {
        nb0 = __ldg(seg_begin + (nbins - 1 - nxt));
        nb1 = __ldg(seg_begin + (nbins - nxt));
    }
    // the lane's record of the current chunk, loaded one chunk ahead; lanes past the end of a
    // bin hold zeros (q = 0 -> exact +0 contributions)
    double4 ra = make_double4(0, 0, 0, 0), rb = ra;
    if (cur < nbins && b0 + lane < b1) {
        ra = ld256_ef(rec + 8 * (int64_t)(b0 + lane));
        rb = ld256_ef(rec + 8 * (int64_t)(b0 + lane) + 4);
    }
    __syncwarp();
    while (cur < nbins) {
        int nn = nxt + W;
        if (TICKET && lane == 0)
            nn = next_ticket();  // consumed at the end of this bin
        const int bin = nbins - 1 - cur;
        int bxl = cx, by = cy, bz = cz;
        if (TICKET) {
            bxl = bin / plane;
            const int rem = bin - bxl * plane;
            by = rem / g.n2;
            bz = rem - by * g.n2;
        }
        const int bx = g.bx0 + bxl;
        if (b1 > b0) {
            double acc[5][2], acc8[3];
#pragma unroll
            for (int t = 0; t < 5; ++t)
                acc[t][0] = acc[t][1] = 0.0;
            acc8[0] = acc8[1] = acc8[2] = 0.0;
            for (int base = b0; base < b1; base += 32) {
                const int m = min(32, b1 - base);
                const double4 ca = ra, cb = rb;
                // prefetch the lane's record of the next chunk (this bin, else the next bin)
                {
                    int64_t p = -1;
                    if (base + 32 < b1) {
                        if (base + 32 + lane < b1)
                            p = base + 32 + lane;
                    } else if (nxt < nbins && nb0 + lane < nb1) {
                        p = nb0 + lane;
                    }
                    ra = rb = make_double4(0, 0, 0, 0);
                    if (p >= 0) {
                        ra = ld256_ef(rec + 8 * p);
                        rb = ld256_ef(rec + 8 * p + 4);
                    }
                }
                __syncwarp();  // previous batches / deposit are done with xz
                {
                    double s[9];
                    coeff9(ca.w, cb.x, cb.y, cb.z, wscale, sigma, s);
                    const double wx0 = 1.0 - ca.x, wy0 = 1.0 - ca.y, wz0 = 1.0 - ca.z;
                    const double qx[3] = {wx0 * wx0, wx0 * ca.x, ca.x * ca.x};
                    const double qy[3] = {wy0 * wy0, wy0 * ca.y, ca.y * ca.y};
                    const double qz[3] = {wz0 * wz0, wz0 * ca.z, ca.z * ca.z};
                    double *col = xz + lane;
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        col[r * L::XS] = qx[r / 3] * qy[r % 3];
                    const double x8 = qx[2] * qy[2];
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        col[(L::R_S + c) * L::XS] = s[c];
#pragma unroll
                    for (int u = 0; u < 3; ++u) {
                        col[(L::R_Q + u) * L::XS] = qz[u];
                        col[(L::R_V + u) * L::XS] = qz[u] * s[8];
                        col[(L::R_V + 3 + u) * L::XS] = x8 * qz[u];
                    }
                    const double t8 = x8 * s[8];
#pragma unroll
                    for (int u = 0; u < 3; ++u)
                        acc8[u] = fma(t8, qz[u], acc8[u]);
                }
                __syncwarp();
                auto pair = [&](int i) {
                    const int o = 8 * i;
                    // 6 LDS.128 per two batches: X[r], s[r], q_z[0..2], V[r]
                    const double2 X = lds128(fx + o), S = lds128(fs + o), V = lds128(fv + o);
                    const double2 Q0 = lds128(fq + o), Q1 = lds128(fq + L::XS + o), Q2 = lds128(fq + 2 * L::XS + o);
                    auto batch = [&](double x, double sv, double q0, double q1, double q2, double v) {
                        dmma(acc[0][0], acc[0][1], x, q0 * sv);
                        dmma(acc[1][0], acc[1][1], x, q1 * sv);
                        dmma(acc[2][0], acc[2][1], x, q2 * sv);
                        dmma(acc[3][0], acc[3][1], x, v);
                        dmma(acc[4][0], acc[4][1], sv, v);
                    };
                    batch(X.x, S.x, Q0.x, Q1.x, Q2.x, V.x);
                    batch(X.y, S.y, Q0.y, Q1.y, Q2.y, V.y);
                };
                const int np8 = (m + 7) >> 3;
                if (O1T_UNROLL > 1 && np8 == 4) {  // a full chunk: the scheduler may hoist the LDS
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        pair(i);
                } else {
#pragma unroll 1
                    for (int i = 0; i < np8; ++i)
                        pair(i);
                }
            }
            // ---- stage [uxy][9 uz + c]
#pragma unroll
            for (int u = 0; u < 3; ++u)
#pragma unroll
                for (int off = 16; off > 0; off >>= 1)
                    acc8[u] += __shfl_xor_sync(0xffffffffu, acc8[u], off);
            __syncwarp();
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int n = 2 * kq + v;
#pragma unroll
                for (int nt = 0; nt < 3; ++nt)
                    stage[rq * 27 + 9 * nt + n] = acc[nt][v];     // T0..T2: (uxy r, uz nt, c n)
                if (n < 3)
                    stage[rq * 27 + 9 * n + 8] = acc[3][v];       // T3: (uxy r, uz n, c 8)
                if (n >= 3 && n < 6)
                    stage[8 * 27 + 9 * (n - 3) + rq] = acc[4][v]; // T4: (uxy 8, uz n - 3, c r)
            }
            if (lane < 3)
                stage[8 * 27 + 9 * lane + 8] = lane == 0 ? acc8[0] : (lane == 1 ? acc8[1] : acc8[2]);
            int64_t wid = -1;
            if (lane < 8) {
                const int X = g.x_begin + bx + (lane >> 2), Y = wrapi(by + ((lane >> 1) & 1), g.n1),
                          Z = wrapi(bz + (lane & 1), g.n2);
                // node row minus 9 sa(a), sa = 9 ax + 3 ay + az
                s_row[lane] = row_ptr(g, X, Y, Z, out, ghost, 243) - 9 * (9 * (lane >> 2) + 3 * ((lane >> 1) & 1) + (lane & 1));
                if (ZERO)
                    wid = row_id(g, X, Y, Z);
            }
            if (ZERO) {
                __syncwarp();  // the warp's zero stores are issued
                if (rel >= 0)
                    flag_release(zp.flags + rel, zp.epoch);
                rel = -1;
                if (wid >= 0)
                    flag_wait(zp.flags + wid, zp.epoch);
            }
            __syncwarp();
#pragma unroll
            for (int a = 0; a < 8; ++a) {
                const int ka = 81 * (a >> 2) + 27 * ((a >> 1) & 1) + 9 * (a & 1);
                double *row = s_row[a];
                red_add_nc(row + doff[0], stage[ka + dst[0]]);
                red_add_nc(row + doff[1], stage[ka + dst[1]]);
            }
            red_add_nc(s_row[a3] + doff[2], stage[ka3 + dst[2]]);
            red_add_nc(s_row[a3 + 4] + doff[2], stage[ka3b + dst[2]]);
            __syncwarp();  // the stage (aliasing xz) is read before the next chunk's prep
        } else {
            if (ZERO) {  // publish now: the zero task of nn reuses the lanes
                __syncwarp();
                if (rel >= 0)
                    flag_release(zp.flags + rel, zp.epoch);
                rel = -1;
            }
            if (nxt < nbins && nb0 + lane < nb1) {
                // empty bin: nothing was prefetched for the successor yet
                ra = ld256_ef(rec + 8 * (int64_t)(nb0 + lane));
                rb = ld256_ef(rec + 8 * (int64_t)(nb0 + lane) + 4);
            }
        }
        if (TICKET)
            nn = __shfl_sync(0xffffffffu, nn, 0);
        if (ZERO)
            zero_task(nn, 0);  // rel is free: released above (or still pending for an empty bin)
        cur = nxt;
        nxt = nn;
        if (!TICKET) {  // bin - W
            cz -= wz;
            if (cz < 0) {
                cz += g.n2;
                --cy;
            }
            cy -= wy;
            if (cy < 0) {
                cy += g.n1;
                --cx;
            }
            cx -= wx;
        }
        b0 = nb0;
        b1 = nb1;
        if (nxt < nbins) {
            nb0 = __ldg(seg_begin + (nbins - 1 - nxt));
            nb1 = __ldg(seg_begin + (nbins - nxt));
        }
    }
    if (ZERO) {
        __syncwarp();
        if (rel >= 0)
            flag_release(zp.flags + rel, zp.epoch);
    }
}

}  // namespace

cudaError_t launch_o1t(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    using L = O1T;
    const bool zero = a.zflags != nullptr;
    static const int minb = [] {
        const char *v = getenv("MM_O1T_MINB");
        return v ? atoi(v) : O1T_MINB;
    }();
    auto kern = zero ? (minb == 6 ? k_asm_o1t<true, 6> : k_asm_o1t<true, 5>)
                     : (minb == 6 ? k_asm_o1t<false, 6> : k_asm_o1t<false, 5>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
    if (e)
        return e;
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L::WARPS * 32, L::SMEM);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t want = (a.nbins + L::WARPS - 1) / L::WARPS;
    int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    unsigned grid = (unsigned)(want < cap ? (want < 1 ? 1 : want) : cap);
    dev::ZeroPlan zp;
    zp.flags = a.zflags;
    zp.epoch = a.zepoch;
    zp.lookahead = 2 * (int)grid * L::WARPS;
    kern<<<grid, L::WARPS * 32, L::SMEM, s>>>(geo, a.rec, a.seg_begin, (int)a.nbins, a.wscale, a.sigma, a.out, a.ghost,
                                              a.work, zp);
    count_launch();
    return cudaGetLastError();
}

}  // namespace mm
