// FP64 tensor-core (DMMA 8x8x4) mass-matrix assembly: order-2 tensor (k_asm_o2t) and the
// scalar kind of both orders (k_asm_pps).  The order-1 tensor kernel (the c2 headline) lives
// in mm_assemble_o1t.cu.  Algorithm 1 of the paper:
//
//   for each support group (here: a support-window bin, R12)
//     D^{ij} <- 0                                             (alg. line 399)
//     for each batch of K_t = 4 particles                     (eq_D_batches)
//       D^{ij} += A^{ij} B   (dense product over the batch)   (eq_AB_batch)
//     deposit D^{ij} into the node-stencil storage
//
// Operand plan (pair products): the tensor-product B-spline makes W_a W_b a
// product of per-axis pair products, so the block of a bin is ONE product over particles with
// X = q_x q_y rows and Z = q_z s^{ij} columns (36 x 54 for TSC tensor; 9 | 36 x 3 | 6 scalar).
//
// Fragment mapping of mma.sync.m8n8k4.f64 (row.col): lane t holds A[t>>2][t&3],
// B[t&3][t>>2] and D[t>>2][2(t&3)+v]; operands are staged in shared memory with a row
// stride of 36 doubles (the 8 rows x 4 particles of a fragment load hit 2 wavefronts).
#include <cstdlib>

#include "mm_device.cuh"

#ifndef O2T_DYN
#define O2T_DYN 4  // k_asm_o2t: tickets per atomic, runs of consecutive bins per CTA (c3 4.537 ->
                   // 4.474 ms incl. the zero-fill; runs of 2: 4.491)
#endif

#ifndef PPS_DYN
#define PPS_DYN 8  // scalar kernels take bins from the work counter in runs of 8 (c4o1 2.05 -> 1.95 ms,
                   // c4o2 6.41 -> 6.32; runs of 4: 2.47 / 6.29, 16: 1.99 / 6.39); 0: static schedule
#endif

namespace mm {

namespace {

using namespace dev;

// Work ticket (see dev::ticket).
__device__ __forceinline__ int atom_add(int *p, int /*one*/)
{
    return ticket(p);
}

// ---- mbarrier + TMA bulk copy (cp.async.bulk) helpers -------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// One-lane bulk copy global -> shared of `bytes` (multiple of 16), completing on `bar`.
__device__ __forceinline__ void tma_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// ------------------------------------------------ order 2, tensor: pair-product GEMM
// Same factorisation as k_asm_o1t with TSC weights: per axis the 6 unordered pair
// products q(P(i,j)) = w_i w_j (P = [[0,1,2],[1,3,4],[2,4,5]]), so the 27x27x9 block is
//
//   M^c[a][b] = sum_p X_p[6 ux + uy] Z_p[9 uz + c],  u_mu = P(a_mu, b_mu)
//   X = q_x(ux) q_y(uy)  (36 rows),   Z = q_z(uz) s^c  (54 rows)
//
// 36 x 54 = 1944 outputs (vs 10 upper 8x8 tiles x 9 = 5760 MMA entries), 5 x 7 = 35 DMMA
// per batch of 4 particles.  One CTA = one bin at a time, 5 warps: warp w owns the D row
// tile w (7 column tiles, 14 accumulator registers).  Prep of a 32-particle chunk is split
// by rows (warps 0-1: X rows, warps 2-4: Z rows; lane = particle) into a double-buffered
// operand tile, so one CTA barrier per chunk suffices.  Flush: 243 runs (node a, b_x, b_y)
// of 27 contiguous doubles (b_z = 0..2 x 9 comps) of node a's row, each a warp-wide RED
// over values gathered from the stage, three runs per table entry (a, b_x).
struct O2T {
    static constexpr int WARPS = 5;
    static constexpr int XS = 36;                          // row stride (doubles)
    static constexpr int ROWS = 90;                        // 36 X + 54 Z
    static constexpr int TILE = ROWS * XS;                 // one operand buffer
    static constexpr int STAGE = 36 * 54;
    // the stage [36][54] aliases the operand buffer of the bin's last chunk (after a barrier)
    // one record buffer: the next chunk's TMA is issued after the barrier that ends the reads
    static constexpr int DOUBLES = 2 * TILE + 256 + 28 + 2 + 162 + 4;  // xz, recs, rowp, bars, units, q
    static constexpr size_t SMEM = (size_t)DOUBLES * 8;
};

// TSC weights of one axis (R3, R4) with u = xi - (b + 1) in [-1/2, 1/2):
// w0 = (1/2 - u)^2 / 2, w1 = 3/4 - u^2, w2 = (1/2 + u)^2 / 2 (same values as weights2).
__device__ __forceinline__ void weights2u(double xi, double &w0, double &w1, double &w2)
{
    unsigned lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(xi));
    const double u = hi >= 0x3fe00000u ? xi - 1.0 : xi;  // xi >= 1/2 (xi in [0,1)): base 0, else -1
    const double h = 0.5 - u, k = 0.5 + u;
    w0 = (0.5 * h) * h;
    w1 = fma(-u, u, 0.75);
    w2 = (0.5 * k) * k;
}

__global__ void __launch_bounds__(O2T::WARPS * 32, 4) k_asm_o2t(Geo g, const double *__restrict__ rec,
                                                                const int32_t *__restrict__ seg_begin,
                                                                int64_t nbins, double wscale, double sigma,
                                                                double *__restrict__ out, double *__restrict__ ghost,
                                                                int *__restrict__ work, double *__restrict__ dblk)
{
    using L = O2T;
    extern __shared__ __align__(16) double dsm_o2t[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *xzb = dsm_o2t;                                  // [2][90][XS]
    double *srec = xzb + 2 * L::TILE;                       // [32 records][8]
    double *tail = srec + 256;
    double **rowp = reinterpret_cast<double **>(tail);                  // [27]
    uint64_t *bars = reinterpret_cast<uint64_t *>(tail + 28);           // [2]
    int4 *s_unit = reinterpret_cast<int4 *>(tail + 30);                // [81]
    int *q = reinterpret_cast<int *>(tail + 30 + 162);                  // cur, tnext, tnext2, issued
    const int plane = g.n1 * g.n2;
    constexpr int RL = 125 * 9;

    // flush unit u = (a, bx): {a, slot(b - a)*9 at by = bz = 0, stage row offsets 54 X(by) for
    // by = 0..2 (16-bit fields), a_z}; X(by) = 6 P(ax, bx) + P(ay, by), P(i,j) = i + j + [i,j > 0]
    for (int u = threadIdx.x; u < 81; u += blockDim.x) {
        const int a = u / 3, bx = u - 3 * a;
        const int ax = a / 9, ay = (a / 3) % 3, az = a % 3;
        const int slot = (bx - ax + 2) * 25 + (0 - ay + 2) * 5 + (0 - az + 2);
        const int px = ax + bx + (ax && bx);
        int m54[3];
        for (int by = 0; by < 3; ++by)
            m54[by] = 54 * (6 * px + ay + by + (ay && by));
        s_unit[u] = make_int4(a, slot * 9, m54[0] | (m54[1] << 16), m54[2] | (az << 16));
    }
    // O2T_DYN: thread 0 draws runs of O2T_DYN consecutive tickets with one atomic
    int tk = 0, tk_end = 0;
    auto next_ticket = [&]() {
        if (tk == tk_end) {
            tk = atomicAdd(work, O2T_DYN);
            tk_end = tk + O2T_DYN;
        }
        return tk++;
    };
    if (threadIdx.x == 0) {
        q[0] = next_ticket();
        q[1] = next_ticket();
        q[2] = next_ticket();
        q[3] = -1;
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    // lane's stage column offsets for a run, by a_z: 9 P(az, bz) + c with l = 9 bz + c
    const int lbz = lane / 9, lc = lane - 9 * lbz;
    const int noff0 = 9 * lbz + lc;                                    // P(0, bz) = bz
    const int noff1 = 9 * (lbz + 1 + (lbz > 0)) + lc;                  // P(1, bz) = 1, 3, 4
    const int noff2 = 9 * (lbz == 0 ? 2 : lbz + 3) + lc;               // P(2, bz) = 2, 4, 5
    const int d1 = noff1 - noff0, d2 = noff2 - noff0;
    const int kq = lane & 3, rq = lane >> 2;
    const bool arow_ok = 8 * warp + rq < 36;
    const bool b6_ok = rq < 6;  // column tile 6: Z rows 48 + rq < 54
    __syncthreads();
    int bin = q[0];
    int chunk = 0;
    int tn0 = 0, tn1 = 0;  // (thread 0) range of the next bin
    while (bin < nbins) {
        const int b0 = seg_begin[bin], b1 = seg_begin[bin + 1];
        if (threadIdx.x == 0) {
            if (b1 > b0 && q[3] != bin)
                tma_load(srec, rec + 8 * (int64_t)b0, min(32, b1 - b0) * 64, &bars[chunk & 1]);
            tn0 = tn1 = 0;
            if (q[1] < nbins) {
                tn0 = seg_begin[q[1]];
                tn1 = seg_begin[q[1] + 1];
            }
        }
        double acc[7][2];
#pragma unroll
        for (int t = 0; t < 7; ++t)
            acc[t][0] = acc[t][1] = 0.0;
        for (int base = b0; base < b1; base += 32, ++chunk) {
            const int m = min(32, b1 - base);
            double *xz = xzb + (chunk & 1) * L::TILE;
            mbar_wait(&bars[chunk & 1], (chunk >> 1) & 1);
            if (lane < m) {
                const double *r = srec + 8 * lane;
                double *col = xz + lane;
                if (warp < 2) {
                    const double2 xy = *reinterpret_cast<const double2 *>(r);
                    double x0, x1, x2, y0, y1, y2;
                    weights2u(xy.x, x0, x1, x2);
                    weights2u(xy.y, y0, y1, y2);
                    const double qy[6] = {y0 * y0, y0 * y1, y0 * y2, y1 * y1, y1 * y2, y2 * y2};
                    // warp 0: ux = P(0,0), P(0,1), P(0,2); warp 1: P(1,1), P(1,2), P(2,2)
                    const double qa = warp == 0 ? x0 : x1;
                    double qx[3];
                    qx[0] = qa * qa;
                    qx[1] = qa * (warp == 0 ? x1 : x2);
                    qx[2] = (warp == 0 ? x0 : x2) * x2;
                    double *dst = col + 18 * warp * L::XS;
#pragma unroll
                    for (int i = 0; i < 3; ++i)
#pragma unroll
                        for (int j = 0; j < 6; ++j)
                            dst[(6 * i + j) * L::XS] = qx[i] * qy[j];
                } else {
                    const double2 zq = *reinterpret_cast<const double2 *>(r + 2);
                    const double2 bxy = *reinterpret_cast<const double2 *>(r + 4);
                    double s[9];
                    coeff9(zq.y, bxy.x, bxy.y, r[6], wscale, sigma, s);
                    double z0, z1, z2;
                    weights2u(zq.x, z0, z1, z2);
                    // warp 2: uz = P(0,0), P(0,1); warp 3: P(0,2), P(1,1); warp 4: P(1,2), P(2,2)
                    const double za = warp == 2 ? z0 * z0 : (warp == 3 ? z0 * z2 : z1 * z2);
                    const double zb = warp == 2 ? z0 * z1 : (warp == 3 ? z1 * z1 : z2 * z2);
                    double *dst = col + (36 + 18 * (warp - 2)) * L::XS;
#pragma unroll
                    for (int c = 0; c < 9; ++c) {
                        dst[c * L::XS] = za * s[c];
                        dst[(9 + c) * L::XS] = zb * s[c];
                    }
                }
            }
            __syncthreads();
            // every warp is past its reads of the other record buffer: prefetch the next chunk
            if (threadIdx.x == 0) {
                const double *src = nullptr;
                int cnt = 0;
                if (base + 32 < b1) {
                    src = rec + 8 * (int64_t)(base + 32);
                    cnt = min(32, b1 - base - 32);
                } else if (q[1] < nbins && tn1 > tn0) {
                    src = rec + 8 * (int64_t)tn0;
                    cnt = min(32, tn1 - tn0);
                    q[3] = q[1];
                }
                if (cnt)
                    tma_load(srec, src, cnt * 64, &bars[(chunk + 1) & 1]);
            }
            const double *pa = xz + (8 * warp + rq) * L::XS + kq;
            const double *pb = xz + (36 + rq) * L::XS + kq;
            auto batch = [&](int kb) {
                const double av = arow_ok ? pa[kb] : 0.0;
                double bv[7];
#pragma unroll
                for (int nt = 0; nt < 6; ++nt)
                    bv[nt] = pb[8 * nt * L::XS + kb];
                bv[6] = b6_ok ? pb[48 * L::XS + kb] : 0.0;
#pragma unroll
                for (int nt = 0; nt < 7; ++nt)
                    dmma(acc[nt][0], acc[nt][1], av, bv[nt]);
            };
            if (m == 32) {
#pragma unroll
                for (int kb = 0; kb < 32; kb += 4)
                    batch(kb);
            } else {
                for (int kb = 0; kb < m; kb += 4)
                    batch(kb);
            }
        }
        if (b0 == b1) {  // empty bin (rare): advance the ticket queue
            if (dblk) {  // two-phase: an empty bin's block is zero
                double *dp = dblk + (int64_t)bin * (36 * 54);
                for (int e = threadIdx.x; e < 36 * 54; e += L::WARPS * 32)
                    dp[e] = 0.0;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                q[0] = q[1];
                q[1] = q[2];
                if (q[2] < nbins)
                    q[2] = next_ticket();
            }
            __syncthreads();
            bin = q[0];
            continue;
        }
        // ---- stage[X row][Z col] in the operand buffer of the bin's last chunk, once every
        //      warp is done reading it
        __syncthreads();
        double *stage = xzb + ((chunk - 1) & 1) * L::TILE;
        {
            const int mr = 8 * warp + rq;
#pragma unroll
            for (int nt = 0; nt < 7; ++nt)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int nc = 8 * nt + 2 * kq + v;
                    if (mr < 36 && nc < 54)
                        stage[mr * 54 + nc] = acc[nt][v];
                }
        }
        const int bxl = (int)(bin / plane), rem = bin - bxl * plane, bx = g.bx0 + bxl;
        const int by = rem / g.n2, bz = rem - by * g.n2;
        const int fin = bin;
        if (threadIdx.x < 27 && !dblk) {
            const int a = threadIdx.x;
            rowp[a] = row_ptr(g, g.x_begin + bx - 1 + a / 9, wrapi(by + (a / 3) % 3, g.n1), wrapi(bz + a % 3, g.n2),
                              out, ghost, RL);
        }
        if (threadIdx.x == 0) {
            q[0] = q[1];
            q[1] = q[2];
            if (q[2] < nbins)
                q[2] = next_ticket();
        }
        __syncthreads();
        bin = q[0];
        if (dblk) {
            // two-phase deposit (mm_nodesum.cu): the stage is the bin's block D[X row][Z col]
            double *dp = dblk + (int64_t)fin * (36 * 54);
            for (int e = threadIdx.x; e < 36 * 54; e += L::WARPS * 32)
                dp[e] = stage[e];
            continue;
        }
        // ---- flush: runs of 27 contiguous doubles (b_z x comps) of node a's row, three runs
        //      (b_y = 0..2, 5 slots apart) per unit (a, b_x).  The next writes of stage / rowp /
        //      q come after the next chunk barrier.
        if (lane < 27) {
#pragma unroll 2
            for (int u = warp; u < 81; u += L::WARPS) {
                const int4 t = s_unit[u];
                const int az = t.w >> 16;
                const int no = noff0 + (d1 & -(az == 1)) + (d2 & -(az == 2));
                double *p = rowp[t.x] + t.y + lane;
                const double v0 = stage[(t.z & 0xffff) + no];
                const double v1 = stage[(t.z >> 16) + no];
                const double v2 = stage[(t.w & 0xffff) + no];
                red_add(p, v0);  // unconditional: a predicated RED costs a branch (BSSY/BSYNC)
                red_add(p + 45, v1);
                red_add(p + 90, v2);
            }
        }
    }
}

// ------------------------------------------------ scalar kind: pair-product GEMM, warp per bin
// The scalar (MPM-style) mass matrix M[a][b] = sum_p sigma q_p W_a W_b with the pair-product
// factorisation of k_asm_o1t / k_asm_o2t: X = q_x q_y (NX = 9 | 36 rows), Z = q_z sigma q
// (NZ = 3 | 6 rows): D = X Z^T over the particles, MT = 2 | 5 row tiles x one column tile,
// i.e. 2 | 5 DMMA per batch of 4 particles (the node-tile plan: 1 | 10).  One warp per bin
// (static interleaved schedule), the lane's record prefetched one chunk ahead, operands staged
// per warp ([X rows | Z rows][32 particles], zero padding rows), deposit through a table in
// global address order (node a's row, slot(b - a)): 64 | 729 REDs per bin.
template <int ORDER>
struct PPS {
    static constexpr int NU = ORDER == 1 ? 3 : 6;
    static constexpr int NX = NU * NU, NZ = NU;
    static constexpr int MT = (NX + 7) / 8;             // row tiles
    static constexpr int ROWS = 8 * MT + 8;             // X rows (padded) then 8 Z rows (padded)
    static constexpr int XS = 36;                       // row stride (doubles)
    static constexpr int WARP_DOUBLES = ROWS * XS;
    static constexpr int WARPS = 8;
    static constexpr int NA = ORDER == 1 ? 8 : 27;      // support nodes
    static constexpr int NDEP = NA * NA;                // (a, b) entries per bin
    static constexpr int NDEP32 = (NDEP + 31) / 32 * 32;
    static constexpr int L = 2 * ORDER + 1, S = L * L * L;
    static constexpr size_t SMEM = (size_t)WARPS * WARP_DOUBLES * 8 + NDEP32 * 4 + WARPS * 32 * 8;
};

template <int ORDER>
__global__ void __launch_bounds__(PPS<ORDER>::WARPS * 32) k_asm_pps(Geo g, const double *__restrict__ rec,
                                                                   const int32_t *__restrict__ seg_begin,
                                                                   int64_t nbins, int rs, double sigma,
                                                                   double *__restrict__ out,
                                                                   double *__restrict__ ghost,
                                                                   double *__restrict__ dblk,
                                                                   int *__restrict__ work)
{
    using L = PPS<ORDER>;
    extern __shared__ __align__(16) double dsm_pps[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *xz = dsm_pps + warp * L::WARP_DOUBLES;
    int32_t *s_dep = reinterpret_cast<int32_t *>(dsm_pps + L::WARPS * L::WARP_DOUBLES);
    double **s_rowp = reinterpret_cast<double **>(s_dep + L::NDEP32) + warp * 32;
    const int plane = g.n1 * g.n2;

    // deposit table in address order of node a's row: a (5 bits) | slot (7 bits) | stage index
    // x * NZ + z (8 bits); padding entries have a = 31 (skipped)
    for (int e = threadIdx.x; e < L::NDEP32; e += blockDim.x) {
        if (e >= L::NDEP) {
            s_dep[e] = 31;
            continue;
        }
        const int a = e / L::NA, b = e - a * L::NA;
        int ax, ay, az, bx, by, bz, x, z;
        if (ORDER == 1) {
            ax = a >> 2, ay = (a >> 1) & 1, az = a & 1, bx = b >> 2, by = (b >> 1) & 1, bz = b & 1;
            x = 3 * (ax + bx) + (ay + by);
            z = az + bz;
        } else {
            ax = a / 9, ay = (a / 3) % 3, az = a % 3, bx = b / 9, by = (b / 3) % 3, bz = b % 3;
            auto P = [](int i, int j) { return i + j + (i && j); };
            x = 6 * P(ax, bx) + P(ay, by);
            z = P(az, bz);
        }
        const int slot = ((bx - ax + ORDER) * L::L + (by - ay + ORDER)) * L::L + (bz - az + ORDER);
        s_dep[e] = a | (slot << 5) | ((x * L::NZ + z) << 12);
    }
    // zero padding rows (X rows NX..8MT-1, Z rows NZ..7) once
    for (int r = 0; r < L::ROWS; ++r)
        if ((r >= L::NX && r < 8 * L::MT) || r >= 8 * L::MT + L::NZ)
            xz[r * L::XS + lane] = 0.0;
    __syncthreads();

    const int nw = gridDim.x * L::WARPS;
    // PPS_DYN > 0: bins from the work counter, a warp drawing runs of PPS_DYN consecutive bins
    // with one atomic (lane 0); else the static interleaved schedule (warp w: w, w + nw, ...)
    int tk = 0, tk_end = 0;
    auto next_bin_of = [&](int static_next) {
        if (PPS_DYN == 0)
            return static_next;
        int t = 0;
        if (lane == 0) {
            if (tk == tk_end) {
                tk = atomicAdd(work, PPS_DYN > 0 ? PPS_DYN : 1);
                tk_end = tk + (PPS_DYN > 0 ? PPS_DYN : 1);
            }
            t = tk++;
        }
        return __shfl_sync(0xffffffffu, t, 0);
    };
    int bin = next_bin_of(blockIdx.x * L::WARPS + warp);
    int bnext = next_bin_of(bin + nw);
    int b0 = 0, b1 = 0, nb0 = 0, nb1 = 0;
    if (bin < nbins) {
        b0 = __ldg(seg_begin + bin);
        b1 = __ldg(seg_begin + bin + 1);
    }
    if (bnext < nbins) {
        nb0 = __ldg(seg_begin + bnext);
        nb1 = __ldg(seg_begin + bnext + 1);
    }
    double4 ra = make_double4(0, 0, 0, 0);
    if (bin < nbins && b0 + lane < b1)
        ra = ld256(rec + rs * (int64_t)(b0 + lane));
    const int kq = lane & 3, rq = lane >> 2;
    const double *xa = xz + rq * L::XS + kq;
    const double *zb = xz + (8 * L::MT + rq) * L::XS + kq;
    // bin coordinates stepped by the mixed-radix digits of nw (no integer division per bin)
    const int wz = nw % g.n2, wy = (nw / g.n2) % g.n1, wx = nw / plane;
    int cx = bin / plane, cy = (bin - cx * plane) / g.n2, cz = bin - cx * plane - cy * g.n2;
    while (bin < nbins) {
        const int bnn = next_bin_of(bnext + nw);
        int nn0 = 0, nn1 = 0;
        if (bnn < nbins) {
            nn0 = __ldg(seg_begin + bnn);
            nn1 = __ldg(seg_begin + bnn + 1);
        }
        if (PPS_DYN > 0) {
            cx = bin / plane;
            cy = (bin - cx * plane) / g.n2;
            cz = bin - cx * plane - cy * g.n2;
        }
        double acc[L::MT][2];
#pragma unroll
        for (int t = 0; t < L::MT; ++t)
            acc[t][0] = acc[t][1] = 0.0;
        for (int base = b0; base < b1; base += 32) {
            const int m = min(32, b1 - base);
            const double4 ca = ra;
            {
                int64_t p = -1;
                if (base + 32 < b1) {
                    if (base + 32 + lane < b1)
                        p = base + 32 + lane;
                } else if (bnext < nbins && nb0 + lane < nb1) {
                    p = nb0 + lane;
                }
                if (p >= 0)
                    ra = ld256(rec + rs * p);
            }
            __syncwarp();
            {
                double qx[L::NU], qy[L::NU], qz[L::NU];
                const bool live = lane < m;
                if (ORDER == 1) {
                    const double wx0 = 1.0 - ca.x, wx1 = ca.x, wy0 = 1.0 - ca.y, wy1 = ca.y, wz0 = 1.0 - ca.z,
                                 wz1 = ca.z;
                    qx[0] = wx0 * wx0, qx[1] = wx0 * wx1, qx[2] = wx1 * wx1;
                    qy[0] = wy0 * wy0, qy[1] = wy0 * wy1, qy[2] = wy1 * wy1;
                    qz[0] = wz0 * wz0, qz[1] = wz0 * wz1, qz[2] = wz1 * wz1;
                } else {
                    double w[3][3];
                    weights2u(ca.x, w[0][0], w[0][1], w[0][2]);
                    weights2u(ca.y, w[1][0], w[1][1], w[1][2]);
                    weights2u(ca.z, w[2][0], w[2][1], w[2][2]);
                    double *qq[3] = {qx, qy, qz};
#pragma unroll
                    for (int ax = 0; ax < 3; ++ax) {
                        qq[ax][0] = w[ax][0] * w[ax][0];
                        qq[ax][1] = w[ax][0] * w[ax][1];
                        qq[ax][2] = w[ax][0] * w[ax][2];
                        qq[ax][3] = w[ax][1] * w[ax][1];
                        qq[ax][4] = w[ax][1] * w[ax][2];
                        qq[ax][5] = w[ax][2] * w[ax][2];
                    }
                }
                const double sq = live ? sigma * ca.w : 0.0;  // zero past the bin's end: exact +0
                double *col = xz + lane;
#pragma unroll
                for (int i = 0; i < L::NU; ++i)
#pragma unroll
                    for (int j = 0; j < L::NU; ++j)
                        col[(L::NU * i + j) * L::XS] = qx[i] * qy[j];
#pragma unroll
                for (int k = 0; k < L::NU; ++k)
                    col[(8 * L::MT + k) * L::XS] = qz[k] * sq;
            }
            __syncwarp();
            auto batch = [&](int kb) {
                const double bv = zb[kb];
#pragma unroll
                for (int mt = 0; mt < L::MT; ++mt)
                    dmma(acc[mt][0], acc[mt][1], xa[8 * mt * L::XS + kb], bv);
            };
            if (m == 32) {
#pragma unroll
                for (int kb = 0; kb < 32; kb += 4)
                    batch(kb);
            } else {
                for (int kb = 0; kb < m; kb += 4)
                    batch(kb);
            }
        }
        if (b1 > b0) {
            __syncwarp();
            double *stage = xz;  // [NX][NZ] after the last batch
#pragma unroll
            for (int mt = 0; mt < L::MT; ++mt)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int x = 8 * mt + rq, z = 2 * kq + v;
                    if (x < L::NX && z < L::NZ)
                        stage[x * L::NZ + z] = acc[mt][v];
                }
            if (dblk) {
                // two-phase deposit (mm_nodesum.cu): the stage is the bin's block D[x][z]
                __syncwarp();
                double *dp = dblk + (int64_t)bin * (L::NX * L::NZ);
                for (int e = lane; e < L::NX * L::NZ; e += 32)
                    dp[e] = stage[e];
                __syncwarp();
                goto next_bin;
            }
            const int bx = g.bx0 + cx, by = cy, bz = cz;
            if (lane < L::NA) {
                const int a = lane;
                const int ax = ORDER == 1 ? a >> 2 : a / 9, ay = ORDER == 1 ? (a >> 1) & 1 : (a / 3) % 3,
                          az = ORDER == 1 ? a & 1 : a % 3;
                s_rowp[a] = row_ptr(g, g.x_begin + bx - (ORDER - 1) + ax, wrapi(by + ay, g.n1), wrapi(bz + az, g.n2),
                                    out, ghost, L::S);
            }
            __syncwarp();
#pragma unroll 4
            for (int i = 0; i < L::NDEP32; i += 32) {
                const int t = s_dep[i + lane];
                const int a = t & 31;
                if (a < L::NA)
                    red_add(s_rowp[a] + ((t >> 5) & 127), stage[t >> 12]);
            }
            // (the stage spans X rows only, which every chunk's prep rewrites)
        } else {
            if (dblk) {  // two-phase: an empty bin's block is zero
                double *dp = dblk + (int64_t)bin * (L::NX * L::NZ);
                for (int e = lane; e < L::NX * L::NZ; e += 32)
                    dp[e] = 0.0;
            }
            if (bnext < nbins && nb0 + lane < nb1)
                ra = ld256(rec + rs * (int64_t)(nb0 + lane));
        }
    next_bin:
        bin = bnext;
        bnext = bnn;
        cz += wz;
        if (cz >= g.n2) {
            cz -= g.n2;
            ++cy;
        }
        cy += wy;
        if (cy >= g.n1) {
            cy -= g.n1;
            ++cx;
        }
        cx += wx;
        b0 = nb0;
        b1 = nb1;
        nb0 = nn0;
        nb1 = nn1;
    }
}

template <int ORDER>
cudaError_t launch_pps(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    using L = PPS<ORDER>;
    // per call: the attribute is per device/context (a process may drive several GPUs)
    cudaError_t e =
        cudaFuncSetAttribute(k_asm_pps<ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
    if (e)
        return e;
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_asm_pps<ORDER>, L::WARPS * 32, L::SMEM);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t want = (a.nbins + L::WARPS - 1) / L::WARPS;
    int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    unsigned grid = (unsigned)(want < cap ? (want < 1 ? 1 : want) : cap);
    k_asm_pps<ORDER><<<grid, L::WARPS * 32, L::SMEM, s>>>(geo, a.rec, a.seg_begin, a.nbins, a.rec_stride, a.sigma,
                                                          a.out, a.ghost, static_cast<double *>(a.dblk), a.work);
    count_launch();
    return cudaGetLastError();
}

// Optional cap on resident assembly CTAs per SM (MM_ASM_CTAS_PER_SM): leaves room for a
// concurrently running sort on another stream.
inline int cta_cap()
{
    static const int cap = [] {
        const char *v = getenv("MM_ASM_CTAS_PER_SM");
        return v ? atoi(v) : 0;
    }();
    return cap;
}

cudaError_t launch_o2t(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{

    using L = O2T;
    // per call: the attribute is per device/context (a process may drive several GPUs)
    cudaError_t e = cudaFuncSetAttribute(k_asm_o2t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
    if (e)
        return e;
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_asm_o2t, L::WARPS * 32, L::SMEM);
    if (cta_cap() > 0 && per_sm > cta_cap())
        per_sm = cta_cap();
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    unsigned grid = (unsigned)(a.nbins < cap ? (a.nbins < 1 ? 1 : a.nbins) : cap);
    k_asm_o2t<<<grid, L::WARPS * 32, L::SMEM, s>>>(geo, a.rec, a.seg_begin, a.nbins, a.wscale, a.sigma, a.out,
                                                   a.ghost, a.work, static_cast<double *>(a.dblk));
    count_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_o1t(const Geo &geo, const AsmArgs &a, cudaStream_t s);  // mm_assemble_o1t.cu

// In-kernel first-writer zeroing (dev::ZeroPlan) is implemented by k_asm_o1t; measured slower
// than the memset, so it is off unless MM_ZERO_O1=1 (A/B measurement, tests).
bool zeroes_inside(int order, int ncomp, int tf32)
{
    static const int z1 = [] {
        const char *v = getenv("MM_ZERO_O1");
        return v ? atoi(v) : 0;
    }();
    return !tf32 && ncomp == 9 && order == 1 && z1;
}

cudaError_t assemble_fp64_enqueue(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    if (a.nbins == 0)
        return cudaSuccess;
    if (geo.order == 1)
        return a.ncomp == 9 ? launch_o1t(geo, a, s) : launch_pps<1>(geo, a, s);
    return a.ncomp == 9 ? launch_o2t(geo, a, s) : launch_pps<2>(geo, a, s);
}

}  // namespace mm
