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

// The same with an L2 evict-first policy (records are streamed once; the L2 should keep the
// output rows the REDs revisit).
__device__ __forceinline__ void tma_load_ef(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
    asm volatile(
        "{\n\t.reg .b64 pol;\n\t"
        "createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n\t"
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n\t}" ::"r"(
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
// per batch of 4 particles.
//
// Deposit with z-segment ownership: a CTA owns a segment of SEG consecutive
// bins along z (same x, y window) and folds each finished bin into a shared-memory RING of
// node planes, ring[slot][X pair 36][dz 5][c 9] (the z pair of the block is expanded into its
// ordered (a_z, b_z): row plane z_bin + a_z, offset dz = b_z - a_z; x and y stay as pairs).
// Node plane z_bin receives nothing from later bins of the segment once bin z_bin is done, so
// it is flushed then: 9 rows x 9 (b_x, b_y) runs of 45 contiguous doubles (5 dz x 9 comps of
// the row), REDs only for the dz present.  An interior plane costs 3645 REDs where the bins
// alone would issue 6561 each (the 3 bins that touch a row add their dz overlap in shared
// memory): 729 (5 + 4/SEG) REDs per bin.
//
// Warp specialisation, 8 warps per CTA:
//   compute warps 0-4: warp w owns the D row tile w (7 column tiles, 14 accumulators); the prep
//     of a 32-particle chunk is split by rows (warps 0-1: X rows, 2-4: Z rows; lane = particle)
//     into a double-buffered operand tile; records TMA-staged one chunk ahead; after a bin the
//     block is staged and folded into the ring; the finished plane is handed over (mbarrier
//     full[slot]) with a descriptor.
//   flush warps 5-7: first-writer zeroing of the output rows (mm_device.cuh), flag waits, the
//     REDs of a handed-over plane, zeroing of its ring slot, then empty[slot].
// Four ring slots: a plane's flush overlaps the next bin's DMMAs (bin z touches planes z..z+2,
// the slot of plane z is reused by plane z+4, first touched by bin z+2).  Segments are taken
// by tickets in descending order of (z segment, x, y): concurrent CTAs work at the same z on
// neighbouring (x, y) windows, so the rows they reduce into stay in L2.
struct O2T {
    static constexpr int CWARPS = 5, FWARPS = 3, WARPS = CWARPS + FWARPS;
    static constexpr int CTHREADS = 32 * CWARPS, FTHREADS = 32 * FWARPS;
    static constexpr int XS = 36;                          // row stride (doubles)
    static constexpr int ROWS = 90;                        // 36 X + 54 Z
    static constexpr int TILE = ROWS * XS;                 // one operand buffer
    static constexpr int NSLOT = 4;                        // ring slots
    static constexpr int PLANE = 36 * 45;                  // one ring plane
    static constexpr int NRUN = 81, RUNLEN = 45;
    // the stage [36][54] of a finished bin aliases the operand buffer of its last chunk
    // layout (doubles): xzb [2][TILE] | ring [NSLOT][PLANE] | srec [32][8] | rowp [9] + pad
    //                   | bars [2 + 2 NSLOT] | runs (int4) [81] | pdesc (int4 x 2) [NSLOT] | q (int) [4]
    static constexpr int OFF_RING = 2 * TILE, OFF_REC = OFF_RING + NSLOT * PLANE, OFF_ROWP = OFF_REC + 256,
                         OFF_BARS = OFF_ROWP + 10, OFF_RUNS = OFF_BARS + 2 + 2 * NSLOT, OFF_DESC = OFF_RUNS + 162,
                         OFF_Q = OFF_DESC + 4 * NSLOT;
    static constexpr size_t SMEM = (size_t)(OFF_Q + 2) * 8;
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



__device__ __forceinline__ void named_bar(int id, int n)
{
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// mbarrier wait with back-off: a waiting warp must not take issue slots from the warps it waits for.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity)
{
    uint32_t ok;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok)
            return;
        __nanosleep(100);
    }
}

// Segment of ticket t (descending order of (z segment, bin plane x, y)).
struct SegPos {
    int zsi, bxl, by;
};
__device__ __forceinline__ SegPos seg_of(int t, int nseg, int npencil, int n1)
{
    const int sg = nseg - 1 - t;
    SegPos p;
    p.zsi = sg / npencil;
    const int pencil = sg - p.zsi * npencil;
    p.bxl = pencil / n1;
    p.by = pencil - p.bxl * n1;
    return p;
}

template <int SEG>
__global__ void __launch_bounds__(O2T::WARPS * 32, 2) k_asm_o2t(Geo g, const double *__restrict__ rec,
                                                                const int32_t *__restrict__ seg_begin, int nbins,
                                                                double wscale, double sigma,
                                                                double *__restrict__ out, double *__restrict__ ghost,
                                                                int *__restrict__ work, ZeroPlan zp)
{
    using L = O2T;
    extern __shared__ __align__(16) double dsm_o2t[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double *xzb = dsm_o2t;                                                   // [2][90][XS]
    double *ring = dsm_o2t + L::OFF_RING;                                    // [NSLOT][36][45]
    double *srec = dsm_o2t + L::OFF_REC;                                     // [32 records][8]
    double **rowp = reinterpret_cast<double **>(dsm_o2t + L::OFF_ROWP);      // [9] rows of a plane
    uint64_t *bars = reinterpret_cast<uint64_t *>(dsm_o2t + L::OFF_BARS);    // [2] TMA
    uint64_t *full = bars + 2, *empty = bars + 2 + L::NSLOT;                 // [NSLOT] each
    int4 *runs = reinterpret_cast<int4 *>(dsm_o2t + L::OFF_RUNS);            // [81]
    int4 *pdesc = reinterpret_cast<int4 *>(dsm_o2t + L::OFF_DESC);           // [NSLOT][2]
    int *q = reinterpret_cast<int *>(dsm_o2t + L::OFF_Q);                    // ticket
    constexpr int RL = 125 * 9;
    const int nzs = (g.n2 + SEG - 1) / SEG;
    const int npencil = nbins / g.n2;
    const int nseg = npencil * nzs;

    // flush run r = (row (ax, ay), b_x, b_y): {row index 3 ax + ay, row offset of the dz = -2
    // slot of (b_x - ax, b_y - ay) (x 9), ring offset of the X pair 6 P(ax, bx) + P(ay, by) (x 45)}
    for (int r = tid; r < L::NRUN; r += blockDim.x) {
        const int row = r / 9, bb = r - 9 * row, ax = row / 3, ay = row - 3 * ax, bx = bb / 3, by = bb - 3 * bx;
        const int slot = (bx - ax + 2) * 25 + (by - ay + 2) * 5;
        const int px = ax + bx + (ax && bx), py = ay + by + (ay && by);
        runs[r] = make_int4(row, 9 * slot, 45 * (6 * px + py), 0);
    }
    for (int e = tid; e < L::NSLOT * L::PLANE; e += blockDim.x)
        ring[e] = 0.0;
    if (tid == 0) {
        q[0] = ticket(work);
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        for (int k = 0; k < L::NSLOT; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp >= L::CWARPS) {
        // ================================ flush warps ================================
        const int ft = tid - L::CTHREADS, fw = warp - L::CWARPS;
        // zero task of ticket ts: the rows first touched by its segment (lookahead 0: zeroed
        // right before its first flush, while they are still needed in L2), all flush threads
        // per row; then one thread publishes them
        auto zero_seg = [&](int ts, bool release) {
            const SegPos sp = seg_of(ts, nseg, npencil, g.n1);
            const int z0 = sp.zsi * SEG, z1 = min(z0 + SEG, g.n2);
            const int bin0 = (sp.bxl * g.n1 + sp.by) * g.n2;
            for (int bz = z0; bz < z1; ++bz) {
                int ux[3], uy[3], uz[3], nx, ny, nz;
                const int cnt = first_rows3(g, bin0 + bz, ux, uy, uz, nx, ny, nz);
                for (int k = 0; k < cnt; ++k) {
                    const int ix = k / (ny * nz), r = k - ix * ny * nz, iy = r / nz, iz = r - iy * nz;
                    const int X = g.x_begin + (ix == 0 ? ux[0] : (ix == 1 ? ux[1] : ux[2]));
                    const int Y = iy == 0 ? uy[0] : (iy == 1 ? uy[1] : uy[2]);
                    const int Z = iz == 0 ? uz[0] : (iz == 1 ? uz[1] : uz[2]);
                    if (!release) {
                        double *p = row_ptr(g, X, Y, Z, out, ghost, RL);
                        for (int e = ft; e < RL; e += L::FTHREADS)
                            p[e] = 0.0;
                    } else if (ft == 0) {
                        flag_release(zp.flags + row_id(g, X, Y, Z), zp.epoch);
                    }
                }
            }
        };
        for (uint32_t i = 0;; ++i) {
            const int sl = i % L::NSLOT;
            mbar_wait_sleep(&full[sl], (i / L::NSLOT) & 1);
            const int4 d0 = pdesc[2 * sl], d1 = pdesc[2 * sl + 1];
            // d0 = {X0 (global x of the window's first row), y, z (unwrapped), dz_lo | dz_hi << 8}
            // d1 = {kind: 0 plane, 1 zero task of ticket d1.y, 2 terminate, ticket, 0, 0}
            if (d1.x == 2)
                break;
            if (d1.x == 1) {
                zero_seg(d1.y, false);
                named_bar(2, L::FTHREADS);
                zero_seg(d1.y, true);
            } else {
                const int Z = d0.z % g.n2;
                if (ft < 9) {
                    const int X = d0.x + ft / 3, Y = wrapi(d0.y + ft % 3, g.n1);
                    rowp[ft] = row_ptr(g, X, Y, Z, out, ghost, RL);
                    if (zp.flags) {
                        const int32_t *f = zp.flags + row_id(g, X, Y, Z);
                        while (flag_acquire(f) != zp.epoch)
                            __nanosleep(64);
                    }
                }
                named_bar(2, L::FTHREADS);
                const double *rp = ring + sl * L::PLANE;
                const int lo = 9 * ((d0.w & 0xff) - 128 + 2), hi = 9 * ((d0.w >> 8) - 128 + 3);
                const bool ok0 = lane >= lo && lane < hi, ok1 = lane + 32 >= lo && lane + 32 < hi && lane < 13;
                const int l1 = lane < 13 ? 32 + lane : 44;
                // 27 runs per warp, 3 at a time: all loads first, then the 6 REDs
                for (int r = fw; r < L::NRUN; r += 3 * L::FWARPS) {
                    double *p[3];
                    double v0[3], v1[3];
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        const int4 u = runs[r + j * L::FWARPS];
                        p[j] = rowp[u.x] + u.y;
                        v0[j] = rp[u.z + lane];
                        v1[j] = rp[u.z + l1];
                    }
#pragma unroll
                    for (int j = 0; j < 3; ++j) {
                        red_add_if(p[j] + lane, v0[j], ok0);
                        red_add_if(p[j] + l1, v1[j], ok1);
                    }
                }
                named_bar(2, L::FTHREADS);
                double *wp = ring + sl * L::PLANE;
                for (int e = ft; e < L::PLANE; e += L::FTHREADS)
                    wp[e] = 0.0;
            }
            named_bar(2, L::FTHREADS);
            if (ft == 0)
                mbar_arrive(&empty[sl]);
        }
        return;
    }

    // ================================ compute warps ================================
    const int kq = lane & 3, rq = lane >> 2;
    const bool arow_ok = 8 * warp + rq < 36;
    const bool b6_ok = rq < 6;  // column tile 6: Z rows 48 + rq < 54
    int t = q[0];
    int chunk = 0;
    uint32_t pi = 0;  // CTA-local hand-over sequence (planes and zero tasks): item pi uses slot pi % NSLOT
    // hand item pl (descriptor) to the flush warps; all compute threads are past its ring adds
    auto publish = [&](uint32_t pl, int4 d0, int4 d1) {
        if (tid == 0) {
            pdesc[2 * (pl % L::NSLOT)] = d0;
            pdesc[2 * (pl % L::NSLOT) + 1] = d1;
            mbar_arrive(&full[pl % L::NSLOT]);
        }
    };
    // wait until the slot of item pl is free (its previous item flushed, its ring plane zeroed)
    auto acquire = [&](uint32_t pl) {
        if (pl >= L::NSLOT)
            mbar_wait_sleep(&empty[pl % L::NSLOT], ((pl / L::NSLOT) - 1) & 1);
    };
    while (t < nseg) {
        const SegPos sp = seg_of(t, nseg, npencil, g.n1);
        const int bx = g.bx0 + sp.bxl, by = sp.by;
        const int zs0 = sp.zsi * SEG, zs1 = min(zs0 + SEG, g.n2);
        const int bin0 = (sp.bxl * g.n1 + by) * g.n2;
        const int X0 = g.x_begin + bx - 1;
        int nb1 = 0;        // (thread 0) end of the next bin
        int pending = -1;   // (thread 0) bin whose first chunk is already in flight
        if (zp.flags) {     // zero task of this segment first: the flush warps run it during bin 0
            acquire(pi);
            publish(pi, make_int4(0, 0, 0, 0), make_int4(1, t, 0, 0));
            ++pi;
        }
        const uint32_t pbase = pi;
        for (int bz = zs0; bz < zs1; ++bz) {
            const int bin = bin0 + bz;
            const int b0 = seg_begin[bin], b1 = seg_begin[bin + 1];
            if (tid == 0) {
                nb1 = bz + 1 < zs1 ? seg_begin[bin + 2] : 0;
                if (b1 > b0 && pending != bin)
                    tma_load_ef(srec, rec + 8 * (int64_t)b0, min(32, b1 - b0) * 64, &bars[chunk & 1]);
            }
            double acc[7][2];
#pragma unroll
            for (int i = 0; i < 7; ++i)
                acc[i][0] = acc[i][1] = 0.0;
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
                named_bar(1, L::CTHREADS);
                // every compute warp is past its reads of the record buffer: prefetch the next chunk
                if (tid == 0) {
                    const double *src = nullptr;
                    int cnt = 0;
                    if (base + 32 < b1) {
                        src = rec + 8 * (int64_t)(base + 32);
                        cnt = min(32, b1 - base - 32);
                    } else if (nb1 > b1) {
                        src = rec + 8 * (int64_t)b1;  // first chunk of the next bin of the segment
                        cnt = min(32, nb1 - b1);
                        pending = bin + 1;
                    }
                    if (cnt)
                        tma_load_ef(srec, src, cnt * 64, &bars[(chunk + 1) & 1]);
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
            // ring slots of this bin's rows z = bz + a_z: items pz, pz + 1, pz + 2 (the first
            // bin of a segment takes all three, later bins the new top plane only)
            const uint32_t pz = pbase + (uint32_t)(bz - zs0);
            if (bz == zs0) {
                acquire(pz);
                acquire(pz + 1);
            }
            acquire(pz + 2);
            if (b1 > b0) {
                // ---- stage [X row][Z col] in the operand buffer of the bin's last chunk, then
                //      fold it into the ring: thread = (X row, c), the 9 ordered z pairs
                named_bar(1, L::CTHREADS);
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
                named_bar(1, L::CTHREADS);
                double *r0 = ring + (pz % L::NSLOT) * L::PLANE;        // row z = bz (a_z = 0)
                double *r1 = ring + ((pz + 1) % L::NSLOT) * L::PLANE;  // a_z = 1
                double *r2 = ring + ((pz + 2) % L::NSLOT) * L::PLANE;  // a_z = 2
                for (int u = tid; u < 36 * 9; u += L::CTHREADS) {
                    const int mr = u / 9, c = u - 9 * mr;
                    const double *st = stage + mr * 54 + c;
                    double v[6];
#pragma unroll
                    for (int k = 0; k < 6; ++k)
                        v[k] = st[9 * k];
                    const int o = mr * 45 + c;
                    // dz = b_z - a_z (index dz + 2); pair P(a_z, b_z)
                    r0[o + 9 * 2] += v[0];
                    r0[o + 9 * 3] += v[1];
                    r0[o + 9 * 4] += v[2];
                    r1[o + 9 * 1] += v[1];
                    r1[o + 9 * 2] += v[3];
                    r1[o + 9 * 3] += v[4];
                    r2[o + 9 * 0] += v[2];
                    r2[o + 9 * 1] += v[4];
                    r2[o + 9 * 2] += v[5];
                }
            }
            named_bar(1, L::CTHREADS);  // ring adds done before the hand-over (and before the
                                        // next chunk's prep reuses the stage buffer)
            // plane z = bz is complete: bins max(zs0, bz - 2) .. bz contributed (a_z = bz - bin)
            const int dlo = -min(2, bz - zs0);
            publish(pz, make_int4(X0, by, bz, (dlo + 128) | ((2 + 128) << 8)), make_int4(0, 0, 0, 0));
        }
        // planes above the segment: z = zs1 (bins zs1-2, zs1-1: dz in [-2 or -1, 1]), zs1 + 1
        // (bin zs1-1: dz in [-2, 0])
        {
            const int n = zs1 - zs0;
            const uint32_t pz = pbase + (uint32_t)n;
            publish(pz, make_int4(X0, by, zs1, ((n >= 2 ? -2 : -1) + 128) | ((1 + 128) << 8)), make_int4(0, 0, 0, 0));
            publish(pz + 1, make_int4(X0, by, zs1 + 1, (-2 + 128) | ((0 + 128) << 8)), make_int4(0, 0, 0, 0));
            pi = pz + 2;
        }
        // next ticket, taken only now: a ticket is never held unstarted (its zero task runs at
        // its start, so no CTA can hold back rows others wait for)
        if (tid == 0)
            q[0] = ticket(work);
        named_bar(1, L::CTHREADS);
        t = q[0];
        named_bar(1, L::CTHREADS);  // every compute thread has read q[0]
    }
    // terminate the flush warps (after the slot is free, like any item)
    acquire(pi);
    publish(pi, make_int4(0, 0, 0, 0), make_int4(2, 0, 0, 0));
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
                                                                   double *__restrict__ ghost)
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
    int bin = blockIdx.x * L::WARPS + warp;
    int b0 = 0, b1 = 0, nb0 = 0, nb1 = 0;
    if (bin < nbins) {
        b0 = __ldg(seg_begin + bin);
        b1 = __ldg(seg_begin + bin + 1);
    }
    if (bin + nw < nbins) {
        nb0 = __ldg(seg_begin + bin + nw);
        nb1 = __ldg(seg_begin + bin + nw + 1);
    }
    double4 ra = make_double4(0, 0, 0, 0);
    if (bin < nbins && b0 + lane < b1)
        ra = ld256(rec + rs * (int64_t)(b0 + lane));
    const int kq = lane & 3, rq = lane >> 2;
    const double *xa = xz + rq * L::XS + kq;
    const double *zb = xz + (8 * L::MT + rq) * L::XS + kq;
    while (bin < nbins) {
        int nn0 = 0, nn1 = 0;
        if (bin + 2 * nw < nbins) {
            nn0 = __ldg(seg_begin + bin + 2 * nw);
            nn1 = __ldg(seg_begin + bin + 2 * nw + 1);
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
                } else if (bin + nw < nbins && nb0 + lane < nb1) {
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
            const int bxl = bin / plane, rem = bin - bxl * plane, bx = g.bx0 + bxl;
            const int by = rem / g.n2, bz = rem - by * g.n2;
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
        } else if (bin + nw < nbins && nb0 + lane < nb1) {
            ra = ld256(rec + rs * (int64_t)(nb0 + lane));
        }
        bin += nw;
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
                                                          a.out, a.ghost);
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
    // bins per z segment (MM_O2T_SEG = 4 | 8 | 16, default 8)
    static const int seg = [] {
        const char *v = getenv("MM_O2T_SEG");
        const int k = v ? atoi(v) : 8;
        return k == 4 || k == 16 ? k : 8;
    }();
    auto kern = seg == 4 ? k_asm_o2t<4> : (seg == 16 ? k_asm_o2t<16> : k_asm_o2t<8>);
    // per call: the attribute is per device/context (a process may drive several GPUs)
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
    if (e)
        return e;
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, L::WARPS * 32, L::SMEM);
    if (cta_cap() > 0 && per_sm > cta_cap())
        per_sm = cta_cap();
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nseg = a.nbins / geo.n2 * ((geo.n2 + seg - 1) / seg);
    int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    unsigned grid = (unsigned)(nseg < cap ? (nseg < 1 ? 1 : nseg) : cap);
    dev::ZeroPlan zp;
    zp.flags = a.zflags;
    zp.epoch = a.zepoch;
    zp.lookahead = 0;
    kern<<<grid, L::WARPS * 32, L::SMEM, s>>>(geo, a.rec, a.seg_begin, (int)a.nbins, a.wscale, a.sigma, a.out, a.ghost,
                                              a.work, zp);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_o1t(const Geo &geo, const AsmArgs &a, cudaStream_t s);  // mm_assemble_o1t.cu

// MM_ZERO_O1 / MM_ZERO_O2 = 0 | 1 override the defaults (A/B measurement).
bool zeroes_inside(int order, int ncomp, int tf32)
{
    static const int z1 = [] {
        const char *v = getenv("MM_ZERO_O1");
        return v ? atoi(v) : 0;
    }();
    static const int z2 = [] {
        const char *v = getenv("MM_ZERO_O2");
        return v ? atoi(v) : 1;
    }();
    return !tf32 && ncomp == 9 && ((order == 1 && z1) || (order == 2 && z2));
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
