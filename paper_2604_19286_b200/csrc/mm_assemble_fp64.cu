// FP64 tensor-core (DMMA 8x8x4) mass-matrix assembly for first- and
// second-order B-splines.  Algorithm 1 of the paper:
//
//   for each support group (here: a support-window bin, R12)
//     D^{ij} <- 0                                             (alg. line 399)
//     for each batch of K_t = 4 particles                     (eq_D_batches)
//       D^{ij} += A^{ij} B   (dense product over the batch)   (eq_AB_batch)
//     deposit D^{ij} into the node-stencil storage
//
// Two operand plans:
//  * pair-product (default for the tensor kind; k_asm_o1t, k_asm_o2t): the tensor-product
//    B-spline makes W_a W_b a product of per-axis pair products, so the block of a bin is
//    ONE product over particles with X = q_x q_y rows and Z = q_z s^{ij} columns
//    (9 x 27 | 36 x 54 outputs) -- see the comments at O1T / O2T;
//  * node tiles (the paper's plan; scalar kind, and MM_ASM_LEGACY=1): rows = support nodes,
//    A = W s^{ij}, B = W^T per component (one 8x8 tile | 10 upper 8x8 tiles).
//
// Fragment mapping of mma.sync.m8n8k4.f64 (row.col): lane t holds A[t>>2][t&3],
// B[t&3][t>>2] and D[t>>2][2(t&3)+v]; operands are staged in shared memory with a row
// stride of 36 doubles (the 8 rows x 4 particles of a fragment load hit 2 wavefronts).
//
// Phases of every kernel: prep (one lane per particle of a chunk: s^{ij} from the record
// (alpha, eq_alpha_matrix) and the weights / products into shared memory), batches (DMMA,
// accumulators in registers), deposit (D staged in shared memory, FP64 REDs in global
// address order through a table, node-row pointers broadcast by shuffles).
#include <cstdlib>

#include "mm_internal.cuh"

namespace mm {

namespace {

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// 256-bit read-only record load (LDG.E.ENL2.256 on sm_100a).
__device__ __forceinline__ double4 ld256(const double *p)
{
    double4 v;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p));
    return v;
}

// Fire-and-forget FP64 reduction into GLOBAL memory (REDG.E.ADD.F64.RN).  Explicit PTX:
// pointers that travel through shuffles/shared memory are generic to the compiler,
// which would otherwise emit a generic ATOM with a shared-memory CAS fallback.
__device__ __forceinline__ void red_add(double *p, double v)
{
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// v != +-0 as an integer test on the two 32-bit halves: a DSETP would occupy the FP64
// pipe that the DMMAs need (ptxas turns a 64-bit integer compare of the bits back into one).
__device__ __forceinline__ bool nonzero_bits(double v)
{
    unsigned lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
    return (lo | (hi << 1)) != 0u;
}

__device__ __forceinline__ int wrapi(int i, int n)
{
    return i < 0 ? i + n : (i >= n ? i - n : i);
}

__device__ __forceinline__ double *shfl_ptr(double *p, int src)
{
    unsigned long long v = (unsigned long long)p;
    unsigned lo = __shfl_sync(0xffffffffu, (unsigned)v, src), hi = __shfl_sync(0xffffffffu, (unsigned)(v >> 32), src);
    return (double *)(((unsigned long long)hi << 32) | lo);
}

// Base address of node row (X unwrapped global, Y/Z wrapped); rowlen = S*C.
__device__ __forceinline__ double *row_ptr(const Geo &g, int X, int Y, int Z, double *out, double *ghost,
                                           int rowlen)
{
    if (g.periodic_x) {
        X = wrapi(X, g.n0);
        return out + ((int64_t)(X * g.n1 + Y) * g.n2 + Z) * rowlen;
    }
    int xl = X - g.x_begin;
    if (xl >= 0 && X < g.x_end)
        return out + ((int64_t)(xl * g.n1 + Y) * g.n2 + Z) * rowlen;
    int plane = (g.order == 1) ? 0 : (X < g.x_begin ? 0 : 1 + (X - g.x_end));
    return ghost + ((int64_t)(plane * g.n1 + Y) * g.n2 + Z) * rowlen;
}

// s^{ij} = sigma q alpha^{ij}, alpha = (delta + omega omega^T + eps omega)/(1+|omega|^2)
// (eq_alpha_matrix with -C(omega)_{ij} = eps_{ijk} omega_k).
template <int NC>
__device__ __forceinline__ void coeff(double q, double Bx, double By, double Bz, double wscale, double sigma,
                                      double s[NC])
{
    if (NC == 1) {
        s[0] = sigma * q;
    } else {
        // FP64 SIMT work shares the pipe with the DMMAs, so this is written for few
        // instructions: f = sigma q / d by a Newton-refined reciprocal, then one FMA per
        // component with f*omega:  s_ij = (f omega_i) omega_j + f delta_ij + eps_ijk f omega_k
        const double o0 = wscale * Bx, o1 = wscale * By, o2 = wscale * Bz;
        const double d = fma(o0, o0, fma(o1, o1, fma(o2, o2, 1.0)));
        double r;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
        r = fma(r, fma(-d, r, 1.0), r);
        r = fma(r, fma(-d, r, 1.0), r);
        const double f = (sigma * q) * r;
        const double f0 = f * o0, f1 = f * o1, f2 = f * o2;
        s[0] = fma(f0, o0, f);
        s[1] = fma(f0, o1, f2);
        s[2] = fma(f0, o2, -f1);
        s[3] = fma(f1, o0, -f2);
        s[4] = fma(f1, o1, f);
        s[5] = fma(f1, o2, f0);
        s[6] = fma(f2, o0, f1);
        s[7] = fma(f2, o1, -f0);
        s[8] = fma(f2, o2, f);
    }
}

// Per-axis B-spline weights at the support nodes:
// w_k = phi(xi - (b + k)).
__device__ __forceinline__ void weights1(double xi, double w[2])
{
    w[0] = 1.0 - xi;  // phi1(xi)
    w[1] = xi;        // phi1(xi - 1) = 1 - |xi - 1| = xi for xi in [0, 1) (up to rounding of 1 - xi)
}

__device__ __forceinline__ void weights2(double xi, double w[3])
{
    double b = xi >= 0.5 ? 0.0 : -1.0;  // R4: tie -> base 0
    double t0 = fabs(xi - b), t1 = xi - (b + 1.0), t2 = fabs(xi - (b + 2.0));
    w[0] = 0.5 * (1.5 - t0) * (1.5 - t0);  // 1/2 < |t0| <= 3/2
    w[1] = 0.75 - t1 * t1;                 // |t1| <= 1/2
    w[2] = 0.5 * (1.5 - t2) * (1.5 - t2);  // 1/2 <= |t2| <= 3/2
}

// Work ticket: atom.inc with limit 2^31-1 (== +1 for any reachable count).  Unlike atom.add,
// ptxas does not warp-aggregate inc (it is not associative), so no shuffle of the result
// is placed right after the atomic and the ticket can be requested one bin ahead.
__device__ __forceinline__ int atom_add(int *p, int /*one*/)
{
    unsigned r;
    asm volatile("atom.global.inc.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(0x7fffffffu) : "memory");
    return (int)r;
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

constexpr int WARPS = 8;

// ---- diagnostics build (-DMM_EXPERIMENT_TIMERS): per-phase SM cycles of the order-1 kernel
#ifdef MM_EXPERIMENT_TIMERS
__device__ unsigned long long g_phase[4];  // 0 TMA wait, 1 prep, 2 batches, 3 deposit/other
#define MM_TDECL unsigned long long t_acc[4] = {0, 0, 0, 0}, t_last = clock64();
#define MM_TMARK(k)                                  \
    do {                                             \
        unsigned long long t_now = clock64();        \
        t_acc[(k)] += t_now - t_last;                \
        t_last = t_now;                              \
    } while (0)
#define MM_TFLUSH()                                  \
    do {                                             \
        if (lane == 0)                               \
            for (int k = 0; k < 4; ++k)              \
                atomicAdd(&g_phase[k], t_acc[k]);    \
    } while (0)
#else
#define MM_TDECL
#define MM_TMARK(k)
#define MM_TFLUSH()
#endif

// ---------------------------------------------------------------- order 1
// Shared memory per warp (doubles):
//   sh_w [8 nodes][WS]  node-major, WS = 36: batch reads hit 2 wavefronts (minimum)
//   sh_s [32][SS]       SS = 10 (even -> 16-B aligned pairs for LDS.128)
//   stage [8][8][NC]    deposit staging (aliases the above)
template <int NC>
struct O1 {
    static constexpr int WS = 36;
    static constexpr int SS = NC == 9 ? 10 : 2;
    static constexpr int PREP = 8 * WS + 32 * SS;
    static constexpr int STAGE = 64 * NC;
    static constexpr int SIZE = PREP > STAGE ? PREP : STAGE;
    static constexpr int NDEP = 64 * NC / 32;  // deposit elements per lane
    static constexpr size_t SMEM = (size_t)(WARPS * 2 * 256 + WARPS * SIZE + WARPS * 2) * 8 + 64 * NC * 4;
};

template <int NC>
__global__ void __launch_bounds__(WARPS * 32, 3) k_asm_o1(Geo g, const double *__restrict__ rec,
                                                          const int32_t *__restrict__ seg_begin, int64_t nbins,
                                                          double wscale, double sigma, double *__restrict__ out,
                                                          double *__restrict__ ghost, int *__restrict__ work)
{
    using L = O1<NC>;
    // dynamic shared memory: [WARPS][2][256] TMA-staged record chunks | [WARPS][SIZE] prep/stage |
    // [WARPS][2] mbarriers | [64*NC] deposit table
    extern __shared__ __align__(128) double dsm1[];
    double(*s_rec)[2][32 * 8] = reinterpret_cast<double(*)[2][32 * 8]>(dsm1);
    double(*smem)[L::SIZE] = reinterpret_cast<double(*)[L::SIZE]>(dsm1 + WARPS * 2 * 256);
    uint64_t(*s_bar)[2] = reinterpret_cast<uint64_t(*)[2]>(dsm1 + WARPS * 2 * 256 + WARPS * L::SIZE);
    int32_t *s_tab = reinterpret_cast<int32_t *>(dsm1 + WARPS * 2 * 256 + WARPS * L::SIZE + WARPS * 2);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *sm = smem[warp];
    double *sh_w = sm;
    double *sh_s = sm + 8 * L::WS;
    const int plane = g.n1 * g.n2;
    constexpr int RL = 27 * NC;
    (void)work;

    // deposit table (per CTA): element e of D[a][b][c] in address order ->
    // node a (3 bits) | offset (slot*NC + c) within node a's row
    for (int e = threadIdx.x; e < 64 * NC; e += blockDim.x) {
        const int a = e / (8 * NC), rr = e - a * 8 * NC, b = rr / NC, c = rr - b * NC;
        const int slot = ((b >> 2) - (a >> 2) + 1) * 9 + (((b >> 1) & 1) - ((a >> 1) & 1) + 1) * 3 + ((b & 1) - (a & 1) + 1);
        s_tab[e] = a | ((slot * NC + c) << 3);
    }
    if (lane == 0) {
        mbar_init(&s_bar[warp][0], 1);
        mbar_init(&s_bar[warp][1], 1);
        fence_mbar_init();
    }
    __syncthreads();

    // Static interleaved schedule (warp w: bins w, w + W, ...): consecutive warps work on
    // consecutive bins (L2 locality of the deposits) and every future bin is known, so the
    // bin ranges are loaded one bin ahead and each 2-KB record chunk is fetched with one
    // cp.async.bulk into a double-buffered shared-memory slot one chunk ahead.
    const int nw = gridDim.x * WARPS;
    int bin = blockIdx.x * WARPS + warp;
    int b0 = 0, b1 = 0, nb0 = 0, nb1 = 0;
    if (bin < nbins) {
        b0 = __ldg(seg_begin + bin);
        b1 = __ldg(seg_begin + bin + 1);
    }
    if (bin + nw < nbins) {
        nb0 = __ldg(seg_begin + bin + nw);
        nb1 = __ldg(seg_begin + bin + nw + 1);
    }
    uint32_t chunk = 0;  // buffer (chunk & 1), mbarrier parity (chunk >> 1) & 1
    MM_TDECL
    if (lane == 0 && bin < nbins && b1 > b0)
        tma_load(&s_rec[warp][0][0], rec + 8 * (int64_t)b0, min(32, b1 - b0) * 64, &s_bar[warp][0]);
    while (bin < nbins) {
        // bin ranges two bins ahead (consumed when this bin's successor prefetches)
        int nn0 = 0, nn1 = 0;
        if (bin + 2 * nw < nbins) {
            nn0 = __ldg(seg_begin + bin + 2 * nw);
            nn1 = __ldg(seg_begin + bin + 2 * nw + 1);
        }
        double acc[NC][2];
#pragma unroll
        for (int c = 0; c < NC; ++c)
            acc[c][0] = acc[c][1] = 0.0;
        for (int base = b0; base < b1; base += 32, ++chunk) {
            const int m = min(32, b1 - base);
            const uint32_t buf = chunk & 1u;
            // prefetch the next chunk of this bin, else the first chunk of the next bin
            if (lane == 0) {
                if (base + 32 < b1)
                    tma_load(&s_rec[warp][buf ^ 1][0], rec + 8 * (int64_t)(base + 32), min(32, b1 - base - 32) * 64,
                             &s_bar[warp][buf ^ 1]);
                else if (bin + nw < nbins && nb1 > nb0)
                    tma_load(&s_rec[warp][buf ^ 1][0], rec + 8 * (int64_t)nb0, min(32, nb1 - nb0) * 64,
                             &s_bar[warp][buf ^ 1]);
            }
            MM_TMARK(3);
            mbar_wait(&s_bar[warp][buf], (chunk >> 1) & 1u);
            MM_TMARK(0);
            if (lane < m) {
                const double *r = &s_rec[warp][buf][8 * lane];
                const double2 ra = *reinterpret_cast<const double2 *>(r);      // xi_x, xi_y
                const double2 rb = *reinterpret_cast<const double2 *>(r + 2);  // xi_z, q
                double s[NC];
                if (NC == 9) {
                    const double2 rc = *reinterpret_cast<const double2 *>(r + 4);  // Bx, By
                    coeff<NC>(rb.y, rc.x, rc.y, r[6], wscale, sigma, s);
                } else {
                    coeff<NC>(rb.y, 0, 0, 0, wscale, sigma, s);
                }
                double wx[2], wy[2], wz[2];
                weights1(ra.x, wx);
                weights1(ra.y, wy);
                weights1(rb.x, wz);
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    sh_s[lane * L::SS + c] = s[c];
#pragma unroll
                for (int a = 0; a < 8; ++a)
                    sh_w[a * L::WS + lane] = (wx[a >> 2] * wy[(a >> 1) & 1]) * wz[a & 1];
            }
            __syncwarp();
            MM_TMARK(1);
            const double *wrow = sh_w + (lane >> 2) * L::WS + (lane & 3);
            const double *srow = sh_s + (lane & 3) * L::SS;
            auto batch = [&](int kb) {
                const double w = wrow[kb];
                const double *sp = srow + kb * L::SS;
                if (NC == 9) {
#pragma unroll
                    for (int c = 0; c < 8; c += 2) {
                        const double2 sv = *reinterpret_cast<const double2 *>(sp + c);
                        dmma(acc[c][0], acc[c][1], sv.x * w, w);
                        dmma(acc[c + 1][0], acc[c + 1][1], sv.y * w, w);
                    }
                    dmma(acc[NC - 1][0], acc[NC - 1][1], sp[8] * w, w);
                } else {
                    dmma(acc[0][0], acc[0][1], sp[0] * w, w);
                }
            };
            if (m == 32) {
#pragma unroll
                for (int kb = 0; kb < 32; kb += 4)
                    batch(kb);
            } else {
                for (int kb = 0; kb < m; kb += 4)
                    batch(kb);
            }
            __syncwarp();
            MM_TMARK(2);
        }
        MM_TMARK(2);
        if (b1 > b0) {
            // ---- deposit: stage D[a][b][c], then RED in address order via the table
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                sm[(lane >> 2) * 8 * NC + (2 * (lane & 3)) * NC + c] = acc[c][0];
                sm[(lane >> 2) * 8 * NC + (2 * (lane & 3) + 1) * NC + c] = acc[c][1];
            }
            // row pointers of the 8 support nodes: lane a (mod 8) computes node a's
            const int bx = bin / plane, rem = bin - bx * plane;
            const int by = rem / g.n2, bz = rem - by * g.n2;
            const int a8 = lane & 7;
            double *myrow = row_ptr(g, g.x_begin + bx + (a8 >> 2), wrapi(by + ((a8 >> 1) & 1), g.n1),
                                    wrapi(bz + (a8 & 1), g.n2), out, ghost, RL);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < L::NDEP; ++i) {
                const double v = sm[i * 32 + lane];
                const int t = s_tab[i * 32 + lane];
                double *row = shfl_ptr(myrow, t & 7);
#ifdef MM_EXPERIMENT_NO_FLUSH
                if (v == 12345.678)  // diagnostics build: deposit skipped
#else
                if (nonzero_bits(v))
#endif
                    red_add(row + (t >> 3), v);
            }
            __syncwarp();
        } else if (lane == 0 && bin + nw < nbins && nb1 > nb0) {
            // empty bin: nothing was prefetched for the successor yet
            tma_load(&s_rec[warp][chunk & 1u][0], rec + 8 * (int64_t)nb0, min(32, nb1 - nb0) * 64,
                     &s_bar[warp][chunk & 1u]);
        }
        MM_TMARK(3);
        bin += nw;
        b0 = nb0;
        b1 = nb1;
        nb0 = nn0;
        nb1 = nn1;
    }
    MM_TFLUSH();
}

// ------------------------------------------------ order 1, tensor: pair-product GEMM
// The tensor-product B-spline (eq_shape_bspline) makes W_a W_b a product over the axes
// of per-axis PAIR products q_mu(a_mu + b_mu):  q(0) = w0 w0, q(1) = w0 w1, q(2) = w1 w1
// (CIC: w0 = 1 - xi, w1 = xi).  So the 8x8x9 block of a bin is
//
//   M^c[a][b] = sum_p s^c_p W_a W_b = sum_p X_p[ux uy] Z_p[uz c]   (u_mu = a_mu + b_mu)
//   X_p[3 ux + uy] = q_x(ux) q_y(uy)   (9 values),   Z_p[9 uz + c] = q_z(uz) s^c_p   (27)
//
// one dense product over particles with 9 x 27 = 243 outputs (instead of 64 x 9), and
// no per-batch A-element scaling: the operands are the prep's products.  DMMA tiles:
// m = (ux,uy) (9 -> 2 row tiles), n = (uz,c) (27 -> 4 column tiles), 8 DMMA per batch
// of 4 particles.  Deposit: M^c[a][b] = stage[X row u(a,b)][Z col u(a,b), c] through a
// table, REDs in the same address order as the node-tile kernel.
struct O1T {
    static constexpr int WARPS = 4;
    static constexpr int XS = 36;                 // row stride (doubles): 2 wavefronts per batch LDS
    static constexpr int ROWS = 36;               // 9 X rows + 27 Z rows
    static constexpr int WARP_DOUBLES = ROWS * XS;  // 1296 (stage of 243 aliases it)
    static constexpr size_t SMEM = (size_t)WARPS * WARP_DOUBLES * 8 + 576 * 4 + WARPS * 8 * 8;  // + node rows
};

__global__ void __launch_bounds__(O1T::WARPS * 32) k_asm_o1t(Geo g, const double *__restrict__ rec,
                                                             const int32_t *__restrict__ seg_begin, int64_t nbins,
                                                             double wscale, double sigma, double *__restrict__ out,
                                                             double *__restrict__ ghost)
{
    using L = O1T;
    extern __shared__ __align__(16) double dsm_o1t[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *xz = dsm_o1t + warp * L::WARP_DOUBLES;
    double *stage = xz;  // [9][27] after the last batch of a bin
    int32_t *s_dep = reinterpret_cast<int32_t *>(dsm_o1t + L::WARPS * L::WARP_DOUBLES);
    double **s_row = reinterpret_cast<double **>(s_dep + 576) + warp * 8;  // this warp's bin: node rows
    const int plane = g.n1 * g.n2;

    // deposit table, element e = (a, b, c) in address order of node a's row:
    // a (3 bits) | slot*9 + c (8 bits) | stage index (X row * 27 + Z col, 8 bits)
    for (int e = threadIdx.x; e < 576; e += blockDim.x) {
        const int a = e / 72, r = e - a * 72, b = r / 9, c = r - b * 9;
        const int ax = a >> 2, ay = (a >> 1) & 1, az = a & 1, bx = b >> 2, by = (b >> 1) & 1, bz = b & 1;
        const int slot = (bx - ax + 1) * 9 + (by - ay + 1) * 3 + (bz - az + 1);
        const int m = 3 * (ax + bx) + (ay + by), n = 9 * (az + bz) + c;
        s_dep[e] = a | ((slot * 9 + c) << 3) | ((m * 27 + n) << 11);
    }
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
    // the lane's record of the current chunk, loaded one chunk ahead
    double4 ra = make_double4(0, 0, 0, 0), rb = ra;
    if (bin < nbins && b0 + lane < b1) {
        ra = ld256(rec + 8 * (int64_t)(b0 + lane));
        rb = ld256(rec + 8 * (int64_t)(b0 + lane) + 4);
    }
    // batch-loop operand addresses: A row (lane>>2) (+8 for lanes 0-3), B rows 9 + 8nt + (lane>>2)
    const int kq = lane & 3, rq = lane >> 2;
    const double *xa = xz + rq * L::XS + kq;
    const double *xa1 = xz + 8 * L::XS + kq;                 // row 8 (lanes 0-3 only)
    const double *zb = xz + (9 + rq) * L::XS + kq;
    const bool z3 = rq < 3;                                  // rows 9 + 24 + rq < 36
    while (bin < nbins) {
        int nn0 = 0, nn1 = 0;
        if (bin + 2 * nw < nbins) {
            nn0 = __ldg(seg_begin + bin + 2 * nw);
            nn1 = __ldg(seg_begin + bin + 2 * nw + 1);
        }
        double acc[8][2];
#pragma unroll
        for (int t = 0; t < 8; ++t)
            acc[t][0] = acc[t][1] = 0.0;
        for (int base = b0; base < b1; base += 32) {
            const int m = min(32, b1 - base);
            const double4 ca = ra, cb = rb;
            // prefetch the lane's record of the next chunk (this bin, else the next bin)
            {
                int64_t p = -1;
                if (base + 32 < b1) {
                    if (base + 32 + lane < b1)
                        p = base + 32 + lane;
                } else if (bin + nw < nbins && nb0 + lane < nb1) {
                    p = nb0 + lane;
                }
                if (p >= 0) {
                    ra = ld256(rec + 8 * p);
                    rb = ld256(rec + 8 * p + 4);
                }
            }
            __syncwarp();  // previous batches / deposit are done with xz
            if (lane < m) {
                double s[9];
                coeff<9>(ca.w, cb.x, cb.y, cb.z, wscale, sigma, s);
                double qx[3], qy[3], qz[3];
                {
                    const double w0 = 1.0 - ca.x, w1 = ca.x;
                    qx[0] = w0 * w0, qx[1] = w0 * w1, qx[2] = w1 * w1;
                }
                {
                    const double w0 = 1.0 - ca.y, w1 = ca.y;
                    qy[0] = w0 * w0, qy[1] = w0 * w1, qy[2] = w1 * w1;
                }
                {
                    const double w0 = 1.0 - ca.z, w1 = ca.z;
                    qz[0] = w0 * w0, qz[1] = w0 * w1, qz[2] = w1 * w1;
                }
                double *col = xz + lane;
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j)
                        col[(3 * i + j) * L::XS] = qx[i] * qy[j];
#pragma unroll
                for (int k = 0; k < 3; ++k)
#pragma unroll
                    for (int c = 0; c < 9; ++c)
                        col[(9 + 9 * k + c) * L::XS] = qz[k] * s[c];
            }
            __syncwarp();
            auto batch = [&](int kb) {
                const double a0 = xa[kb];
                const double a1 = lane < 4 ? xa1[kb] : 0.0;
                double bv[4];
#pragma unroll
                for (int nt = 0; nt < 3; ++nt)
                    bv[nt] = zb[8 * nt * L::XS + kb];
                bv[3] = z3 ? zb[24 * L::XS + kb] : 0.0;
#pragma unroll
                for (int nt = 0; nt < 4; ++nt) {
                    dmma(acc[nt][0], acc[nt][1], a0, bv[nt]);
                    dmma(acc[4 + nt][0], acc[4 + nt][1], a1, bv[nt]);
                }
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
            // stage[X row][Z col]: D tile (mt, nt) element (rq, 2kq + v)
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                    for (int v = 0; v < 2; ++v) {
                        const int mr = 8 * mt + rq, nc = 8 * nt + 2 * kq + v;
                        if (mr < 9 && nc < 27)
                            stage[mr * 27 + nc] = acc[4 * mt + nt][v];
                    }
            const int bx = bin / plane, rem = bin - bx * plane;
            const int by = rem / g.n2, bz = rem - by * g.n2;
            if (lane < 8)
                s_row[lane] = row_ptr(g, g.x_begin + bx + (lane >> 2), wrapi(by + ((lane >> 1) & 1), g.n1),
                                      wrapi(bz + (lane & 1), g.n2), out, ghost, 27 * 9);
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 18; ++i) {
                const int t = s_dep[i * 32 + lane];
                const double v = stage[t >> 11];
                double *row = s_row[t & 7];
                red_add(row + ((t >> 3) & 255), v);  // unconditional (+0 contributions are harmless)
            }
        } else if (bin + nw < nbins && nb0 + lane < nb1) {
            // empty bin: nothing was prefetched for the successor yet
            ra = ld256(rec + 8 * (int64_t)(nb0 + lane));
            rb = ld256(rec + 8 * (int64_t)(nb0 + lane) + 4);
        }
        bin += nw;
        b0 = nb0;
        b1 = nb1;
        nb0 = nn0;
        nb1 = nn1;
    }
}

// ---------------------------------------------------------------- order 2
// 27-node support padded to 32 = 4 row blocks of 8; the 10 upper 8x8 tiles
// (r <= c) per component (spatial symmetry, eq_spatial_symmetry); the lower
// tiles follow by mirroring.  One GROUP of NC warps assembles one bin, warp c
// owning component c (tensor: the CTA = 9 warps; scalar: a single warp, GPC
// groups per CTA).  Each warp preps its own share of the chunk (its lane's
// particle: s^c and the per-axis weights, then W rows a = c, c+NC, ...) into a
// double-buffered weight tile, so one group barrier per chunk suffices.  The
// tiles are mirrored into a full 27 x 27 x NC stage in shared memory and
// flushed with REDs in global address order: runs of 3 z-adjacent slots x NC
// components are contiguous in the [g][slot][comp] layout (27*8 B, tensor).
template <int NC>
struct O2 {
    static constexpr int WPG = NC;                   // warps per group
    static constexpr int GPC = NC == 9 ? 1 : 4;      // groups per CTA
    static constexpr int THREADS = WPG * GPC * 32;
    static constexpr int CH = 64;                    // particles per chunk (2 per lane in the prep)
    static constexpr int WS = CH + 4;                // weight tile row stride (doubles; 2 wavefronts/LDS)
    static constexpr int WBUF = 32 * WS;             // one weight tile [32 nodes][WS]
    static constexpr int RBUF = CH * 8;              // one TMA-staged record chunk (doubles)
    static constexpr int STAGE = 378 * NC;          // upper triangle (a <= b) of the 27x27 block
    static constexpr int GROUP_DOUBLES = 2 * RBUF + 2 * WBUF + STAGE + 32 + 2;  // recs, W, stage, rowp, mbar
    static constexpr size_t SMEM = (size_t)GPC * GROUP_DOUBLES * 8 + (730 * 2 + 640) * 2 + 8 * GPC + 32 * GPC;
};

__device__ __forceinline__ void group_sync(int nthreads, int id)
{
    if (nthreads == 32)
        __syncwarp();
    else
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// s^{c} of one component (c = 3i + j) — eq_alpha_matrix, same expression as coeff<9>.
__device__ __forceinline__ double coeff_one(int c, double q, double Bx, double By, double Bz, double wscale,
                                            double sigma)
{
    // same expressions as coeff<9> (Newton-refined reciprocal, one FMA per component)
    const double o0 = wscale * Bx, o1 = wscale * By, o2 = wscale * Bz;
    const double d = fma(o0, o0, fma(o1, o1, fma(o2, o2, 1.0)));
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    r = fma(r, fma(-d, r, 1.0), r);
    r = fma(r, fma(-d, r, 1.0), r);
    const double f = (sigma * q) * r;
    const double f0 = f * o0, f1 = f * o1, f2 = f * o2;
    const int i = c / 3, j = c - 3 * i;
    const double fi = i == 0 ? f0 : (i == 1 ? f1 : f2);
    const double oj = j == 0 ? o0 : (j == 1 ? o1 : o2);
    // f delta_ij + eps_ijk f omega_k
    const double add = c == 0 || c == 4 || c == 8 ? f
                       : c == 1 ? f2 : c == 2 ? -f1 : c == 3 ? -f2 : c == 5 ? f0 : c == 6 ? f1 : -f0;
    return fma(fi, oj, add);
}

template <int NC>
__global__ void __launch_bounds__(O2<NC>::THREADS, NC == 9 ? 3 : 2) k_asm_o2(Geo g, const double *__restrict__ rec,
                                                            const int32_t *__restrict__ seg_begin, int64_t nbins,
                                                            double wscale, double sigma, double *__restrict__ out,
                                                            double *__restrict__ ghost, int *__restrict__ work)
{
    using L = O2<NC>;
    extern __shared__ __align__(16) double dsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = warp / L::WPG, comp = warp - grp * L::WPG;
    const int gtid = threadIdx.x - grp * L::WPG * 32;  // thread index inside the group
    constexpr int GT = L::WPG * 32;                     // threads per group
    double *gsm = dsm + grp * L::GROUP_DOUBLES;
    double *srec = gsm;                        // [2][CH records][8]  (TMA-staged chunks)
    double *wbuf = gsm + 2 * L::RBUF;          // [2][32 nodes][WS]
    double *stage = wbuf + 2 * L::WBUF;        // [378 upper pairs][NC]
    double **rowp = reinterpret_cast<double **>(stage + L::STAGE);  // [27]
    uint64_t *bars = reinterpret_cast<uint64_t *>(stage + L::STAGE + 32);  // [2]
    int16_t *s_slot = reinterpret_cast<int16_t *>(dsm + L::GPC * L::GROUP_DOUBLES);  // [27][27] slot(b-a)
    int16_t *s_tri = s_slot + 730;                                                    // [27][27] upper index
    int16_t *s_stoff = s_tri + 730;  // [10 tiles][2][32 lanes] stage offset of the lane's entry, -1 = none
    int64_t *s_bin = reinterpret_cast<int64_t *>(s_stoff + 640) + grp;  // next-bin broadcast (8-B aligned)
    const int plane = g.n1 * g.n2;
    constexpr int RL = 125 * NC;

    for (int e = threadIdx.x; e < 729; e += blockDim.x) {
        const int a = e / 27, b = e - 27 * a;
        s_slot[e] = (int16_t)((b / 9 - a / 9 + 2) * 25 + ((b / 3) % 3 - (a / 3) % 3 + 2) * 5 + (b % 3 - a % 3 + 2));
        const int i = a < b ? a : b, j = a < b ? b : a;
        s_tri[e] = (int16_t)(i * 27 - i * (i - 1) / 2 + (j - i));
    }
    for (int e = threadIdx.x; e < 640; e += blockDim.x) {
        const int t = e / 64, v = (e / 32) & 1, l = e & 31;
        const int tr = t < 4 ? 0 : (t < 7 ? 1 : (t < 9 ? 2 : 3));
        const int tc = t < 4 ? t : (t < 7 ? t - 3 : (t < 9 ? t - 5 : 3));
        const int a = 8 * tr + (l >> 2), b = 8 * tc + 2 * (l & 3) + v;
        s_stoff[e] = (a < 27 && b < 27 && a <= b) ? (int16_t)(a * 27 - a * (a - 1) / 2 + (b - a)) : (int16_t)-1;
    }
    // dynamic, in-order bin scheduling.  Thread 0 of the group keeps a two-deep ticket
    // queue (tnext = the bin after the current one, tnext2 = the one after that) so that
    // the atomic, the bin-range loads and the first-chunk TMA of a bin are all issued at
    // least one bin before they are needed.
    // (thread 0 only; kept in shared memory to spare registers of the other 287 threads)
    int *q = reinterpret_cast<int *>(s_bin + L::GPC) + 8 * grp;  // tnext, tnext2, -, -, issued
    int tn0 = 0, tn1 = 0;                                         // (gtid 0) range of bin tnext
    if (gtid == 0) {
        *s_bin = atom_add(work, 1);
        q[0] = atom_add(work, 1);
        q[1] = atom_add(work, 1);
        q[4] = -1;
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    int64_t bin = *s_bin;
    int chunk = 0;  // global chunk counter -> buffer (chunk & 1), mbarrier parity (chunk >> 1) & 1
    while (bin < nbins) {
        const int b0 = seg_begin[bin], b1 = seg_begin[bin + 1];
        if (gtid == 0) {
            if (b1 > b0 && q[4] != bin)
                tma_load(srec + (chunk & 1) * L::RBUF, rec + 8 * (int64_t)b0, min(L::CH, b1 - b0) * 64,
                         &bars[chunk & 1]);
            const int tnext = q[0];
            tn0 = tn1 = 0;
            if (tnext < nbins) {  // loads in flight until the last chunk of this bin
                tn0 = seg_begin[tnext];
                tn1 = seg_begin[tnext + 1];
            }
        }
        double acc[10][2];
#pragma unroll
        for (int t = 0; t < 10; ++t)
            acc[t][0] = acc[t][1] = 0.0;
        for (int base = b0; base < b1; base += L::CH, ++chunk) {
            const int m = min(L::CH, b1 - base);
            double *wt = wbuf + (chunk & 1) * L::WBUF;
            // prep (every warp, lane = particle): s^comp and this warp's W rows, from the
            // TMA-staged record chunk
            mbar_wait(&bars[chunk & 1], (chunk >> 1) & 1);
            double s_me[L::CH / 32];  // s of particles lane, lane + 32, ...
#pragma unroll
            for (int j = 0; j < L::CH / 32; ++j) {
                const int p = lane + 32 * j;
                s_me[j] = 0.0;
                if (p < m) {
                    const double *r = srec + (chunk & 1) * L::RBUF + 8 * p;
                    const double2 ra = *reinterpret_cast<const double2 *>(r);
                    const double2 rb = *reinterpret_cast<const double2 *>(r + 2);
                    if (NC == 9) {
                        const double2 rc = *reinterpret_cast<const double2 *>(r + 4);
                        s_me[j] = coeff_one(comp, rb.y, rc.x, rc.y, r[6], wscale, sigma);
                    } else {
                        s_me[j] = sigma * rb.y;
                    }
                    double wx[3], wy[3], wz[3];
                    weights2(ra.x, wx);
                    weights2(ra.y, wy);
                    weights2(rb.x, wz);
                    // runtime node digits: select instead of indexing (keeps wx/wy/wz in registers)
                    auto sel = [](const double *w, int i) { return i == 0 ? w[0] : (i == 1 ? w[1] : w[2]); };
                    if (NC == 9) {
                        // warp c owns nodes a = c + 9k: digits (k, c/3, c%3)
                        const double wyc = sel(wy, comp / 3), wzc = sel(wz, comp % 3);
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int a = comp + 9 * k;
                            if (a < 32)
                                wt[a * L::WS + p] = a < 27 ? (wx[k < 3 ? k : 0] * wyc) * wzc : 0.0;
                        }
                    } else {
                        for (int a = 0; a < 32; ++a)
                            wt[a * L::WS + p] =
                                a < 27 ? (sel(wx, a / 9) * sel(wy, (a / 3) % 3)) * sel(wz, a % 3) : 0.0;
                    }
                }
            }
            group_sync(GT, 1 + grp);
            // every warp is past its reads of the other record buffer: prefetch the next chunk
            if (gtid == 0) {
                const double *src = nullptr;
                int cnt = 0;
                if (base + L::CH < b1) {
                    src = rec + 8 * (int64_t)(base + L::CH);
                    cnt = min(L::CH, b1 - base - L::CH);
                } else if (q[0] < nbins && tn1 > tn0) {
                    src = rec + 8 * (int64_t)tn0;
                    cnt = min(L::CH, tn1 - tn0);
                    q[4] = q[0];
                }
                if (cnt)
                    tma_load(srec + ((chunk + 1) & 1) * L::RBUF, src, cnt * 64, &bars[(chunk + 1) & 1]);
            }
            const double *wcol = wt + (lane >> 2) * L::WS + (lane & 3);
            auto batch = [&](int kb) {
                double w[4];
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    w[r] = wcol[8 * r * L::WS + kb];
                const double s = __shfl_sync(0xffffffffu, (kb & 32) ? s_me[L::CH / 32 - 1] : s_me[0],
                                             (kb & 31) + (lane & 3));
                double A[4];
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    A[r] = s * w[r];
                dmma(acc[0][0], acc[0][1], A[0], w[0]);
                dmma(acc[1][0], acc[1][1], A[0], w[1]);
                dmma(acc[2][0], acc[2][1], A[0], w[2]);
                dmma(acc[3][0], acc[3][1], A[0], w[3]);
                dmma(acc[4][0], acc[4][1], A[1], w[1]);
                dmma(acc[5][0], acc[5][1], A[1], w[2]);
                dmma(acc[6][0], acc[6][1], A[1], w[3]);
                dmma(acc[7][0], acc[7][1], A[2], w[2]);
                dmma(acc[8][0], acc[8][1], A[2], w[3]);
                dmma(acc[9][0], acc[9][1], A[3], w[3]);
            };
            if (m == L::CH) {
#pragma unroll 2
                for (int kb = 0; kb < L::CH; kb += 4)
                    batch(kb);
            } else {
                for (int kb = 0; kb < m; kb += 4)
                    batch(kb);
            }
        }
        if (b0 == b1) {  // empty bin (rare): just advance the ticket
            if (gtid == 0) {
                *s_bin = q[0];
                q[0] = q[1];
                if (q[1] < nbins)
                    q[1] = atom_add(work, 1);
            }
            group_sync(GT, 1 + grp);
            bin = *s_bin;
            group_sync(GT, 1 + grp);
            continue;
        }
        // ---- stage the full 27x27 block of component `comp` (mirror of the upper tiles)
        const int bx = (int)(bin / plane), rem = (int)(bin - (int64_t)bx * plane);
        const int by = rem / g.n2, bz = rem - by * g.n2;
        if (gtid < 27) {
            const int a = gtid;
            rowp[a] = row_ptr(g, g.x_begin + bx - 1 + a / 9, wrapi(by + (a / 3) % 3, g.n1),
                              wrapi(bz + a % 3, g.n2), out, ghost, RL);
        }
        if (gtid == 0) {
            *s_bin = q[0];
            q[0] = q[1];
            if (q[1] < nbins)
                q[1] = atom_add(work, 1);
        }
        // M_ab = M_ba (eq_spatial_symmetry): keep the a <= b entries (table s_stoff)
#pragma unroll
        for (int t = 0; t < 10; ++t) {
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int o = s_stoff[(2 * t + v) * 32 + lane];
                if (o >= 0)
                    stage[o * NC + comp] = acc[t][v];
            }
        }
        group_sync(GT, 1 + grp);
        bin = *s_bin;
        // ---- flush in address order.  Tensor: 243 runs (node a, b_x, b_y) of 27 contiguous
        //      doubles (b_z = 0..2 x 9 comps) -> row(a) + slot(b0 - a)*9 + lane.  The next
        //      write of stage/rowp/s_bin comes after the next chunk barrier.
        if (NC == 9) {
            // warp c flushes runs (a, b_x, b_y) = (a, c/3, c%3) for a = 0..26
            const int b0c = 9 * (comp / 3) + 3 * (comp % 3);
            const int bzl = lane / 9, cl = lane - 9 * bzl;
            if (lane < 27) {
#pragma unroll 3
                for (int a = 0; a < 27; ++a) {
                    const int ab0 = a * 27 + b0c;
                    const double v = stage[s_tri[ab0 + bzl] * 9 + cl];
#ifdef MM_EXPERIMENT_NO_FLUSH
                    if (v == 12345.678)  // diagnostics build: deposit skipped
#else
                    if (nonzero_bits(v))
#endif
                        red_add(rowp[a] + s_slot[ab0] * 9 + lane, v);
                }
            }
        } else {
            for (int e = gtid; e < 729; e += GT) {
                const double v = stage[s_tri[e]];
                if (nonzero_bits(v))
                    red_add(rowp[e / 27] + s_slot[e], v);
            }
        }
    }
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
                                                                int *__restrict__ work)
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
    if (threadIdx.x == 0) {
        q[0] = atom_add(work, 1);
        q[1] = atom_add(work, 1);
        q[2] = atom_add(work, 1);
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
                    coeff<9>(zq.y, bxy.x, bxy.y, r[6], wscale, sigma, s);
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
            __syncthreads();
            if (threadIdx.x == 0) {
                q[0] = q[1];
                q[1] = q[2];
                if (q[2] < nbins)
                    q[2] = atom_add(work, 1);
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
        const int bx = (int)(bin / plane), rem = bin - bx * plane;
        const int by = rem / g.n2, bz = rem - by * g.n2;
        if (threadIdx.x < 27) {
            const int a = threadIdx.x;
            rowp[a] = row_ptr(g, g.x_begin + bx - 1 + a / 9, wrapi(by + (a / 3) % 3, g.n1), wrapi(bz + a % 3, g.n2),
                              out, ghost, RL);
        }
        if (threadIdx.x == 0) {
            q[0] = q[1];
            q[1] = q[2];
            if (q[2] < nbins)
                q[2] = atom_add(work, 1);
        }
        __syncthreads();
        bin = q[0];
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
            const int bx = bin / plane, rem = bin - bx * plane;
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
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(k_asm_pps<ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
        if (e)
            return e;
        attr = true;
    }
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

template <typename K>
unsigned grid_for(K kernel, int64_t items)
{
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, WARPS * 32, 0);
    if (per_sm < 1)
        per_sm = 1;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t want = (items + WARPS - 1) / WARPS;
    int64_t cap = (int64_t)sms * per_sm;
    return (unsigned)(want < cap ? (want < 1 ? 1 : want) : cap);
}

template <int NC>
cudaError_t launch_o1(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    using L = O1<NC>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_asm_o1<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
        if (e)
            return e;
        attr = true;
    }
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_asm_o1<NC>, WARPS * 32, L::SMEM);
    if (cta_cap() > 0 && per_sm > cta_cap())
        per_sm = cta_cap();
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t want = (a.nbins + WARPS - 1) / WARPS;
    int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    unsigned grid = (unsigned)(want < cap ? (want < 1 ? 1 : want) : cap);
    k_asm_o1<NC><<<grid, WARPS * 32, L::SMEM, s>>>(geo, a.rec, a.seg_begin, a.nbins, a.wscale, a.sigma, a.out,
                                                   a.ghost, a.work);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_o2t(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    using L = O2T;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_asm_o2t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
        if (e)
            return e;
        attr = true;
    }
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_asm_o2t, L::WARPS * 32, L::SMEM);
    if (cta_cap() > 0 && per_sm > cta_cap())
        per_sm = cta_cap();
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    unsigned grid = (unsigned)(a.nbins < cap ? (a.nbins < 1 ? 1 : a.nbins) : cap);
    k_asm_o2t<<<grid, L::WARPS * 32, L::SMEM, s>>>(geo, a.rec, a.seg_begin, a.nbins, a.wscale, a.sigma, a.out,
                                                   a.ghost, a.work);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_o1t(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    using L = O1T;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_asm_o1t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
        if (e)
            return e;
        attr = true;
    }
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_asm_o1t, L::WARPS * 32, L::SMEM);
    if (cta_cap() > 0 && per_sm > cta_cap())
        per_sm = cta_cap();
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t want = (a.nbins + L::WARPS - 1) / L::WARPS;
    int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    unsigned grid = (unsigned)(want < cap ? (want < 1 ? 1 : want) : cap);
    k_asm_o1t<<<grid, L::WARPS * 32, L::SMEM, s>>>(geo, a.rec, a.seg_begin, a.nbins, a.wscale, a.sigma, a.out,
                                                   a.ghost);
    count_launch();
    return cudaGetLastError();
}

// MM_ASM_LEGACY=1 selects the node-tile kernels (A = W s, B = W^T per component) for the
// tensor kind, for A/B measurements against the pair-product kernels.
inline bool legacy_tiles()
{
    static const bool v = [] {
        const char *e = getenv("MM_ASM_LEGACY");
        return e && e[0] == '1';
    }();
    return v;
}

template <int NC>
cudaError_t launch_o2(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    using L = O2<NC>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_asm_o2<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
        if (e)
            return e;
        attr = true;
    }
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_asm_o2<NC>, L::THREADS, L::SMEM);
    if (cta_cap() > 0 && per_sm > cta_cap())
        per_sm = cta_cap();
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t want = (a.nbins + L::GPC - 1) / L::GPC;
    int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    unsigned grid = (unsigned)(want < cap ? (want < 1 ? 1 : want) : cap);
    k_asm_o2<NC><<<grid, L::THREADS, L::SMEM, s>>>(geo, a.rec, a.seg_begin, a.nbins, a.wscale, a.sigma, a.out,
                                                   a.ghost, a.work);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t assemble_fp64_enqueue(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    if (a.nbins == 0)
        return cudaSuccess;
    if (geo.order == 1) {
        if (a.ncomp == 9)
            return legacy_tiles() ? launch_o1<9>(geo, a, s) : launch_o1t(geo, a, s);
        return launch_pps<1>(geo, a, s);  // (the node-tile kernels assume 64-B records)
    } else {
        if (a.ncomp == 9)
            return legacy_tiles() ? launch_o2<9>(geo, a, s) : launch_o2t(geo, a, s);
        return launch_pps<2>(geo, a, s);
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace mm

#ifdef MM_EXPERIMENT_TIMERS
// diagnostics build only: per-phase SM cycles summed over warps since the last call
extern "C" int mm_debug_phases(unsigned long long *out4)
{
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out4, mm::g_phase, sizeof(unsigned long long) * 4);
    unsigned long long z[4] = {0, 0, 0, 0};
    return (int)cudaMemcpyToSymbol(mm::g_phase, z, sizeof(z));
}
#endif
