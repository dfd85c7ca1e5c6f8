// FP64 tensor-core (DMMA 8x8x4) mass-matrix assembly for first- and
// second-order B-splines.  Algorithm 1 of the paper:
//
//   for each support group (here: a support-window bin, R12)
//     D^{ij} <- 0                                             (alg. line 399)
//     for each batch of K_t = 4 particles                     (eq_D_batches)
//       A^{ij}_{ak} = W_{a p_k} s^{ij}_{p_k},  B_{kb} = W_{b p_k}  (eq_AB_batch)
//       D^{ij} += A^{ij} B                    one DMMA per tile and component
//     deposit D^{ij} into the node-stencil storage
//
// Fragment mapping of mma.sync.m8n8k4.f64 (row.col): lane t holds
// A[t>>2][t&3], B[t&3][t>>2] and D[t>>2][2(t&3)+v].  With rows = support
// nodes and k = particles, lane t needs exactly ONE weight, w = W_{t>>2}(p_{t&3}):
// it is its B element unscaled and, times s^{ij}, its A element.
//
// Per-particle work (alpha, s, W) is done once per particle by one lane on a
// chunk of particles read with coalesced 16-B loads and staged in shared
// memory; the batch loop then reads w and s from shared memory.
#include "mm_internal.cuh"

namespace mm {

namespace {

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ int wrapi(int i, int n)
{
    return i < 0 ? i + n : (i >= n ? i - n : i);
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
        double o0 = wscale * Bx, o1 = wscale * By, o2 = wscale * Bz;
        double d = 1.0 + (o0 * o0 + o1 * o1 + o2 * o2);
        double f = __ddiv_rn(sigma * q, d);
        s[0] = f * (1.0 + o0 * o0);
        s[1] = f * (o0 * o1 + o2);
        s[2] = f * (o0 * o2 - o1);
        s[3] = f * (o1 * o0 - o2);
        s[4] = f * (1.0 + o1 * o1);
        s[5] = f * (o1 * o2 + o0);
        s[6] = f * (o2 * o0 + o1);
        s[7] = f * (o2 * o1 - o0);
        s[8] = f * (1.0 + o2 * o2);
    }
}

// Per-axis B-spline weights at the support nodes:
// w_k = phi(xi - (b + k)).
__device__ __forceinline__ void weights1(double xi, double w[2])
{
    w[0] = 1.0 - xi;                     // phi1(xi)
    w[1] = 1.0 - fabs(xi - 1.0);         // phi1(xi - 1)
}

__device__ __forceinline__ void weights2(double xi, double w[3])
{
    double b = xi >= 0.5 ? 0.0 : -1.0;   // R4: tie -> base 0
    double t0 = fabs(xi - b), t1 = xi - (b + 1.0), t2 = fabs(xi - (b + 2.0));
    w[0] = 0.5 * (1.5 - t0) * (1.5 - t0);    // 1/2 < |t0| <= 3/2
    w[1] = 0.75 - t1 * t1;                   // |t1| <= 1/2
    w[2] = 0.5 * (1.5 - t2) * (1.5 - t2);    // 1/2 <= |t2| <= 3/2
}

constexpr int WARPS = 8;

// ---------------------------------------------------------------- order 1
template <int NC>
struct O1Smem {
    static constexpr int PREP = 32 * (NC + 8);
    static constexpr int STAGE = 64 * NC;
    static constexpr int SIZE = PREP > STAGE ? PREP : STAGE;
};

template <int NC>
__global__ void __launch_bounds__(WARPS * 32) k_asm_o1(Geo g, const double *__restrict__ rec,
                                                       const int32_t *__restrict__ seg_begin, int64_t nbins,
                                                       double wscale, double sigma, double *__restrict__ out,
                                                       double *__restrict__ ghost)
{
    __shared__ __align__(16) double smem[WARPS][O1Smem<NC>::SIZE];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *sm = smem[warp];
    double *sh_s = sm;             // [32][NC]
    double *sh_w = sm + 32 * NC;   // [32][8]
    const int64_t nwarps = (int64_t)gridDim.x * WARPS;
    const int plane = g.n1 * g.n2;
    constexpr int RL = 27 * NC;

    for (int64_t bin = (int64_t)blockIdx.x * WARPS + warp; bin < nbins; bin += nwarps) {
        const int b0 = seg_begin[bin], b1 = seg_begin[bin + 1];
        if (b0 == b1)
            continue;
        double acc[NC][2];
#pragma unroll
        for (int c = 0; c < NC; ++c)
            acc[c][0] = acc[c][1] = 0.0;

        for (int base = b0; base < b1; base += 32) {
            const int m = min(32, b1 - base);
            if (lane < m) {
                const double2 *r = reinterpret_cast<const double2 *>(rec + 8 * (int64_t)(base + lane));
                double2 r0 = __ldg(r), r1 = __ldg(r + 1);
                double s[NC];
                if (NC == 9) {
                    double2 r2 = __ldg(r + 2), r3 = __ldg(r + 3);
                    coeff<NC>(r1.y, r2.x, r2.y, r3.x, wscale, sigma, s);
                } else {
                    coeff<NC>(r1.y, 0, 0, 0, wscale, sigma, s);
                }
                double wx[2], wy[2], wz[2];
                weights1(r0.x, wx);
                weights1(r0.y, wy);
                weights1(r1.x, wz);
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    sh_s[lane * NC + c] = s[c];
#pragma unroll
                for (int a = 0; a < 8; ++a)
                    sh_w[lane * 8 + a] = wx[a >> 2] * wy[(a >> 1) & 1] * wz[a & 1];
            }
            __syncwarp();
            for (int kb = 0; kb < m; kb += 4) {
                const int p = kb + (lane & 3);
                const double w = sh_w[p * 8 + (lane >> 2)];
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    dmma(acc[c][0], acc[c][1], sh_s[p * NC + c] * w, w);
            }
            __syncwarp();
        }

        // ---- deposit: stage D[a][b][c] in shared memory, then RED in address order
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            sm[(lane >> 2) * 8 * NC + (2 * (lane & 3)) * NC + c] = acc[c][0];
            sm[(lane >> 2) * 8 * NC + (2 * (lane & 3) + 1) * NC + c] = acc[c][1];
        }
        __syncwarp();
        const int bx = (int)(bin / plane), rem = (int)(bin - (int64_t)bx * plane);
        const int by = rem / g.n2, bz = rem - by * g.n2;
        const int X0 = g.x_begin + bx;  // order 1: window base = cell
        for (int e = lane; e < 64 * NC; e += 32) {
            const int a = e / (8 * NC), rr = e - a * 8 * NC, b = rr / NC, c = rr - b * NC;
            const double v = sm[e];
            if (v != 0.0) {
                const int ax = a >> 2, ay = (a >> 1) & 1, az = a & 1;
                const int slot = ((b >> 2) - ax + 1) * 9 + (((b >> 1) & 1) - ay + 1) * 3 + ((b & 1) - az + 1);
                double *row = row_ptr(g, X0 + ax, wrapi(by + ay, g.n1), wrapi(bz + az, g.n2), out, ghost, RL);
                atomicAdd(row + slot * NC + c, v);
            }
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- order 2
// 27-node support padded to 32 = 4 row blocks of 8; the 10 upper 8x8 tiles
// (r <= c) per component (spatial symmetry, eq_spatial_symmetry); the lower
// tiles are deposited as mirrors.  A warp owns CG of the NC components of one bin.
__constant__ int8_t kTileR[10] = {0, 0, 0, 0, 1, 1, 1, 2, 2, 3};
__constant__ int8_t kTileC[10] = {0, 1, 2, 3, 1, 2, 3, 2, 3, 3};

template <int NC, int CG>
__global__ void __launch_bounds__(WARPS * 32) k_asm_o2(Geo g, const double *__restrict__ rec,
                                                       const int32_t *__restrict__ seg_begin, int64_t nbins,
                                                       double wscale, double sigma, double *__restrict__ out,
                                                       double *__restrict__ ghost)
{
    constexpr int NG = NC / CG;
    constexpr int CH = 16;  // particles staged per chunk
    constexpr int SM = CH * (32 + CG) > 640 ? CH * (32 + CG) : 640;
    __shared__ __align__(16) double smem[WARPS][SM];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *sh_w = smem[warp];            // [CH][32]
    double *sh_s = smem[warp] + CH * 32;  // [CH][CG]
    const int64_t nwarps = (int64_t)gridDim.x * WARPS;
    const int plane = g.n1 * g.n2;
    constexpr int RL = 125 * NC;
    const int64_t nitems = nbins * NG;

    for (int64_t item = (int64_t)blockIdx.x * WARPS + warp; item < nitems; item += nwarps) {
        const int64_t bin = item / NG;
        const int grp = (int)(item - bin * NG);
        const int b0 = seg_begin[bin], b1 = seg_begin[bin + 1];
        if (b0 == b1)
            continue;
        double acc[CG][10][2];
#pragma unroll
        for (int c = 0; c < CG; ++c)
#pragma unroll
            for (int t = 0; t < 10; ++t)
                acc[c][t][0] = acc[c][t][1] = 0.0;

        for (int base = b0; base < b1; base += CH) {
            const int m = min(CH, b1 - base);
            if (lane < m) {
                const double2 *r = reinterpret_cast<const double2 *>(rec + 8 * (int64_t)(base + lane));
                double2 r0 = __ldg(r), r1 = __ldg(r + 1);
                double s[NC];
                if (NC == 9) {
                    double2 r2 = __ldg(r + 2), r3 = __ldg(r + 3);
                    coeff<NC>(r1.y, r2.x, r2.y, r3.x, wscale, sigma, s);
                } else {
                    coeff<NC>(r1.y, 0, 0, 0, wscale, sigma, s);
                }
                double wx[3], wy[3], wz[3];
                weights2(r0.x, wx);
                weights2(r0.y, wy);
                weights2(r1.x, wz);
#pragma unroll
                for (int c = 0; c < CG; ++c)
                    sh_s[lane * CG + c] = s[grp * CG + c];
#pragma unroll
                for (int a = 0; a < 27; ++a)
                    sh_w[lane * 32 + a] = wx[a / 9] * wy[(a / 3) % 3] * wz[a % 3];
#pragma unroll
                for (int a = 27; a < 32; ++a)
                    sh_w[lane * 32 + a] = 0.0;
            }
            __syncwarp();
            for (int kb = 0; kb < m; kb += 4) {
                const int p = kb + (lane & 3);
                double w[4];
#pragma unroll
                for (int r = 0; r < 4; ++r)
                    w[r] = sh_w[p * 32 + 8 * r + (lane >> 2)];
#pragma unroll
                for (int c = 0; c < CG; ++c) {
                    const double s = sh_s[p * CG + c];
                    double A[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r)
                        A[r] = s * w[r];
                    dmma(acc[c][0][0], acc[c][0][1], A[0], w[0]);
                    dmma(acc[c][1][0], acc[c][1][1], A[0], w[1]);
                    dmma(acc[c][2][0], acc[c][2][1], A[0], w[2]);
                    dmma(acc[c][3][0], acc[c][3][1], A[0], w[3]);
                    dmma(acc[c][4][0], acc[c][4][1], A[1], w[1]);
                    dmma(acc[c][5][0], acc[c][5][1], A[1], w[2]);
                    dmma(acc[c][6][0], acc[c][6][1], A[1], w[3]);
                    dmma(acc[c][7][0], acc[c][7][1], A[2], w[2]);
                    dmma(acc[c][8][0], acc[c][8][1], A[2], w[3]);
                    dmma(acc[c][9][0], acc[c][9][1], A[3], w[3]);
                }
            }
            __syncwarp();
        }

        // ---- deposit: per component, stage the 10 tiles in shared memory, then
        //      RED each valid entry (a, b < 27) and, off the diagonal tiles, its mirror.
        const int bx = (int)(bin / plane), rem = (int)(bin - (int64_t)bx * plane);
        const int by = rem / g.n2, bz = rem - by * g.n2;
        const int X0 = g.x_begin + bx - 1;  // window base node along axis 0
        double *stage = smem[warp];
#pragma unroll
        for (int c = 0; c < CG; ++c) {
            __syncwarp();
#pragma unroll
            for (int t = 0; t < 10; ++t) {
                stage[t * 64 + (lane >> 2) * 8 + 2 * (lane & 3)] = acc[c][t][0];
                stage[t * 64 + (lane >> 2) * 8 + 2 * (lane & 3) + 1] = acc[c][t][1];
            }
            __syncwarp();
            const int comp = grp * CG + c;
#pragma unroll 1
            for (int e = lane; e < 640; e += 32) {
                const int t = e >> 6, tr = kTileR[t], tc = kTileC[t];
                const int a = 8 * tr + ((e >> 3) & 7), b = 8 * tc + (e & 7);
                if (a >= 27 || b >= 27)
                    continue;
                const double v = stage[e];
                const int ax = a / 9, ay = (a / 3) % 3, az = a % 3;
                const int bxx = b / 9, byy = (b / 3) % 3, bzz = b % 3;
                const int sab = (bxx - ax + 2) * 25 + (byy - ay + 2) * 5 + (bzz - az + 2);
                double *ra = row_ptr(g, X0 + ax, wrapi(by + ay, g.n1), wrapi(bz + az, g.n2), out, ghost, RL);
                atomicAdd(ra + sab * NC + comp, v);
                if (tr != tc) {
                    double *rb = row_ptr(g, X0 + bxx, wrapi(by + byy, g.n1), wrapi(bz + bzz, g.n2), out, ghost, RL);
                    atomicAdd(rb + (124 - sab) * NC + comp, v);  // slot(-d) = S-1-slot(d)
                }
            }
        }
        __syncwarp();
    }
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

}  // namespace

cudaError_t assemble_fp64_enqueue(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    if (a.nbins == 0)
        return cudaSuccess;
    if (geo.order == 1) {
        if (a.ncomp == 9) {
            k_asm_o1<9><<<grid_for(k_asm_o1<9>, a.nbins), WARPS * 32, 0, s>>>(
                geo, a.rec, a.seg_begin, a.nbins, a.wscale, a.sigma, a.out, a.ghost);
        } else {
            k_asm_o1<1><<<grid_for(k_asm_o1<1>, a.nbins), WARPS * 32, 0, s>>>(
                geo, a.rec, a.seg_begin, a.nbins, a.wscale, a.sigma, a.out, a.ghost);
        }
    } else {
        if (a.ncomp == 9) {
            k_asm_o2<9, 3><<<grid_for(k_asm_o2<9, 3>, a.nbins * 3), WARPS * 32, 0, s>>>(
                geo, a.rec, a.seg_begin, a.nbins, a.wscale, a.sigma, a.out, a.ghost);
        } else {
            k_asm_o2<1, 1><<<grid_for(k_asm_o2<1, 1>, a.nbins), WARPS * 32, 0, s>>>(
                geo, a.rec, a.seg_begin, a.nbins, a.wscale, a.sigma, a.out, a.ghost);
        }
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace mm
