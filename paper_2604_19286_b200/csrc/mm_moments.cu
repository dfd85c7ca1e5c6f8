// NEXT-4: the assembly's machinery for the other particle <-> grid operations
// of a PIC cycle.
//
// * Moment deposition: "the same tensor-contraction approach extends to any
//   particle-to-grid scatter operation, where one MMA operand encodes the deposited quantities
//   and the other encodes the interpolation weights":
//       mom[g][m] = sigma sum_p Q_p^m W_pg,  Q = q (1, v) (nq = 4: rho, J) or
//                   q (1, v, vv^T upper) (nq = 10: implicit-moment quantities)
//   per support-window bin (the sort's bins, R12) as ONE product over its particles on
//   FP64 DMMA tiles: D[a][m] = sum_k W_a(k) Q_m(k), A = the node weights (8 | 27 rows -> 1 | 4
//   row tiles), B = the quantities (4 | 10 -> 1 | 2 column tiles of 8).  CIC with nq = 4 is the
//   paper's half-occupied (8,8,4) tile; nq = 10 fills 10 of 16 columns.  The block is then added
//   into the node rows (nq contiguous doubles per node) with REDs, ghost planes for slabs.
//   Velocities are read through the sort's permutation (the records carry xi, q and B).
//
// * Field gather, PAPER.md:96 ("B(x_p) being the magnetic field interpolated to the particle
//   position"): F_p = sum_g W_pg F_g for the sorted particles of each bin, the window's nodal
//   values staged once per bin.  The result is written into the handle's records (the B the
//   next mm_assemble reads: gather -> alpha -> mass matrix without a re-sort) and optionally to an
//   array in the caller's particle order.  8 | 27 x 3 FMAs against 64 + 24 B per particle: HBM-
//   bound by an order of magnitude, so it runs on the FP64 SIMT pipe, not on DMMA tiles.
#include "mm_device.cuh"

namespace mm {
namespace {

using namespace dev;

template <int ORDER>
struct Mo {
    static constexpr int N = ORDER == 1 ? 8 : 27;   // support nodes
    static constexpr int MT = (N + 7) / 8;          // row tiles
    static constexpr int XS = 36;                   // row stride (doubles)
};

// per-axis weights at the window's nodes (CIC: w = (1 - xi, xi); TSC: weights2u of DESIGN.md §7)
template <int ORDER>
__device__ __forceinline__ void axis_weights(double xi, double w[3])
{
    if (ORDER == 1) {
        w[0] = 1.0 - xi;
        w[1] = xi;
        w[2] = 0.0;
    } else {
        unsigned lo, hi;
        asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(xi));
        const double u = hi >= 0x3fe00000u ? xi - 1.0 : xi;  // xi >= 1/2: base 0, else -1 (R4)
        const double h = 0.5 - u, k = 0.5 + u;
        w[0] = (0.5 * h) * h;
        w[1] = fma(-u, u, 0.75);
        w[2] = (0.5 * k) * k;
    }
}

template <int ORDER, int NQ>
__global__ void __launch_bounds__(128) k_moments(Geo g, const double *__restrict__ rec, int rs,
                                                 const int32_t *__restrict__ perm,
                                                 const int32_t *__restrict__ seg_begin, int64_t nbins,
                                                 const double *__restrict__ v, double sigma,
                                                 double *__restrict__ out, double *__restrict__ ghost)
{
    using L = Mo<ORDER>;
    constexpr int NT = (NQ + 7) / 8;               // column tiles
    constexpr int ROWS = 8 * L::MT + 8 * NT;        // W rows (padded) then Q rows (padded)
    constexpr int NE = L::N * NQ;                   // block entries
    extern __shared__ __align__(16) double dsm_mo[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *xz = dsm_mo + warp * (ROWS * L::XS + NE + 32);
    double *stage = xz + ROWS * L::XS;             // [N][NQ]
    double **rowp = reinterpret_cast<double **>(stage + NE);
    const int plane = g.n1 * g.n2;
    // padding rows of the operand tiles are zero once and for all
    for (int r = 0; r < ROWS; ++r)
        if ((r >= L::N && r < 8 * L::MT) || r >= 8 * L::MT + NQ)
            xz[r * L::XS + lane] = 0.0;
    __syncwarp();
    const int kq = lane & 3, rq = lane >> 2;
    const int64_t W = (int64_t)gridDim.x * 4;
    for (int64_t bin = blockIdx.x * 4 + warp; bin < nbins; bin += W) {
        const int b0 = __ldg(seg_begin + bin), b1 = __ldg(seg_begin + bin + 1);
        if (b1 == b0)
            continue;
        double acc[L::MT][NT][2];
#pragma unroll
        for (int i = 0; i < L::MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j)
                acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int base = b0; base < b1; base += 32) {
            const int m = min(32, b1 - base);
            double xi[3] = {0.0, 0.0, 0.0}, qq = 0.0, vx = 0.0, vy = 0.0, vz = 0.0;
            if (lane < m) {
                const double *r = rec + (int64_t)rs * (base + lane);
                xi[0] = r[0], xi[1] = r[1], xi[2] = r[2], qq = r[3];
                const int p = __ldg(perm + base + lane);
                if (p >= 0) {
                    vx = __ldg(v + 3 * (int64_t)p), vy = __ldg(v + 3 * (int64_t)p + 1), vz = __ldg(v + 3 * (int64_t)p + 2);
                }
            }
            __syncwarp();
            {
                double wx[3], wy[3], wz[3];
                axis_weights<ORDER>(xi[0], wx);
                axis_weights<ORDER>(xi[1], wy);
                axis_weights<ORDER>(xi[2], wz);
                double *col = xz + lane;
#pragma unroll
                for (int a = 0; a < L::N; ++a) {
                    const int ax = a / ((ORDER + 1) * (ORDER + 1)), ay = (a / (ORDER + 1)) % (ORDER + 1),
                              az = a % (ORDER + 1);
                    col[a * L::XS] = (wx[ax] * wy[ay]) * wz[az];
                }
                const double s = sigma * qq;  // 0 past the bin's end / on padding records
                double Q[10] = {s, s * vx, s * vy, s * vz, 0, 0, 0, 0, 0, 0};
                if (NQ == 10) {
                    Q[4] = s * (vx * vx), Q[5] = s * (vx * vy), Q[6] = s * (vx * vz);
                    Q[7] = s * (vy * vy), Q[8] = s * (vy * vz), Q[9] = s * (vz * vz);
                }
#pragma unroll
                for (int q = 0; q < NQ; ++q)
                    col[(8 * L::MT + q) * L::XS] = Q[q];
            }
            __syncwarp();
            for (int kb = 0; kb < m; kb += 4) {
                double bv[NT];
#pragma unroll
                for (int j = 0; j < NT; ++j)
                    bv[j] = xz[(8 * L::MT + 8 * j + rq) * L::XS + kb + kq];
#pragma unroll
                for (int i = 0; i < L::MT; ++i) {
                    const double av = xz[(8 * i + rq) * L::XS + kb + kq];
#pragma unroll
                    for (int j = 0; j < NT; ++j)
                        dmma(acc[i][j][0], acc[i][j][1], av, bv[j]);
                }
            }
        }
        __syncwarp();
        // D tile (i, j) element (rq, 2 kq + v): node 8 i + rq, quantity 8 j + 2 kq + v
#pragma unroll
        for (int i = 0; i < L::MT; ++i)
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int a = 8 * i + rq, q = 8 * j + 2 * kq + u;
                    if (a < L::N && q < NQ)
                        stage[a * NQ + q] = acc[i][j][u];
                }
        const int bxl = (int)(bin / plane), rem = (int)(bin - (int64_t)bxl * plane), bx = g.bx0 + bxl;
        const int by = rem / g.n2, bz = rem - by * g.n2;
        if (lane < L::N) {
            const int a = lane, ax = a / ((ORDER + 1) * (ORDER + 1)), ay = (a / (ORDER + 1)) % (ORDER + 1),
                      az = a % (ORDER + 1);
            rowp[a] = row_ptr(g, g.x_begin + bx - (ORDER - 1) + ax, wrapi(by + ay, g.n1), wrapi(bz + az, g.n2), out,
                              ghost, NQ);
        }
        __syncwarp();
        for (int e = lane; e < NE; e += 32)
            red_add(rowp[e / NQ] + e % NQ, stage[e]);
        __syncwarp();
    }
}

template <int ORDER>
__global__ void __launch_bounds__(128) k_gather(Geo g, double *__restrict__ rec, const int32_t *__restrict__ perm,
                                                const int32_t *__restrict__ seg_begin, int64_t nbins,
                                                const double *__restrict__ F, double *__restrict__ Fp)
{
    using L = Mo<ORDER>;
    __shared__ double sF[4][L::N * 3];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int plane = g.n1 * g.n2;
    const int64_t W = (int64_t)gridDim.x * 4;
    for (int64_t bin = blockIdx.x * 4 + warp; bin < nbins; bin += W) {
        const int b0 = __ldg(seg_begin + bin), b1 = __ldg(seg_begin + bin + 1);
        if (b1 == b0)
            continue;
        const int bxl = (int)(bin / plane), rem = (int)(bin - (int64_t)bxl * plane), bx = g.bx0 + bxl;
        const int by = rem / g.n2, bz = rem - by * g.n2;
        __syncwarp();
        if (lane < L::N) {  // the window's nodal field (whole periodic domain, global x)
            const int a = lane, ax = a / ((ORDER + 1) * (ORDER + 1)), ay = (a / (ORDER + 1)) % (ORDER + 1),
                      az = a % (ORDER + 1);
            int X = g.x_begin + bx - (ORDER - 1) + ax;
            X = X < 0 ? X + g.n0 : (X >= g.n0 ? X - g.n0 : X);
            const double *f = F + 3 * (((int64_t)X * g.n1 + wrapi(by + ay, g.n1)) * g.n2 + wrapi(bz + az, g.n2));
            sF[warp][3 * a] = __ldg(f), sF[warp][3 * a + 1] = __ldg(f + 1), sF[warp][3 * a + 2] = __ldg(f + 2);
        }
        __syncwarp();
        for (int s = b0 + lane; s < b1; s += 32) {
            const int p = __ldg(perm + s);
            if (p < 0)
                continue;  // padding record: its B stays 0
            double *r = rec + 8 * (int64_t)s;
            double wx[3], wy[3], wz[3];
            axis_weights<ORDER>(r[0], wx);
            axis_weights<ORDER>(r[1], wy);
            axis_weights<ORDER>(r[2], wz);
            double b[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int a = 0; a < L::N; ++a) {
                const int ax = a / ((ORDER + 1) * (ORDER + 1)), ay = (a / (ORDER + 1)) % (ORDER + 1),
                          az = a % (ORDER + 1);
                const double wa = (wx[ax] * wy[ay]) * wz[az];
                b[0] = fma(wa, sF[warp][3 * a], b[0]);
                b[1] = fma(wa, sF[warp][3 * a + 1], b[1]);
                b[2] = fma(wa, sF[warp][3 * a + 2], b[2]);
            }
            r[4] = b[0], r[5] = b[1], r[6] = b[2];
            if (Fp) {
                Fp[3 * (int64_t)p] = b[0], Fp[3 * (int64_t)p + 1] = b[1], Fp[3 * (int64_t)p + 2] = b[2];
            }
        }
    }
}

unsigned grid_of(int64_t nbins, int per_sm)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (nbins + 3) / 4, cap = (int64_t)sms * per_sm;
    return (unsigned)(want < cap ? (want < 1 ? 1 : want) : cap);
}

template <int ORDER, int NQ>
cudaError_t launch_moments(const Geo &g, const double *rec, int rs, const int32_t *perm, const int32_t *seg,
                           int64_t nbins, const double *v, double sigma, double *out, double *ghost, cudaStream_t s)
{
    using L = Mo<ORDER>;
    constexpr int NT = (NQ + 7) / 8;
    const size_t smem = (size_t)4 * ((8 * L::MT + 8 * NT) * L::XS + L::N * NQ + 32) * 8;
    cudaError_t e = cudaFuncSetAttribute(k_moments<ORDER, NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e)
        return e;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_moments<ORDER, NQ>, 128, smem);
    k_moments<ORDER, NQ><<<grid_of(nbins, per_sm > 0 ? per_sm : 1), 128, smem, s>>>(g, rec, rs, perm, seg, nbins, v,
                                                                                     sigma, out, ghost);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t moments_enqueue(const Geo &g, int nq, const double *rec, int rs, const int32_t *perm,
                            const int32_t *seg_begin, int64_t nbins, const double *v, double sigma, double *out,
                            double *ghost, cudaStream_t s)
{
    if (nbins == 0)
        return cudaSuccess;
    if (g.order == 1)
        return nq == 4 ? launch_moments<1, 4>(g, rec, rs, perm, seg_begin, nbins, v, sigma, out, ghost, s)
                       : launch_moments<1, 10>(g, rec, rs, perm, seg_begin, nbins, v, sigma, out, ghost, s);
    return nq == 4 ? launch_moments<2, 4>(g, rec, rs, perm, seg_begin, nbins, v, sigma, out, ghost, s)
                   : launch_moments<2, 10>(g, rec, rs, perm, seg_begin, nbins, v, sigma, out, ghost, s);
}

cudaError_t gather_enqueue(const Geo &g, double *rec, const int32_t *perm, const int32_t *seg_begin, int64_t nbins,
                           const double *F, double *Fp, cudaStream_t s)
{
    if (nbins == 0)
        return cudaSuccess;
    int per_sm = 0;
    if (g.order == 1) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather<1>, 128, 0);
        k_gather<1><<<grid_of(nbins, per_sm > 0 ? per_sm : 1), 128, 0, s>>>(g, rec, perm, seg_begin, nbins, F, Fp);
    } else {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gather<2>, 128, 0);
        k_gather<2><<<grid_of(nbins, per_sm > 0 ? per_sm : 1), 128, 0, s>>>(g, rec, perm, seg_begin, nbins, F, Fp);
    }
    count_launch();
    return cudaGetLastError();
}

}  // namespace mm
