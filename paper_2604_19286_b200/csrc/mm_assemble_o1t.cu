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
//   T3       A as above                                   B[k][n] = V_k[n]  (columns 0-2 kept)
//   T4       A'[c][k] = s_k[c] (c < 8)                    B[k][n] = V_k[n]  (columns 3-5 kept)
//            V = (qz0 s8, qz1 s8, qz2 s8, X8 qz0, X8 qz1, X8 qz2, 0, 0)
//   SIMT     (uxy = 8, uz, c = 8): three FMAs per particle in the prep, reduced per bin.
// The B values are formed in registers from compact per-particle rows (X, s, xi_z, V) staged
// in shared memory once per chunk: 23 staged values per particle instead of the 36 operand
// columns of a fully staged plan, 4 LDS.128 per two batches (a shared-memory load costs
// 32 lanes x its width regardless of broadcast, so the per-lane bytes are what count), the
// pair products q_z recomputed from xi_z in registers, and 5 instead of 8 DMMAs per batch
// (640 instead of 1024 executed FLOP per particle; F_unique = 648).
//
// Deposit: the 243 sums are staged in shared memory and added into the 8 node rows of the bin
// (576 entries) with REDs in the address order of each row, into an output zeroed just before
// the launch.  Bins are visited in DESCENDING order (static interleaved schedule: warp w takes
// bins nbins-1-w, nbins-1-w-W, ...), so the first REDs hit the rows the memset wrote last,
// which are still in L2.  Records are read with an L2 evict-first hint (streamed once), so the
// 126 MB L2 keeps node rows rather than records.
#include "mm_device.cuh"

#ifndef O1T_MINB
#define O1T_MINB 5  // resident CTAs per SM the register allocation targets (96 registers)
#endif

namespace mm {

namespace {

using namespace dev;

struct O1T {
    static constexpr int WARPS = 4;
    static constexpr int XS = 40;   // row stride (doubles), = 8 mod 16: LDS.128 fragment loads conflict-free
    static constexpr int ROWS = 24; // 0-7 X, 8-15 s[0..7], 16 xi_z, 17-22 V, 23 zeros
    static constexpr int R_S = 8, R_Z = 16, R_V = 17, R_ZERO = 23;
    static constexpr int WD = ROWS * XS;  // the stage [9][27] aliases rows 0..6
    static constexpr size_t SMEM = (size_t)WARPS * WD * 8 + 576 * 4 + WARPS * 8 * 8;
};

__global__ void __launch_bounds__(O1T::WARPS * 32, O1T_MINB)
    k_asm_o1t(Geo g, const double *__restrict__ rec, const int32_t *__restrict__ seg_begin, int64_t nbins,
              double wscale, double sigma, double *__restrict__ out, double *__restrict__ ghost)
{
    using L = O1T;
    extern __shared__ __align__(16) double dsm_o1t[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *xz = dsm_o1t + warp * L::WD;
    double *stage = xz;  // [9 uxy][27 = 9 uz + c] after the last batch of a bin
    int32_t *s_dep = reinterpret_cast<int32_t *>(dsm_o1t + L::WARPS * L::WD);
    double **s_row = reinterpret_cast<double **>(s_dep + 576) + warp * 8;                // node rows
    const int plane = g.n1 * g.n2;

    // RED table, element e = (a, b, c) in address order of node a's row:
    // a (3 bits) | slot*9 + c (8 bits) | stage index (uxy * 27 + 9 uz + c, 8 bits)
    for (int e = threadIdx.x; e < 576; e += blockDim.x) {
        const int a = e / 72, r = e - a * 72, b = r / 9, c = r - b * 9;
        const int ax = a >> 2, ay = (a >> 1) & 1, az = a & 1, bx = b >> 2, by = (b >> 1) & 1, bz = b & 1;
        const int slot = (bx - ax + 1) * 9 + (by - ay + 1) * 3 + (bz - az + 1);
        const int m = 3 * (ax + bx) + (ay + by), n = 9 * (az + bz) + c;
        s_dep[e] = a | ((slot * 9 + c) << 3) | ((m * 27 + n) << 11);
    }
    xz[L::R_ZERO * L::XS + lane] = 0.0;
    xz[L::R_ZERO * L::XS + 32 + (lane & 7)] = 0.0;
    __syncthreads();

    const int kq = lane & 3, rq = lane >> 2;
    const double *fx = xz + rq * L::XS + 2 * kq;                               // X[r]
    const double *fs = xz + (L::R_S + rq) * L::XS + 2 * kq;                    // s[r]
    const double *fz = xz + L::R_Z * L::XS + 2 * kq;                           // xi_z -> qz[0..2]
    // T3 and T4 share ONE B operand, V = (qz0 s8, qz1 s8, qz2 s8, X8 qz0, X8 qz1, X8 qz2, 0, 0):
    // T3 (A = X) keeps its columns 0-2, T4 (A = s) its columns 3-5; the other columns are
    // never read, so no lane needs a select
    const double *fv = xz + (rq < 6 ? L::R_V + rq : L::R_ZERO) * L::XS + 2 * kq;

    const int64_t W = (int64_t)gridDim.x * L::WARPS;
    int64_t t = blockIdx.x * L::WARPS + warp;  // this warp's k-th bin is nbins - 1 - (t + k W)
    int b0 = 0, b1 = 0, nb0 = 0, nb1 = 0;
    if (t < nbins) {
        b0 = __ldg(seg_begin + (nbins - 1 - t));
        b1 = __ldg(seg_begin + (nbins - t));
    }
    if (t + W < nbins) {
        nb0 = __ldg(seg_begin + (nbins - 1 - t - W));
        nb1 = __ldg(seg_begin + (nbins - t - W));
    }
    // the lane's record of the current chunk, loaded one chunk ahead; lanes past the end of a
    // bin hold zeros (q = 0 -> exact +0 contributions)
    double4 ra = make_double4(0, 0, 0, 0), rb = ra;
    if (t < nbins && b0 + lane < b1) {
        ra = ld256_ef(rec + 8 * (int64_t)(b0 + lane));
        rb = ld256_ef(rec + 8 * (int64_t)(b0 + lane) + 4);
    }
    for (; t < nbins; t += W) {
        const int64_t bin = nbins - 1 - t;
        int nn0 = 0, nn1 = 0;
        if (t + 2 * W < nbins) {
            nn0 = __ldg(seg_begin + (nbins - 1 - t - 2 * W));
            nn1 = __ldg(seg_begin + (nbins - t - 2 * W));
        }
        const int bxl = (int)(bin / plane), rem = (int)(bin - (int64_t)bxl * plane), bx = g.bx0 + bxl;
        const int by = rem / g.n2, bz = rem - by * g.n2;
        if (b1 > b0) {
            {
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
                        } else if (t + W < nbins && nb0 + lane < nb1) {
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
                        col[L::R_Z * L::XS] = ca.z;
#pragma unroll
                        for (int u = 0; u < 3; ++u) {
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
                        // 4 LDS.128 (16 wavefronts) per two batches: X[r], s[r], xi_z, V[r]
                        const double2 X = lds128(fx + o), S = lds128(fs + o), Z = lds128(fz + o), V = lds128(fv + o);
                        auto batch = [&](double x, double sv, double z, double v) {
                            const double w0 = 1.0 - z;
                            const double q0 = w0 * w0, q1 = w0 * z, q2 = z * z;
                            dmma(acc[0][0], acc[0][1], x, q0 * sv);
                            dmma(acc[1][0], acc[1][1], x, q1 * sv);
                            dmma(acc[2][0], acc[2][1], x, q2 * sv);
                            dmma(acc[3][0], acc[3][1], x, v);
                            dmma(acc[4][0], acc[4][1], sv, v);
                        };
                        batch(X.x, S.x, Z.x, V.x);
                        batch(X.y, S.y, Z.y, V.y);
                    };
                    const int np8 = (m + 7) >> 3;
#pragma unroll 1
                    for (int i = 0; i < np8; ++i)
                        pair(i);
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
                    const int cc = 2 * kq + v;
#pragma unroll
                    for (int nt = 0; nt < 3; ++nt)
                        stage[rq * 27 + 9 * nt + cc] = acc[nt][v];     // T0..T2: (uxy r, uz nt, c)
                    if (cc < 3)
                        stage[rq * 27 + 9 * cc + 8] = acc[3][v];       // T3: (uxy r, uz cc, c 8)
                    else if (cc < 6)
                        stage[8 * 27 + 9 * (cc - 3) + rq] = acc[4][v]; // T4: (uxy 8, uz cc - 3, c r)
                }
                if (lane < 3)
                    stage[8 * 27 + 9 * lane + 8] = lane == 0 ? acc8[0] : (lane == 1 ? acc8[1] : acc8[2]);
                if (lane < 8)
                    s_row[lane] = row_ptr(g, g.x_begin + bx + (lane >> 2), wrapi(by + ((lane >> 1) & 1), g.n1),
                                          wrapi(bz + (lane & 1), g.n2), out, ghost, 243);
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 18; ++i) {
                    const int e = s_dep[i * 32 + lane];
                    red_add(s_row[e & 7] + ((e >> 3) & 255), stage[e >> 11]);
                }
            }
        } else if (t + W < nbins && nb0 + lane < nb1) {
            // empty bin: nothing was prefetched for the successor yet
            ra = ld256_ef(rec + 8 * (int64_t)(nb0 + lane));
            rb = ld256_ef(rec + 8 * (int64_t)(nb0 + lane) + 4);
        }
        b0 = nb0;
        b1 = nb1;
        nb0 = nn0;
        nb1 = nn1;
    }
}

}  // namespace

cudaError_t launch_o1t(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    using L = O1T;
    cudaError_t e = cudaFuncSetAttribute(k_asm_o1t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
    if (e)
        return e;
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_asm_o1t, L::WARPS * 32, L::SMEM);
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

}  // namespace mm
