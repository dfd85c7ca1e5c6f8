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

// A warp's stream of 32-particle chunks over its bins (bin, bin + W, ...; empty bins skipped).
struct ChunkIt {
    int64_t bin;
    int base, end;  // [base, end): this chunk's slots in the bin's segment; base == end: done
};
__device__ __forceinline__ ChunkIt first_chunk(int64_t bin, int64_t W, int64_t nbins, const int32_t *seg)
{
    for (; bin < nbins; bin += W) {
        const int b0 = __ldg(seg + bin), b1 = __ldg(seg + bin + 1);
        if (b1 > b0)
            return {bin, b0, b1};
    }
    return {nbins, 0, 0};
}
__device__ __forceinline__ ChunkIt next_chunk(const ChunkIt &c, int64_t W, int64_t nbins, const int32_t *seg)
{
    if (c.base + 32 < c.end)
        return {c.bin, c.base + 32, c.end};
    return first_chunk(c.bin + W, W, nbins, seg);
}

// Per-lane inputs of one chunk: record (xi, q) and the permutation entry, loaded one chunk
// ahead; the velocity (a dependent, random read through perm) is issued as soon as perm has
// arrived, i.e. one chunk ahead as well but after the current chunk's compute.
struct MoIn {
    double4 r;  // xi x, y, z, q (zeros past the bin's end)
    int p;      // caller index, -1 for padding / past the end
};
__device__ __forceinline__ MoIn load_mo(const ChunkIt &c, int lane, const double *rec, int rs, const int32_t *perm)
{
    MoIn in;
    in.r = make_double4(0, 0, 0, 0);
    in.p = -1;
    if (c.base + lane < c.end) {
        in.r = ld256(rec + (int64_t)rs * (c.base + lane));
        in.p = __ldg(perm + c.base + lane);
    }
    return in;
}

template <int ORDER, int NQ>
__global__ void __launch_bounds__(128, ORDER == 1 ? 6 : 4) k_moments(Geo g, const double *__restrict__ rec, int rs,
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
    // three-stage pipeline over the warp's chunks: records + perm two chunks ahead, the
    // velocities (random reads through perm) one chunk ahead
    const bool v16 = ((uintptr_t)v & 15) == 0;
    auto load_v = [&](const MoIn &x) {
        double3 r3 = make_double3(0, 0, 0);
        if (x.p >= 0) {
            const double *a = v + 3 * (int64_t)x.p;
            if (v16 && (x.p & 1) == 0) {  // 24 B at a random place: two requests instead of three
                const double2 u = __ldg(reinterpret_cast<const double2 *>(a));
                r3 = make_double3(u.x, u.y, __ldg(a + 2));
            } else if (v16) {
                const double2 u = __ldg(reinterpret_cast<const double2 *>(a + 1));
                r3 = make_double3(__ldg(a), u.x, u.y);
            } else {
                r3 = make_double3(__ldg(a), __ldg(a + 1), __ldg(a + 2));
            }
        }
        return r3;
    };
    ChunkIt cur = first_chunk(blockIdx.x * 4 + warp, W, nbins, seg_begin);
    ChunkIt nxt = next_chunk(cur, W, nbins, seg_begin);
    MoIn in = load_mo(cur, lane, rec, rs, perm);
    MoIn nin = load_mo(nxt, lane, rec, rs, perm);
    double3 vv = load_v(in);
    double acc[L::MT][NT][2];
#pragma unroll
    for (int i = 0; i < L::MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
            acc[i][j][0] = acc[i][j][1] = 0.0;
    while (cur.bin < nbins) {
        const ChunkIt nxt2 = next_chunk(nxt, W, nbins, seg_begin);
        const MoIn nin2 = load_mo(nxt2, lane, rec, rs, perm);
        const double3 nvv = load_v(nin);
        const int m = min(32, cur.end - cur.base);
        __syncwarp();  // the previous chunk's DMMAs / deposit are done with xz
        {
            double wx[3], wy[3], wz[3];
            axis_weights<ORDER>(in.r.x, wx);
            axis_weights<ORDER>(in.r.y, wy);
            axis_weights<ORDER>(in.r.z, wz);
            double *col = xz + lane;
#pragma unroll
            for (int a = 0; a < L::N; ++a) {
                const int ax = a / ((ORDER + 1) * (ORDER + 1)), ay = (a / (ORDER + 1)) % (ORDER + 1),
                          az = a % (ORDER + 1);
                col[a * L::XS] = (wx[ax] * wy[ay]) * wz[az];
            }
            const double s = sigma * in.r.w;  // 0 past the bin's end / on padding records
            const double vx = vv.x, vy = vv.y, vz = vv.z;
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
        if (nxt.bin != cur.bin) {
            // ---- the bin is complete: D tile (i, j) element (rq, 2 kq + u) = node 8 i + rq,
            //      quantity 8 j + 2 kq + u -> stage -> REDs into the node rows
            __syncwarp();
#pragma unroll
            for (int i = 0; i < L::MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j)
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const int a = 8 * i + rq, q = 8 * j + 2 * kq + u;
                        if (a < L::N && q < NQ)
                            stage[a * NQ + q] = acc[i][j][u];
                        acc[i][j][u] = 0.0;
                    }
            const int bin = (int)cur.bin;
            const int bxl = bin / plane, rem = bin - bxl * plane, bx = g.bx0 + bxl;
            const int by = rem / g.n2, bz = rem - by * g.n2;
            if (lane < L::N) {
                const int a = lane, ax = a / ((ORDER + 1) * (ORDER + 1)), ay = (a / (ORDER + 1)) % (ORDER + 1),
                          az = a % (ORDER + 1);
                rowp[a] = row_ptr(g, g.x_begin + bx - (ORDER - 1) + ax, wrapi(by + ay, g.n1), wrapi(bz + az, g.n2),
                                  out, ghost, NQ);
            }
            __syncwarp();
            for (int e = lane; e < NE; e += 32)
                red_add_nc(rowp[e / NQ] + e % NQ, stage[e]);
        }
        cur = nxt;
        nxt = nxt2;
        in = nin;
        nin = nin2;
        vv = nvv;
    }
}

template <int ORDER>
__global__ void __launch_bounds__(128) k_gather(Geo g, double *__restrict__ rec, const int32_t *__restrict__ perm,
                                                const int32_t *__restrict__ seg_begin, int64_t nbins,
                                                const double *__restrict__ F, double *__restrict__ Fp)
{
    using L = Mo<ORDER>;
    __shared__ double sF[4][2][L::N * 3];  // the window's nodal field, double-buffered by bin
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int plane = g.n1 * g.n2;
    const int64_t W = (int64_t)gridDim.x * 4;
    // the window's nodal values of a bin (whole periodic domain, global x), one node per lane
    auto load_f = [&](int64_t bin, double f3[3]) {
        f3[0] = f3[1] = f3[2] = 0.0;
        if (bin < nbins && lane < L::N) {
            const int b = (int)bin, bxl = b / plane, rem = b - bxl * plane, bx = g.bx0 + bxl;
            const int by = rem / g.n2, bz = rem - by * g.n2;
            const int a = lane, ax = a / ((ORDER + 1) * (ORDER + 1)), ay = (a / (ORDER + 1)) % (ORDER + 1),
                      az = a % (ORDER + 1);
            int X = g.x_begin + bx - (ORDER - 1) + ax;
            X = X < 0 ? X + g.n0 : (X >= g.n0 ? X - g.n0 : X);
            const double *f = F + 3 * (((int64_t)X * g.n1 + wrapi(by + ay, g.n1)) * g.n2 + wrapi(bz + az, g.n2));
            f3[0] = __ldg(f), f3[1] = __ldg(f + 1), f3[2] = __ldg(f + 2);
        }
    };
    // two chunks of records + perm in flight (the per-particle work is a few FMAs)
    auto load_rp = [&](const ChunkIt &c, double4 &r, int &p) {
        r = make_double4(0, 0, 0, 0);
        p = -1;
        if (c.base + lane < c.end) {
            r = ld256(rec + 8 * (int64_t)(c.base + lane));
            p = __ldg(perm + c.base + lane);
        }
    };
    const bool fp16 = ((uintptr_t)Fp & 15) == 0;
    ChunkIt cur = first_chunk(blockIdx.x * 4 + warp, W, nbins, seg_begin);
    ChunkIt nxt = next_chunk(cur, W, nbins, seg_begin);
    double4 r, nr;
    int p, np_;
    load_rp(cur, r, p);
    load_rp(nxt, nr, np_);
    double f3[3];
    load_f(cur.bin, f3);
    int fb = 0;
    int64_t fbin = -1;
    while (cur.bin < nbins) {
        if (cur.bin != fbin) {  // new bin: its window's field (loaded one bin ahead) into shared memory
            fb ^= 1;
            if (lane < L::N)
                sF[warp][fb][3 * lane] = f3[0], sF[warp][fb][3 * lane + 1] = f3[1], sF[warp][fb][3 * lane + 2] = f3[2];
            fbin = cur.bin;
            __syncwarp();
            // the field of the next bin the stream reaches
            load_f(first_chunk(cur.bin + W, W, nbins, seg_begin).bin, f3);
        }
        const ChunkIt nxt2 = next_chunk(nxt, W, nbins, seg_begin);
        double4 nr2;
        int np2;
        load_rp(nxt2, nr2, np2);
        if (p >= 0) {
            double wx[3], wy[3], wz[3];
            axis_weights<ORDER>(r.x, wx);
            axis_weights<ORDER>(r.y, wy);
            axis_weights<ORDER>(r.z, wz);
            const double *sf = sF[warp][fb];
            double b[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int a = 0; a < L::N; ++a) {
                const int ax = a / ((ORDER + 1) * (ORDER + 1)), ay = (a / (ORDER + 1)) % (ORDER + 1),
                          az = a % (ORDER + 1);
                const double wa = (wx[ax] * wy[ay]) * wz[az];
                b[0] = fma(wa, sf[3 * a], b[0]);
                b[1] = fma(wa, sf[3 * a + 1], b[1]);
                b[2] = fma(wa, sf[3 * a + 2], b[2]);
            }
            // the record's second sector {B, 0} as ONE full 32-B store (no partial-sector write)
            double *rr = rec + 8 * (int64_t)(cur.base + lane) + 4;
            asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(rr), "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(0.0)
                         : "memory");
            if (Fp) {
                // 24 B at a random place: two requests (16-B aligned pair + single) instead of three
                double *f = Fp + 3 * (int64_t)p;
                if (fp16) {
                    if ((p & 1) == 0) {
                        asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(f), "d"(b[0]), "d"(b[1]) : "memory");
                        f[2] = b[2];
                    } else {
                        f[0] = b[0];
                        asm volatile("st.global.v2.f64 [%0], {%1,%2};" ::"l"(f + 1), "d"(b[1]), "d"(b[2]) : "memory");
                    }
                } else {
                    f[0] = b[0], f[1] = b[1], f[2] = b[2];
                }
            }
        }
        cur = nxt;
        nxt = nxt2;
        r = nr;
        p = np_;
        nr = nr2;
        np_ = np2;
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
