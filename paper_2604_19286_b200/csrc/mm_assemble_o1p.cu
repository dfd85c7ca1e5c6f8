// Order-1 FP64 DMMA assembly, software-pipelined (the production order-1 kernel).
//
// Same arithmetic as k_asm_o1 (mm_assemble_fp64.cu; Algorithm 1):
// per support-window bin (= cell for CIC), batches of K_t = 4 particles,
// A^{ij}_{ak} = W_a(p_k) s^{ij}(p_k), B_{kb} = W_b(p_k), D^{ij} += A^{ij} B on
// mma.sync.m8n8k4.f64, then the node-stencil deposit.  What differs is the schedule.
// Per-phase timers showed a warp of k_asm_o1 spent only ~50% of its time in the DMMA
// batch loop (prep 21%, deposit 28%).  Here every warp runs one instruction stream in
// which, while the DMMAs of chunk c are issued,
//   * the records of chunk c+2 arrive by TMA (cp.async.bulk, 2 KB, double-buffered),
//   * the per-particle prep of chunk c+1 (alpha, s, W) is computed in registers, and
//   * the REDs of the previous bin's staged tile are issued,
// so the FP64 pipe keeps DMMA work while the other units do the rest.
//
// Work split: a warp owns units of U consecutive bins (their records are contiguous);
// unit k of warp w is k*W + w (W = warps in the grid), so concurrently processed bins
// are neighbours and the deposited node rows stay L2-resident.
#include "mm_internal.cuh"

namespace mm {

namespace {

constexpr int W1 = 4;    // warps per CTA
constexpr int U = 16;    // bins per unit
constexpr int CH = 32;   // particles per chunk
constexpr int WS = 36;   // weight tile row stride (doubles)

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void red_add(double *p, double v)
{
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
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
    return ghost + ((int64_t)(0 * g.n1 + Y) * g.n2 + Z) * rowlen;  // order 1: ghost plane x_end
}

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

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

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

template <int NC>
struct P1 {
    static constexpr int SS = NC == 9 ? 10 : 2;        // s row stride (even: LDS.128 pairs)
    static constexpr int PREP = 8 * WS + CH * SS;       // weight tile + s rows
    static constexpr int STAGE = 64 * NC;               // staged D[a][b][c]
    static constexpr int PSZ = PREP > STAGE ? PREP : STAGE;
    static constexpr int NDEP = 64 * NC / 32;           // deposit elements per lane
    // per warp: R[2][CH*8] records | P[2][PSZ] prep/stage | seg[3][U+1] ints | bar[2]
    static constexpr int WARP_DOUBLES = (2 * CH * 8 + 2 * PSZ + (3 * (U + 1) + 1) / 2 + 1 + 2 + 15) / 16 * 16;  // 128-B aligned
    static constexpr size_t SMEM = (size_t)W1 * WARP_DOUBLES * 8 + 64 * NC * 4;
};

// A chunk of the warp's stream: unit u (< 0: end), seg slot, bin i of the unit,
// records [base, base + cnt), end of its bin.
struct Chunk {
    int u, slot, i, base, cnt, end;
};

}  // namespace

template <int NC>
__global__ void __launch_bounds__(W1 * 32) k_asm_o1p(Geo g, const double *__restrict__ rec,
                                                     const int32_t *__restrict__ seg_begin, int nbins, double wscale,
                                                     double sigma, double *__restrict__ out,
                                                     double *__restrict__ ghost)
{
    using L = P1<NC>;
    extern __shared__ __align__(128) double dsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *wsm = dsm + warp * L::WARP_DOUBLES;
    double *R = wsm;                                   // [2][CH*8]
    double *P = wsm + 2 * CH * 8;                      // [2][PSZ]
    int *seg = reinterpret_cast<int *>(P + 2 * L::PSZ);  // [3][U+1]
    uint64_t *bar = reinterpret_cast<uint64_t *>(wsm + L::WARP_DOUBLES - 2);
    int *s_tab = reinterpret_cast<int *>(dsm + W1 * L::WARP_DOUBLES);
    const int plane = g.n1 * g.n2;
    constexpr int RL = 27 * NC;

    for (int e = threadIdx.x; e < 64 * NC; e += blockDim.x) {
        const int a = e / (8 * NC), rr = e - a * 8 * NC, b = rr / NC, c = rr - b * NC;
        const int slot = ((b >> 2) - (a >> 2) + 1) * 9 + (((b >> 1) & 1) - ((a >> 1) & 1) + 1) * 3 + ((b & 1) - (a & 1) + 1);
        s_tab[e] = a | ((slot * NC + c) << 3);
    }
    if (lane == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int nunits = (nbins + U - 1) / U;
    const int nw = gridDim.x * W1;
    int unit_next = blockIdx.x * W1 + warp;  // next unit to load
    int slot_next = 0;

    // load the seg_begin entries of the next unit of this warp into the next slot
    auto load_unit = [&](int &u, int &slot) {
        u = unit_next < nunits ? unit_next : -1;
        slot = slot_next;
        if (u >= 0) {
            if (lane <= U) {
                const int idx = min(u * U + lane, nbins);
                seg[slot * (U + 1) + lane] = __ldg(seg_begin + idx);
            }
            __syncwarp();
            unit_next += nw;
            slot_next = slot_next == 2 ? 0 : slot_next + 1;
        }
    };
    // first chunk at or after bin i of unit (u, slot); loads further units as needed
    auto first_chunk = [&](int u, int slot, int i) {
        Chunk c;
        for (;;) {
            if (u < 0) {
                c.u = -1;
                c.slot = 0;
                c.i = 0;
                c.base = 0;
                c.cnt = 0;
                c.end = 0;
                return c;
            }
            const int *sg = seg + slot * (U + 1);
            const int nb = min(U, nbins - u * U);
            while (i < nb && sg[i + 1] == sg[i])
                ++i;
            if (i < nb) {
                c.u = u;
                c.slot = slot;
                c.i = i;
                c.base = sg[i];
                c.end = sg[i + 1];
                c.cnt = min(CH, c.end - c.base);
                return c;
            }
            load_unit(u, slot);
            i = 0;
        }
    };
    auto next_chunk = [&](const Chunk &c) {
        if (c.u < 0)
            return c;
        if (c.base + CH < c.end) {
            Chunk n = c;
            n.base = c.base + CH;
            n.cnt = min(CH, c.end - n.base);
            return n;
        }
        return first_chunk(c.u, c.slot, c.i + 1);
    };

    int u0, s0;
    load_unit(u0, s0);
    Chunk C0 = first_chunk(u0, s0, 0);
    Chunk C1 = next_chunk(C0);
    Chunk C2 = next_chunk(C1);

    // preamble: records of C0 (and C1 in flight), prep of C0
    if (C0.u >= 0) {
        if (lane == 0) {
            tma_load(R, rec + 8 * (int64_t)C0.base, C0.cnt * 64, &bar[0]);
            if (C1.u >= 0)
                tma_load(R + CH * 8, rec + 8 * (int64_t)C1.base, C1.cnt * 64, &bar[1]);
        }
        mbar_wait(&bar[0], 0);
    }

    double *myrow = nullptr;  // node-row pointer of lane & 7 for the pending deposit
    bool pend = false;
    double acc[NC][2];
#pragma unroll
    for (int c = 0; c < NC; ++c)
        acc[c][0] = acc[c][1] = 0.0;

    // prep of one particle (record r) into registers
    auto prep_regs = [&](const double *r, double s[NC], double w8[8]) {
        const double2 ra = *reinterpret_cast<const double2 *>(r);
        const double2 rb = *reinterpret_cast<const double2 *>(r + 2);
        if (NC == 9) {
            const double2 rc = *reinterpret_cast<const double2 *>(r + 4);
            coeff<NC>(rb.y, rc.x, rc.y, r[6], wscale, sigma, s);
        } else {
            coeff<NC>(rb.y, 0, 0, 0, wscale, sigma, s);
        }
        const double wx0 = 1.0 - ra.x, wx1 = 1.0 - fabs(ra.x - 1.0);
        const double wy0 = 1.0 - ra.y, wy1 = 1.0 - fabs(ra.y - 1.0);
        const double wz0 = 1.0 - rb.x, wz1 = 1.0 - fabs(rb.x - 1.0);
        const double xy00 = wx0 * wy0, xy01 = wx0 * wy1, xy10 = wx1 * wy0, xy11 = wx1 * wy1;
        w8[0] = xy00 * wz0;
        w8[1] = xy00 * wz1;
        w8[2] = xy01 * wz0;
        w8[3] = xy01 * wz1;
        w8[4] = xy10 * wz0;
        w8[5] = xy10 * wz1;
        w8[6] = xy11 * wz0;
        w8[7] = xy11 * wz1;
    };
    auto prep_store = [&](double *Pb, const double s[NC], const double w8[8]) {
        double *sh_w = Pb, *sh_s = Pb + 8 * WS;
#pragma unroll
        for (int c = 0; c < NC; ++c)
            sh_s[lane * L::SS + c] = s[c];
#pragma unroll
        for (int a = 0; a < 8; ++a)
            sh_w[a * WS + lane] = w8[a];
    };
    if (C0.u >= 0) {
        double s[NC], w8[8];
        prep_regs(R + 8 * lane, s, w8);
        prep_store(P, s, w8);
        __syncwarp();
    }

    uint32_t c = 0;  // chunk counter: R/P buffer (c & 1), mbarrier parity (c >> 1) & 1
    while (C0.u >= 0) {
        const int buf = c & 1;
        // (1) records of C2 -> R[buf] (consumed by the prep of C0 last iteration)
        if (lane == 0 && C2.u >= 0)
            tma_load(R + buf * CH * 8, rec + 8 * (int64_t)C2.base, C2.cnt * 64, &bar[buf]);
        // (2) records of C1 have arrived?
        double s1[NC], w1[8];
        const bool have1 = C1.u >= 0;
        if (have1) {
            mbar_wait(&bar[buf ^ 1], ((c + 1) >> 1) & 1);
            prep_regs(R + (buf ^ 1) * CH * 8 + 8 * lane, s1, w1);  // FP64 work overlaps the DMMAs below
        }
        // (3) DMMA batches of C0, interleaved with the pending deposit REDs
        const double *Pb = P + buf * L::PSZ;
        const double *wrow = Pb + (lane >> 2) * WS + (lane & 3);
        const double *srow = Pb + 8 * WS + (lane & 3) * L::SS;
        const double *stage = P + (buf ^ 1) * L::PSZ;  // previous bin's staged tile (if pend)
        auto batch = [&](int kb) {
            const double w = wrow[kb];
            const double *sp = srow + kb * L::SS;
            if (NC == 9) {
#pragma unroll
                for (int cc = 0; cc < 8; cc += 2) {
                    const double2 sv = *reinterpret_cast<const double2 *>(sp + cc);
                    dmma(acc[cc][0], acc[cc][1], sv.x * w, w);
                    dmma(acc[cc + 1][0], acc[cc + 1][1], sv.y * w, w);
                }
                dmma(acc[NC - 1][0], acc[NC - 1][1], sp[8] * w, w);
            } else {
                dmma(acc[0][0], acc[0][1], sp[0] * w, w);
            }
        };
        auto dep = [&](int i) {
            const double v = stage[i * 32 + lane];
            const int t = s_tab[i * 32 + lane];
            double *row = shfl_ptr(myrow, t & 7);
            if (pend && v != 0.0)
                red_add(row + (t >> 3), v);
        };
        if (C0.cnt == CH) {
#pragma unroll
            for (int kb = 0; kb < CH; kb += 4) {
                batch(kb);
#pragma unroll
                for (int i = (kb / 4) * L::NDEP / 8; i < (kb / 4 + 1) * L::NDEP / 8; ++i)
                    dep(i);
            }
        } else {
            for (int kb = 0; kb < C0.cnt; kb += 4)
                batch(kb);
#pragma unroll
            for (int i = 0; i < L::NDEP; ++i)
                dep(i);
        }
        pend = false;
        __syncwarp();  // all lanes done with the stage (P[buf^1]) and with P[buf]
        // (4) prep of C1 -> P[buf^1]
        if (have1)
            prep_store(P + (buf ^ 1) * L::PSZ, s1, w1);
        // (5) end of C0's bin: stage D into P[buf], row pointers; REDs go out during C1
        if (C0.base + CH >= C0.end) {
            double *st = P + buf * L::PSZ;
#pragma unroll
            for (int cc = 0; cc < NC; ++cc) {
                st[(lane >> 2) * 8 * NC + (2 * (lane & 3)) * NC + cc] = acc[cc][0];
                st[(lane >> 2) * 8 * NC + (2 * (lane & 3) + 1) * NC + cc] = acc[cc][1];
                acc[cc][0] = acc[cc][1] = 0.0;
            }
            const int bin = C0.u * U + C0.i;
            const int bx = bin / plane, rem = bin - bx * plane;
            const int by = rem / g.n2, bz = rem - by * g.n2;
            const int a8 = lane & 7;
            myrow = row_ptr(g, g.x_begin + bx + (a8 >> 2), wrapi(by + ((a8 >> 1) & 1), g.n1),
                            wrapi(bz + (a8 & 1), g.n2), out, ghost, RL);
            pend = true;
        }
        __syncwarp();
        C0 = C1;
        C1 = C2;
        C2 = next_chunk(C2);
        ++c;
        // the stage written above sits in P[buf]; the next iteration's stage pointer is
        // P[(c & 1) ^ 1] = P[buf]  (consistent)
    }
    // drain: REDs of the last staged bin
    if (pend) {
        const double *stage = P + ((c & 1) ^ 1) * L::PSZ;
#pragma unroll
        for (int i = 0; i < L::NDEP; ++i) {
            const double v = stage[i * 32 + lane];
            const int t = s_tab[i * 32 + lane];
            double *row = shfl_ptr(myrow, t & 7);
            if (v != 0.0)
                red_add(row + (t >> 3), v);
        }
    }
}

template <int NC>
cudaError_t launch_o1p(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    using L = P1<NC>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_asm_o1p<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L::SMEM);
        if (e)
            return e;
        attr = true;
    }
    int dev = 0, sms = 148, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_asm_o1p<NC>);
    int per_sm = smem_sm / (int)(L::SMEM + 1024);
    if (fa.numRegs > 0)
        per_sm = min(per_sm, 65536 / (fa.numRegs * W1 * 32));
    per_sm = max(1, min(per_sm, 16));
    const int64_t nunits = (a.nbins + U - 1) / U;
    int64_t grid = (int64_t)sms * per_sm;
    if (grid * W1 > nunits)
        grid = (nunits + W1 - 1) / W1;
    k_asm_o1p<NC><<<(unsigned)grid, W1 * 32, L::SMEM, s>>>(geo, a.rec, a.seg_begin, (int)a.nbins, a.wscale, a.sigma,
                                                          a.out, a.ghost);
    count_launch();
    return cudaGetLastError();
}

cudaError_t assemble_o1p_enqueue(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    if (a.nbins == 0)
        return cudaSuccess;
    return a.ncomp == 9 ? launch_o1p<9>(geo, a, s) : launch_o1p<1>(geo, a, s);
}

}  // namespace mm
