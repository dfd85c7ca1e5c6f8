// TF32 / 3xTF32 variant of the assembly on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM), "reported separately" from the
// FP64 DMMA path (north_star; PAPER.md:186 reduced-precision inputs with wider
// accumulation, PAPER.md:431 TF32 inputs / FP32 accumulation).
//
// Mapping (one CTA = one support-window bin at a time, Algorithm 1):
//   rows    m = c*NN + a   (component c, support node a)  -> M = 128 per MMA (HALVES of them)
//   columns n = b          (support node b, padded to NP) -> N = NP (8 or 32)
//   K       8 particles per tcgen05.mma (32 B of TF32)
//   A[m][k] = tf32(s_c(p_k) W_a(p_k)),  B[n][k] = tf32(W_b(p_k))      (eq_AB_batch)
//   D[m][n] += A B^T in TMEM (FP32)                                    (eq_mma_accumulate)
// 3xTF32: x = hi + lo with hi = rna(x), lo = rna(x - hi); D += Ah Bh + Ah Bl + Al Bh.
// Operands are built by the CTA's threads in shared memory in the UMMA K-major
// no-swizzle canonical layout (8-row x 16-B core matrices; LBO = 128 B between the two
// K halves, SBO = 256 B between 8-row groups) and consumed by one elected thread's MMA.
// The epilogue reads TMEM with tcgen05.ld, stages the block in shared memory and
// flushes FP32 REDs in global address order (output FP32, R17).
#include "mm_internal.cuh"

namespace mm {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint32_t tf32_rna(float x)
{
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ void red_add_f32(float *p, float v)
{
    asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}

__device__ __forceinline__ int wrapi(int i, int n)
{
    return i < 0 ? i + n : (i >= n ? i - n : i);
}

__device__ __forceinline__ float *row_ptr_f(const Geo &g, int X, int Y, int Z, float *out, float *ghost, int rowlen)
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

// ---- UMMA descriptors --------------------------------------------------------
// Shared-memory matrix descriptor, K-major, no swizzle (layout type 0), version 1.
__device__ __forceinline__ uint64_t umma_desc(const void *base, uint32_t lbo, uint32_t sbo)
{
    const uint64_t a = smem_u32(base);
    return ((a >> 4) & 0x3FFFull) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// Instruction descriptor: D = F32, A = B = TF32, both K-major, M = 128, N.
__host__ __device__ constexpr uint32_t idesc_tf32(int N)
{
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, int acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(acc)
        : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t *bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
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

__device__ __forceinline__ void tc_fence_before()
{
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after()
{
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 32 lanes x 8 consecutive 32-bit TMEM columns -> registers (one row per thread).
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float v[8])
{
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 8; ++i)
        v[i] = __uint_as_float(r[i]);
}

// ---- per-particle coefficients / weights (same expressions as the FP64 path) ---
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

template <int ORDER>
__device__ __forceinline__ void axis_weights(double xi, double w[3])
{
    if (ORDER == 1) {
        w[0] = 1.0 - xi;
        w[1] = 1.0 - fabs(xi - 1.0);
        w[2] = 0.0;
    } else {
        double b = xi >= 0.5 ? 0.0 : -1.0;
        double t0 = fabs(xi - b), t1 = xi - (b + 1.0), t2 = fabs(xi - (b + 2.0));
        w[0] = 0.5 * (1.5 - t0) * (1.5 - t0);
        w[1] = 0.75 - t1 * t1;
        w[2] = 0.5 * (1.5 - t2) * (1.5 - t2);
    }
}

template <int ORDER, int NC, bool X3>
struct T32 {
    static constexpr int N1 = ORDER + 1;
    static constexpr int NN = N1 * N1 * N1;          // support nodes: 8 | 27
    static constexpr int NP = ORDER == 1 ? 8 : 32;   // MMA N (nodes padded)
    static constexpr int ROWS = NC * NN;             // 72 | 243 | 8 | 27
    static constexpr int HALVES = (ROWS + 127) / 128;
    static constexpr int CH = 32;                    // particles per chunk = 4 K-steps
    static constexpr int KS = CH / 8;
    static constexpr int L = 2 * ORDER + 1;
    static constexpr int S = L * L * L;
    static constexpr int THREADS = 128;              // one warpgroup: warp w reads TMEM lanes 32w..32w+31
    static constexpr int TMEM_COLS = HALVES * NP <= 32 ? 32 : 64;
    static constexpr int PARTS = X3 ? 2 : 1;         // hi (+ lo)
    // shared memory (bytes)
    static constexpr int A_BYTES = PARTS * KS * HALVES * 128 * 32;
    static constexpr int B_BYTES = PARTS * KS * NP * 32;
    static constexpr int PS_BYTES = CH * NC * 8;
    static constexpr int PA_BYTES = CH * 9 * 8;
    static constexpr int PW_BYTES = CH * NN * 8;
    static constexpr int STAGE_BYTES = NN * NN * NC * 4;
    static constexpr int OFF_A = 0;
    static constexpr int OFF_B = OFF_A + A_BYTES;
    static constexpr int OFF_PS = OFF_B + B_BYTES;
    static constexpr int OFF_PA = OFF_PS + PS_BYTES;
    static constexpr int OFF_PW = OFF_PA + PA_BYTES;
    static constexpr int OFF_ST = OFF_PW + PW_BYTES;
    static constexpr int OFF_ROWP = (OFF_ST + STAGE_BYTES + 15) / 16 * 16;
    static constexpr int OFF_SLOT = OFF_ROWP + 32 * 8;
    static constexpr int OFF_BAR = (OFF_SLOT + NN * NN * 2 + 15) / 16 * 16;
    static constexpr int SMEM = OFF_BAR + 32;
};

// byte offset of element (row, k) (k < 8) inside one 128-row (or NP-row) K-major sub-tile
__device__ __forceinline__ uint32_t kmajor_off(int row, int k)
{
    return (uint32_t)((row >> 3) * 256 + (k >> 2) * 128 + (row & 7) * 16 + (k & 3) * 4);
}

template <int ORDER, int NC, bool X3>
__global__ void __launch_bounds__(128) k_asm_tf32(Geo g, const double *__restrict__ rec,
                                                  const int32_t *__restrict__ seg_begin, int64_t nbins, double wscale,
                                                  double sigma, float *__restrict__ out, float *__restrict__ ghost)
{
    using T = T32<ORDER, NC, X3>;
    extern __shared__ __align__(1024) unsigned char smem[];
    unsigned char *sA = smem + T::OFF_A;  // [PARTS][KS][HALVES][128 rows x 32 B]
    unsigned char *sB = smem + T::OFF_B;  // [PARTS][KS][NP rows x 32 B]
    double *ps = reinterpret_cast<double *>(smem + T::OFF_PS);  // [CH][NC]
    double *pa = reinterpret_cast<double *>(smem + T::OFF_PA);  // [CH][9]
    double *pw = reinterpret_cast<double *>(smem + T::OFF_PW);  // [CH][NN]
    float *stage = reinterpret_cast<float *>(smem + T::OFF_ST); // [NN][NN][NC]
    float **rowp = reinterpret_cast<float **>(smem + T::OFF_ROWP);
    int16_t *s_slot = reinterpret_cast<int16_t *>(smem + T::OFF_SLOT);  // [NN][NN]
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + T::OFF_BAR);    // [0] MMA done
    uint32_t *s_taddr = reinterpret_cast<uint32_t *>(smem + T::OFF_BAR + 8);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int plane = g.n1 * g.n2;
    constexpr int RL = T::S * NC;
    constexpr uint32_t IDESC = idesc_tf32(T::NP);

    for (int e = tid; e < T::NN * T::NN; e += T::THREADS) {
        const int a = e / T::NN, b = e - T::NN * a;
        const int ax = a / (T::N1 * T::N1), ay = (a / T::N1) % T::N1, az = a % T::N1;
        const int bx = b / (T::N1 * T::N1), by = (b / T::N1) % T::N1, bz = b % T::N1;
        s_slot[e] = (int16_t)(((bx - ax + ORDER) * T::L + (by - ay + ORDER)) * T::L + (bz - az + ORDER));
    }
    // zero the operand buffers once: padding rows (m >= ROWS, n >= NN) stay zero
    for (int e = tid; e < (T::A_BYTES + T::B_BYTES) / 16; e += T::THREADS)
        reinterpret_cast<uint4 *>(smem)[e] = make_uint4(0, 0, 0, 0);
    if (tid == 0)
        mbar_init(&bar[0], 1);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_taddr)),
                     "n"(T::TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *s_taddr;
    uint32_t mma_phase = 0;

    for (int64_t bin = blockIdx.x; bin < nbins; bin += gridDim.x) {
        const int b0 = seg_begin[bin], b1 = seg_begin[bin + 1];
        if (b0 == b1)
            continue;
        int ks_total = 0;
        for (int base = b0; base < b1; base += T::CH) {
            const int m = min(T::CH, b1 - base);
            // ---- prep: one thread per particle (s in FP64, per-axis weights)
            if (tid < m) {
                const double *r = rec + 8 * (int64_t)(base + tid);
                const double2 ra = *reinterpret_cast<const double2 *>(r);
                const double2 rb = *reinterpret_cast<const double2 *>(r + 2);
                double s[NC];
                if (NC == 9) {
                    const double2 rc = *reinterpret_cast<const double2 *>(r + 4);
                    coeff<NC>(rb.y, rc.x, rc.y, r[6], wscale, sigma, s);
                } else {
                    coeff<NC>(rb.y, 0, 0, 0, wscale, sigma, s);
                }
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    ps[tid * NC + c] = s[c];
                double w[3];
                axis_weights<ORDER>(ra.x, w);
                pa[tid * 9 + 0] = w[0]; pa[tid * 9 + 1] = w[1]; pa[tid * 9 + 2] = w[2];
                axis_weights<ORDER>(ra.y, w);
                pa[tid * 9 + 3] = w[0]; pa[tid * 9 + 4] = w[1]; pa[tid * 9 + 5] = w[2];
                axis_weights<ORDER>(rb.x, w);
                pa[tid * 9 + 6] = w[0]; pa[tid * 9 + 7] = w[1]; pa[tid * 9 + 8] = w[2];
            } else if (tid < T::CH) {
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    ps[tid * NC + c] = 0.0;  // tail of the last K-step: s = 0 (and W = 0 below)
            }
            __syncthreads();
            for (int e = tid; e < T::CH * T::NN; e += T::THREADS) {
                const int p = e / T::NN, a = e - p * T::NN;
                double w = 0.0;
                if (p < m) {
                    const double *wa = pa + p * 9;
                    w = (wa[a / (T::N1 * T::N1)] * wa[3 + (a / T::N1) % T::N1]) * wa[6 + a % T::N1];
                }
                pw[p * T::NN + a] = w;
            }
            // the previous chunk's MMAs must be done before the operand tiles are rebuilt
            if (ks_total > 0) {
                mbar_wait(&bar[0], mma_phase);
                mma_phase ^= 1u;
            }
            __syncthreads();
            // ---- operands: A rows m = c*NN + a, B rows n = b; TF32 (hi, lo)
            for (int e = tid; e < T::ROWS * (T::CH / 4); e += T::THREADS) {
                const int row = e / (T::CH / 4), k4 = e - row * (T::CH / 4);  // 4 particles per 16 B
                const int c = row / T::NN, a = row - c * T::NN;
                const int half = row >> 7, rr = row & 127;
                uint32_t hi[4], lo[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int p = 4 * k4 + j;
                    const float x = (float)(ps[p * NC + c] * pw[p * T::NN + a]);
                    hi[j] = tf32_rna(x);
                    lo[j] = tf32_rna(x - __uint_as_float(hi[j]));
                }
                const int ks = k4 >> 1, kk = (k4 & 1) * 4;
                unsigned char *dst = sA + (ks * T::HALVES + half) * 4096 + kmajor_off(rr, kk);
                *reinterpret_cast<uint4 *>(dst) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                if (X3)
                    *reinterpret_cast<uint4 *>(dst + T::KS * T::HALVES * 4096) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            }
            for (int e = tid; e < T::NN * (T::CH / 4); e += T::THREADS) {
                const int n = e / (T::CH / 4), k4 = e - n * (T::CH / 4);
                uint32_t hi[4], lo[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float x = (float)pw[(4 * k4 + j) * T::NN + n];
                    hi[j] = tf32_rna(x);
                    lo[j] = tf32_rna(x - __uint_as_float(hi[j]));
                }
                const int ks = k4 >> 1, kk = (k4 & 1) * 4;
                unsigned char *dst = sB + ks * (T::NP * 32) + kmajor_off(n, kk);
                *reinterpret_cast<uint4 *>(dst) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                if (X3)
                    *reinterpret_cast<uint4 *>(dst + T::KS * T::NP * 32) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            // ---- one thread issues the MMAs of the chunk's K-steps
            if (tid == 0) {
                tc_fence_after();
                const int nks = (m + 7) / 8;
                for (int ks = 0; ks < nks; ++ks) {
#pragma unroll
                    for (int h = 0; h < T::HALVES; ++h) {
                        const uint32_t d = tmem + h * T::NP;
                        const unsigned char *Ah = sA + (ks * T::HALVES + h) * 4096;
                        const unsigned char *Bh = sB + ks * (T::NP * 32);
                        const int acc0 = (ks_total + ks) > 0 ? 1 : 0;
                        umma_tf32(d, umma_desc(Ah, 128, 256), umma_desc(Bh, 128, 256), IDESC, acc0);
                        if (X3) {
                            const unsigned char *Al = Ah + T::KS * T::HALVES * 4096;
                            const unsigned char *Bl = Bh + T::KS * T::NP * 32;
                            umma_tf32(d, umma_desc(Ah, 128, 256), umma_desc(Bl, 128, 256), IDESC, 1);
                            umma_tf32(d, umma_desc(Al, 128, 256), umma_desc(Bh, 128, 256), IDESC, 1);
                        }
                    }
                }
                umma_commit(&bar[0]);
            }
            ks_total += (m + 7) / 8;
            __syncthreads();
        }
        // ---- epilogue: wait for the accumulators, TMEM -> registers -> stage[a][b][c]
        mbar_wait(&bar[0], mma_phase);
        mma_phase ^= 1u;
        tc_fence_after();
        const int bx = (int)(bin / plane), rem = (int)(bin - (int64_t)bx * plane);
        const int by = rem / g.n2, bz = rem - by * g.n2;
        if (tid < T::NN) {
            const int a = tid;
            const int ax = a / (T::N1 * T::N1), ay = (a / T::N1) % T::N1, az = a % T::N1;
            rowp[a] = row_ptr_f(g, g.x_begin + bx - (ORDER - 1) + ax, wrapi(by + ay, g.n1), wrapi(bz + az, g.n2), out,
                                ghost, RL);
        }
        {
            const int quarter = warp & 3;      // TMEM lanes 32*quarter .. +31
            constexpr int NCG = T::THREADS / 128;  // column groups (warps sharing a lane quarter)
            const int cgrp = warp >> 2;
#pragma unroll
            for (int h = 0; h < T::HALVES; ++h) {
                const int row = h * 128 + quarter * 32 + lane;
                for (int c0 = cgrp * 8; c0 < T::NP; c0 += 8 * NCG) {
                    float v[8];
                    tmem_ld8(tmem + ((uint32_t)(quarter * 32) << 16) + h * T::NP + c0, v);
                    if (row < T::ROWS) {
                        const int c = row / T::NN, a = row - c * T::NN;
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const int b = c0 + j;
                            if (b < T::NN)
                                stage[(a * T::NN + b) * NC + c] = v[j];
                        }
                    }
                }
            }
        }
        tc_fence_before();
        __syncthreads();
        // ---- flush in address order: e = (a*NN + b)*NC + c -> row(a) + slot(a,b)*NC + c
        for (int e = tid; e < T::NN * T::NN * NC; e += T::THREADS) {
            const int ab = NC == 1 ? e : e / NC;
            const int c = e - ab * NC;
            const float v = stage[e];
            if (v != 0.0f)
                red_add_f32(rowp[ab / T::NN] + s_slot[ab] * NC + c, v);
        }
        __syncthreads();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(T::TMEM_COLS) : "memory");
}

template <int ORDER, int NC, bool X3>
cudaError_t launch_tf32(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    using T = T32<ORDER, NC, X3>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_asm_tf32<ORDER, NC, X3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             T::SMEM);
        if (e)
            return e;
        attr = true;
    }
    int per_sm = 0, dev = 0, sms = 148, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // resident CTAs per SM from smem / threads / registers (the occupancy API reports 1 for
    // this kernel), then capped by TMEM columns below
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_asm_tf32<ORDER, NC, X3>);
    per_sm = smem_sm / (T::SMEM + 1024);
    per_sm = min(per_sm, 2048 / T::THREADS);
    if (fa.numRegs > 0)
        per_sm = min(per_sm, 65536 / (fa.numRegs * T::THREADS));
    per_sm = min(per_sm, 16);
    if (per_sm < 1)
        per_sm = 1;
    if (per_sm * T::TMEM_COLS > 512)
        per_sm = 512 / T::TMEM_COLS;
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > a.nbins)
        grid = a.nbins;
    k_asm_tf32<ORDER, NC, X3><<<(unsigned)grid, T::THREADS, T::SMEM, s>>>(
        geo, a.rec, a.seg_begin, a.nbins, a.wscale, a.sigma, reinterpret_cast<float *>(a.out),
        reinterpret_cast<float *>(a.ghost));
    count_launch();
    return cudaGetLastError();
}

}  // namespace

cudaError_t assemble_tf32_enqueue(const Geo &geo, const AsmArgs &a, int x3, cudaStream_t s)
{
    if (a.nbins == 0)
        return cudaSuccess;
    if (geo.order == 1) {
        if (a.ncomp == 9)
            return x3 ? launch_tf32<1, 9, true>(geo, a, s) : launch_tf32<1, 9, false>(geo, a, s);
        return x3 ? launch_tf32<1, 1, true>(geo, a, s) : launch_tf32<1, 1, false>(geo, a, s);
    }
    if (a.ncomp == 9)
        return x3 ? launch_tf32<2, 9, true>(geo, a, s) : launch_tf32<2, 9, false>(geo, a, s);
    return x3 ? launch_tf32<2, 1, true>(geo, a, s) : launch_tf32<2, 1, false>(geo, a, s);
}

}  // namespace mm
