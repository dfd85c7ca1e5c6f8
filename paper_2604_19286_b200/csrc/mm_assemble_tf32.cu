// TF32 / 3xTF32 variant of the assembly on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, FP32 accumulators in TMEM), "reported separately" from the
// FP64 DMMA path (north_star; PAPER.md:186 reduced-precision inputs with wider
// accumulation, PAPER.md:431 TF32 inputs / FP32 accumulation).
//
// Operand plan: the pair-product factorisation of the FP64 kernels (mm_assemble_fp64.cu,
// O1T / O2T): per bin (support group, Algorithm 1)
//
//   M^c[a][b] = sum_p X_p[ux uy] Z_p[uz c],  X = q_x q_y (NX = 9 | 36),  Z = q_z s^c (NZ = 3C | 6C)
//
// with q_mu the per-axis pair products of the B-spline weights (u_mu = a_mu + b_mu for CIC,
// the unordered pair index for TSC).  One tcgen05.mma (M = 128, K = 8 particles) covers BPC
// bins at once: bin j owns A rows [MB j, MB j + NZ) (A = Z, MB = 128 / BPC) and B rows
// [NB j, NB j + NX) (B = X), so D[MB j + z][NB j + x] is bin j's block; the off-diagonal
// blocks of D are unused.  The tensor work is tiny next to the HBM traffic, so the wasted
// blocks cost nothing measurable, and the layout puts bin j's rows in TMEM lanes that its
// own warp(s) can read (tcgen05.ld: warp w reads lanes 32 (w % 4) .. +31).
//   order 1:         BPC = 4, MB = 32, NB = 16, N = 64    (warp j = bin j)
//   order 2 scalar:  BPC = 4, MB = 32, NB = 48, N = 192   (6 Z rows per bin: two warps per bin
//                    amortise the per-chunk overhead over twice the rows of the 4-warp layout)
//   order 2 tensor:  BPC = 2, MB = 64, NB = 64, N = 128
// 8 warps per CTA: each bin has 2 (order 1) or 4 (order 2) warps that split its X / Z rows in
// the prep and its entries in the deposit; warps 0-3 read the accumulators (lane quarter = warp).
// Per 32-particle chunk: prep (FP32 from the FP64 record; the support base is decided in FP64
// exactly as in the sort), rounded to TF32 and stored straight into 128-B-swizzled K-major tiles
// (one 128-B row per M / N row; conflict-free for lane = particle) in a double buffer ->
// one thread issues 4 K-steps (x3 for 3xTF32: D += Ah Bh + Ah Bl + Al Bh) and commits to the
// buffer's mbarrier.  Epilogue per group: tcgen05.ld -> staged block -> FP32 REDs in global
// address order (the FP64 kernels' deposit tables).
#include "mm_internal.cuh"

namespace mm {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}

// Round to TF32, nearest with ties away from zero (the rounding of cvt.rna.tf32.f32, DESIGN.md
// R16) on the bit pattern: + half an ulp of the 10-bit mantissa to the magnitude, then truncate.
// Finite inputs only (the operands are products of weights and s).
__device__ __forceinline__ uint32_t tf32_rna(float x)
{
    return (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
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
// Shared-memory matrix descriptor, K-major, 128-B swizzle (layout type 2, version 1): rows of
// 128 B (32 TF32 K-elements), 8-row atoms of 1024 B (SBO), 16-B chunk index XOR (row & 7);
// the K-step start advances by 32 B inside the swizzled row.  Atoms 1024-B aligned.
__device__ __forceinline__ uint64_t umma_desc_sw128(const void *base)
{
    const uint64_t a = smem_u32(base);
    return ((a >> 4) & 0x3FFFull) | ((uint64_t)(16 >> 4) << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
           (2ull << 61);
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



__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float v[16])
{
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                   "=r"(r[15])
                 : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i)
        v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_wait_ld()
{
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}


// s^{ij} = sigma q alpha^{ij} (eq_alpha_matrix) in FP32
template <int NC>
__device__ __forceinline__ void coeff_f(float q, float Bx, float By, float Bz, float wscale, float sigma, float s[NC])
{
    if (NC == 1) {
        s[0] = sigma * q;
    } else {
        const float o0 = wscale * Bx, o1 = wscale * By, o2 = wscale * Bz;
        const float d = fmaf(o0, o0, fmaf(o1, o1, fmaf(o2, o2, 1.0f)));
        // reciprocal + one Newton step (<= 1 ulp; no division subroutine call in the prep)
        float r;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
        r = fmaf(r, fmaf(-d, r, 1.0f), r);
        const float f = (sigma * q) * r;
        const float f0 = f * o0, f1 = f * o1, f2 = f * o2;
        s[0] = fmaf(f0, o0, f);
        s[1] = fmaf(f0, o1, f2);
        s[2] = fmaf(f0, o2, -f1);
        s[3] = fmaf(f1, o0, -f2);
        s[4] = fmaf(f1, o1, f);
        s[5] = fmaf(f1, o2, f0);
        s[6] = fmaf(f2, o0, f1);
        s[7] = fmaf(f2, o1, -f0);
        s[8] = fmaf(f2, o2, f);
    }
}

// Per-axis pair products of the B-spline weights.  order 1 (CIC, w = (1 - xi, xi)):
// q = (w0 w0, w0 w1, w1 w1), index u = a + b.  order 2 (TSC, R3, R4): the
// support base is decided in FP64 (xi >= 1/2: base 0, else -1) exactly as in the sort, then
// u = xi - (b + 1) in [-1/2, 1/2) is rounded to FP32; w = ((1/2 - u)^2 / 2, 3/4 - u^2,
// (1/2 + u)^2 / 2); q = (w0 w0, w0 w1, w0 w2, w1 w1, w1 w2, w2 w2), index P(a, b).
template <int ORDER>
__device__ __forceinline__ void pair_products(double xi, float q[ORDER == 1 ? 3 : 6])
{
    if (ORDER == 1) {
        const float w1 = (float)xi, w0 = 1.0f - w1;  // abs. error <= 2^-25 either way, off the FP64 pipe
        q[0] = w0 * w0;
        q[1] = w0 * w1;
        q[2] = w1 * w1;
    } else {
        // base decided in FP64 as in the sort; the shift by one in FP32 (absolute error <= 2^-25,
        // far below the TF32 / 3xTF32 operand rounding) keeps the subtraction off the FP64 pipe
        const float u = xi >= 0.5 ? (float)xi - 1.0f : (float)xi;
        const float h = 0.5f - u, k = 0.5f + u;
        const float w0 = (0.5f * h) * h, w1 = fmaf(-u, u, 0.75f), w2 = (0.5f * k) * k;
        q[0] = w0 * w0;
        q[1] = w0 * w1;
        q[2] = w0 * w2;
        q[3] = w1 * w1;
        q[4] = w1 * w2;
        q[5] = w2 * w2;
    }
}

template <int ORDER, int NC, bool X3>
struct PP {
    static constexpr int NU = ORDER == 1 ? 3 : 6;      // pair products per axis
    static constexpr int NX = NU * NU;                  // X rows: 9 | 36
    static constexpr int NZ = NU * NC;                  // Z rows: 27 | 3 | 54 | 6
    static constexpr int BPC = (ORDER == 1 || NC == 1) ? 4 : 2;  // bins per CTA group
    static constexpr int THREADS = 256, WPB = 8 / BPC;  // warps per bin
    static constexpr int MB = 128 / BPC;                // A (Z) rows per bin
    static constexpr int NB = ORDER == 1 ? 16 : (NC == 1 ? 48 : 64);  // B (X) rows per bin
    static constexpr int N = BPC * NB;                  // MMA N: 64 | 128
    static_assert(NZ <= MB && NX <= NB, "bin block does not fit");
    static constexpr int CH = 32;                       // particles per chunk (4 K-steps of 8)
    static constexpr int PARTS = X3 ? 2 : 1;
    // operand tiles of a 32-particle chunk, K-major with 128-B swizzle: one 128-B row per M / N
    // row (K = 32 TF32), A = 128 rows (16 KB), B = N rows
    static constexpr int A_BYTES = 128 * 128, B_BYTES = N * 128;
    static constexpr int PART_BYTES = A_BYTES + B_BYTES;
    static constexpr int BUF_BYTES = PARTS * PART_BYTES;
    static constexpr int ROWS = NX + NZ;                // operand rows per bin (X then Z)
    static constexpr int L = 2 * ORDER + 1, S = L * L * L, RL = S * NC;
    static constexpr int NDEP = 64 * NC;                // order-1 deposit entries per bin
    static constexpr int NUNIT = 81;                    // order-2 flush units (a, b_x)
    static constexpr int OFF_OP = 0;
    static constexpr int OFF_STG = OFF_OP + 2 * BUF_BYTES;  // epilogue blocks [BPC][NX][NZ]
    static constexpr int OFF_TAB = OFF_STG + (BPC * NX * NZ * 4 + 15) / 16 * 16;
    static constexpr bool OT = ORDER == 2 && NC == 1;  // order-2 scalar: table deposit (runs of 3 are too short)
    static constexpr int NDEP2 = 736;                   // 27 x 27 entries, padded to 32
    static constexpr int TAB_BYTES = ORDER == 1 ? NDEP * 4 : (OT ? NDEP2 * 4 : NUNIT * 16);
    static constexpr int OFF_ROWP = (OFF_TAB + TAB_BYTES + 15) / 16 * 16;
    static constexpr int OFF_BAR = OFF_ROWP + BPC * 32 * 8;
    static constexpr int SMEM = OFF_BAR + 16 * 8;
    static constexpr int TMEM_COLS = N <= 64 ? 64 : (N <= 128 ? 128 : 256);  // power of two >= N
};

// Prep of one warp's share [R0, R1) of a bin's operand rows (X rows, then Z rows; lane = particle
// k of the chunk, zeros past the bin's end), written straight into the 128-B-swizzled K-major
// tiles as TF32: element (row m, k) at (m >> 3) 1024 + (m & 7) 128 + ((k >> 2) ^ (m & 7)) 16 +
// (k & 3) 4.  For a fixed row the 32 lanes hit 32 distinct banks (no staging round trip).
template <int ORDER, int NC, bool X3, int ROLE>
__device__ __forceinline__ void prep_tile(const double4 &ca, const double4 &cb, bool live, uint32_t opb, int pj,
                                          uint32_t bl, float fws, float fsig)
{
    using T = PP<ORDER, NC, X3>;
    if constexpr (ROLE >= T::WPB) {
        return;
    } else {
    constexpr int R0 = ROLE * T::ROWS / T::WPB, R1 = (ROLE + 1) * T::ROWS / T::WPB;
    static_assert(T::NB % 8 == 0 && T::MB % 8 == 0, "a bin's tile rows start on a swizzle period");
    float qx[T::NU], qy[T::NU], qz[T::NU], sc[NC];
    // a lane past the bin's end prepares zeros: zero inputs give exact +0 products
#pragma unroll
    for (int i = 0; i < T::NU; ++i)
        qx[i] = qy[i] = qz[i] = 0.0f;
#pragma unroll
    for (int c = 0; c < NC; ++c)
        sc[c] = 0.0f;
    if (live) {
        if (R0 < T::NX) {
            pair_products<ORDER>(ca.x, qx);
            pair_products<ORDER>(ca.y, qy);
        }
        if (R1 > T::NX) {
            pair_products<ORDER>(ca.z, qz);
            coeff_f<NC>((float)ca.w, (float)cb.x, (float)cb.y, (float)cb.z, fws, fsig, sc);
        }
    }
    // tile row m = NB pj + r (X) | MB pj + r - NX (Z), m & 7 a compile-time constant.  The
    // per-slot tile bases are 1024-B aligned, so base | bl (bl = the lane's (k >> 2) 16 + (k & 3) 4)
    // XOR (m & 7) 16 is the swizzled lane offset of the row's phase: ONE LOP3 per phase and X | Z
    // block, the row's atom and phase offsets ((m >> 3) 1024 + (m & 7) 128) are store immediates
    const uint32_t bx = (opb + T::A_BYTES + (T::NB / 8 * pj) * 1024) | bl;
    const uint32_t bz = (opb + (T::MB / 8 * pj) * 1024) | bl;
#pragma unroll
    for (int r7 = 0; r7 < 8; ++r7) {
        const uint32_t lx = bx ^ (uint32_t)(r7 << 4), lz = bz ^ (uint32_t)(r7 << 4);
#pragma unroll
        for (int r = R0; r < R1; ++r) {
            const int mr = r < T::NX ? r : r - T::NX;  // row inside the bin's X or Z block
            if ((mr & 7) != r7)
                continue;
            const float v = r < T::NX ? qx[r / T::NU] * qy[r % T::NU] : qz[(r - T::NX) / NC] * sc[(r - T::NX) % NC];
            const uint32_t d = (r < T::NX ? lx : lz) + (uint32_t)((mr >> 3) * 1024 + r7 * 128);
            const uint32_t hi = tf32_rna(v);
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(d), "r"(hi) : "memory");
            if (X3)
                asm volatile("st.shared.b32 [%0], %1;" ::"r"(d + (uint32_t)T::PART_BYTES),
                             "r"(tf32_rna(v - __uint_as_float(hi)))
                             : "memory");
        }
    }
    }
}

template <int ORDER, int NC, bool X3>
__global__ void __launch_bounds__(256, ORDER == 1 ? 3 : 2) k_asm_tf32(Geo g, const double *__restrict__ rec,
                                                  const int32_t *__restrict__ seg_begin, int64_t nbins, int rs,
                                                  double wscale, double sigma, float *__restrict__ out,
                                                  float *__restrict__ ghost, float *__restrict__ dblk)
{
    using T = PP<ORDER, NC, X3>;
    extern __shared__ __align__(1024) unsigned char smem[];
    float *stg = reinterpret_cast<float *>(smem + T::OFF_STG);   // [BPC][NX][NZ] epilogue blocks
    float *epi = stg;  // epi[pj]: slot pj's accumulators [NX][NZ], read by its deposit
    int *tab = reinterpret_cast<int *>(smem + T::OFF_TAB);
    float **rowp = reinterpret_cast<float **>(smem + T::OFF_ROWP);  // [BPC][32]
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + T::OFF_BAR);  // 3 BPC mbarriers
    uint32_t *s_taddr = reinterpret_cast<uint32_t *>(smem + T::OFF_BAR + 15 * 8);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int plane = g.n1 * g.n2;

    // ---- deposit tables (the FP64 kernels' address order)
    if (ORDER == 1) {
        // entry (a, b, c): a (3 bits) | slot*C + c (8 bits) | epilogue index x*NZ + z (11 bits)
        for (int e = tid; e < T::NDEP; e += T::THREADS) {
            const int a = e / (8 * NC), r = e - a * 8 * NC, b = r / NC, c = r - b * NC;
            const int ax = a >> 2, ay = (a >> 1) & 1, az = a & 1, bx = b >> 2, by = (b >> 1) & 1, bz = b & 1;
            const int slot = (bx - ax + 1) * 9 + (by - ay + 1) * 3 + (bz - az + 1);
            const int x = 3 * (ax + bx) + (ay + by), z = NC * (az + bz) + c;
            tab[e] = a | ((slot * NC + c) << 3) | ((x * T::NZ + z) << 11);
        }
    } else if (T::OT) {
        // entry (a, b): a (5 bits, 31 = padding) | slot (7 bits) | epilogue index x*NZ + z (8 bits)
        for (int e = tid; e < T::NDEP2; e += T::THREADS) {
            if (e >= 729) {
                tab[e] = 31;
                continue;
            }
            const int a = e / 27, b = e - 27 * a;
            const int ax = a / 9, ay = (a / 3) % 3, az = a % 3, bx = b / 9, by = (b / 3) % 3, bz = b % 3;
            auto P = [](int i, int j) { return i + j + (i && j); };
            const int slot = (bx - ax + 2) * 25 + (by - ay + 2) * 5 + (bz - az + 2);
            tab[e] = a | (slot << 5) | ((((6 * P(ax, bx) + P(ay, by)) * T::NZ) + P(az, bz)) << 12);
        }
    } else {
        // unit (a, b_x): {a, slot(b - a)*C at b_y = b_z = 0, epilogue offsets NZ X(b_y), a_z}
        int4 *unit = reinterpret_cast<int4 *>(tab);
        for (int u = tid; u < T::NUNIT; u += T::THREADS) {
            const int a = u / 3, bx = u - 3 * a;
            const int ax = a / 9, ay = (a / 3) % 3, az = a % 3;
            const int slot = (bx - ax + 2) * 25 + (0 - ay + 2) * 5 + (0 - az + 2);
            const int px = ax + bx + (ax && bx);
            int mx[3];
            for (int by = 0; by < 3; ++by)
                mx[by] = T::NZ * (6 * px + ay + by + (ay && by));
            unit[u] = make_int4(a, slot * NC, mx[0] | (mx[1] << 16), mx[2] | (az << 16));
        }
    }
    // zero both operand buffers once: padding rows stay zero
    for (int e = tid; e < 2 * T::BUF_BYTES / 16; e += T::THREADS)
        reinterpret_cast<uint4 *>(smem + T::OFF_OP)[e] = make_uint4(0, 0, 0, 0);
    if (tid < 3 * T::BPC)
        mbar_init(&bar[tid], 1);  // [2 pj + buf] operand buffers, [2 BPC + pj] accumulators
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
    const float fws = (float)wscale, fsig = (float)sigma;

    // prep role of this warp: bin pj, an equal share [r0, r1) of its operand rows (X rows, then
    // Z rows).  order 1: bin j = warps j, 4+j; order 2: bin j = warps {2j, 2j+1, 2j+4, 2j+5}, so
    // warps 0-3 can read bin j's TMEM lane quarters (tcgen05.ld: warp w reads quarter w % 4).
    const int pj = T::BPC == 4 ? (warp & 3) : ((warp >> 1) & 1);
    const int role = T::BPC == 4 ? (warp >> 2) : ((warp & 1) + 2 * (warp >> 2));


    // Each bin slot pj (its 2 | 4 warps) runs independently: its own bins (group grp, slot pj),
    // chunk double buffer parity, mbarriers, named barrier (id 1 + pj) and MMA issue into its own
    // D columns [NB pj, NB pj + NB).  The A tile is shared: an MMA of slot pj also reads the other
    // slots' rows (possibly while they are rewritten), which only produce D lanes outside its
    // quarter(s), never read.
    const int pthreads = 32 * T::WPB;
    // lane part of the swizzled tile offset before the row-phase XOR (see prep_tile)
    const uint32_t bl = (uint32_t)(((lane >> 2) << 4) | ((lane & 3) << 2));
    const bool issuer = role == 0 && lane == 0;
    static_assert(T::CH == 32, "4 K-steps per chunk");
    uint64_t *bar_buf = bar + 2 * pj, *bar_acc = bar + 2 * T::BPC + pj;
    constexpr uint32_t IDESC_J = idesc_tf32(T::NB);
    uint32_t cc = 0, bc = 0;  // chunks / non-empty bins of this slot
    const int nbins32 = (int)nbins;  // < 2^31 (mm_sort_by_cell)
    const int ngroups = (nbins32 + T::BPC - 1) / T::BPC;
    auto range = [&](int grp, int &bb, int &nn) {
        const int bin = grp * T::BPC + pj;
        const bool ok = grp < ngroups && bin < nbins32;
        bb = ok ? __ldg(seg_begin + bin) : 0;
        nn = ok ? __ldg(seg_begin + bin + 1) - bb : 0;
    };
    auto load_rec = [&](int base, int n, int c, double4 &ra, double4 &rb) {
        const int p = T::CH * c + lane;
        if (p < n) {
            const double *r = rec + rs * (int64_t)(base + p);
            ra = *reinterpret_cast<const double4 *>(r);
            if (NC == 9)
                rb = *reinterpret_cast<const double4 *>(r + 4);
        }
    };
    int b0, nb, nb0, nnb;
    range(blockIdx.x, b0, nb);
    range((int)(blockIdx.x + gridDim.x), nb0, nnb);
    double4 ra = make_double4(0, 0, 0, 0), rb = ra;
    load_rec(b0, nb, 0, ra, rb);
    for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const int bin = grp * T::BPC + pj;
        const int nch = (nb + T::CH - 1) / T::CH;
        if (nch == 0)  // nothing was prefetched for the successor yet
            load_rec(nb0, nnb, 0, ra, rb);
        for (int c = 0; c < nch; ++c, ++cc) {
            const int buf = cc & 1;
            unsigned char *op = smem + T::OFF_OP + buf * T::BUF_BYTES;
            const double4 ca = ra, cb = rb;
            if (c + 1 < nch)
                load_rec(b0, nb, c + 1, ra, rb);
            else
                load_rec(nb0, nnb, 0, ra, rb);
            if (cc >= 2)  // the MMAs of this slot that last read this buffer are done
                mbar_wait(&bar_buf[buf], ((cc >> 1) - 1) & 1);
            // ---- prep + TF32 tiles of this warp's row share (compile-time row range per role)
            {
                const bool live = T::CH * c + lane < nb;
                switch (role) {
                case 0: prep_tile<ORDER, NC, X3, 0>(ca, cb, live, smem_u32(op), pj, bl, fws, fsig); break;
                case 1: prep_tile<ORDER, NC, X3, 1>(ca, cb, live, smem_u32(op), pj, bl, fws, fsig); break;
                case 2: prep_tile<ORDER, NC, X3, 2>(ca, cb, live, smem_u32(op), pj, bl, fws, fsig); break;
                default: prep_tile<ORDER, NC, X3, 3>(ca, cb, live, smem_u32(op), pj, bl, fws, fsig); break;
                }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("bar.sync %0, %1;" ::"r"(1 + pj), "r"(pthreads) : "memory");
            if (issuer) {
                tc_fence_after();
                const int nks = (min(T::CH, nb - T::CH * c) + 7) / 8;
                // descriptors: the start-address field (bits 0-13, 16-B units) advances by 2 per
                // K-step (+32 B inside the swizzled row) and by PART_BYTES / 16 to the low parts
                const uint64_t dA = umma_desc_sw128(op), dB = umma_desc_sw128(op + T::A_BYTES + T::NB * pj * 128);
                const uint32_t d = tmem + T::NB * pj;
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    if (ks < nks) {
                        umma_tf32(d, dA + 2 * ks, dB + 2 * ks, IDESC_J, (c > 0 || ks > 0) ? 1 : 0);
                        if (X3) {
                            umma_tf32(d, dA + 2 * ks, dB + 2 * ks + (T::PART_BYTES >> 4), IDESC_J, 1);
                            umma_tf32(d, dA + 2 * ks + (T::PART_BYTES >> 4), dB + 2 * ks, IDESC_J, 1);
                        }
                    }
                }
                umma_commit(&bar_buf[buf]);
                if (c == nch - 1)
                    umma_commit(bar_acc);
            }
        }
        const int nbk = nb;
        b0 = nb0;
        nb = nnb;
        range(grp + 2 * (int)gridDim.x, nb0, nnb);
        if (dblk && nch == 0 && bin < nbins32) {  // two-phase: an empty bin's block is zero
            float *dp = dblk + (int64_t)bin * (T::NX * T::NZ);
            for (int e = 32 * role + lane; e < T::NX * T::NZ; e += 32 * T::WPB)
                dp[e] = 0.0f;
        }
        if (nch == 0 || bin >= nbins32)
            continue;
        if (dblk) {
            // two-phase deposit (mm_nodesum.cu): the bin's block D[x][z] straight from TMEM to its
            // slot of the block buffer with coalesced stores (lane = z); no REDs, no staging.  The
            // next bin's first MMA overwrites these columns only after the slot's next chunk
            // barrier, which every reader reaches after its tcgen05.wait::ld.
            mbar_wait(bar_acc, bc & 1);
            ++bc;
            tc_fence_after();
            if (warp < 4) {
                const int z = T::BPC == 4 ? lane : 32 * (warp & 1) + lane;
                float *dp = dblk + (int64_t)bin * (T::NX * T::NZ);
                const uint32_t tl = tmem + ((uint32_t)(32 * warp) << 16) + T::NB * pj;
#pragma unroll
                for (int x0 = 0; x0 < T::NX; x0 += 16) {
                    float v[16];
                    tmem_ld16(tl + x0, v);
                    tmem_wait_ld();
                    if (z < T::NZ) {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (x0 + i < T::NX)
                                dp[(x0 + i) * T::NZ + z] = v[i];
                    }
                }
            }
            tc_fence_before();
            continue;
        }
        // ---- epilogue of this slot's bin: accumulators -> epi[pj][x][z]
        {
            const int bxl = bin / plane, rem = bin - bxl * plane, bx = g.bx0 + bxl;
            const int by = rem / g.n2, bz = rem - by * g.n2;
            if (ORDER == 1) {
                if (role == 0 && lane < 8) {  // node rows a = lane of this bin, read by the deposit
                    const int a8 = lane;
                    rowp[pj * 32 + a8] = row_ptr_f(g, g.x_begin + bx + (a8 >> 2), wrapi(by + ((a8 >> 1) & 1), g.n1),
                                                   wrapi(bz + (a8 & 1), g.n2), out, ghost, T::RL);
                }
            } else if (role == 0 && lane < 27) {
                const int a = lane;
                rowp[pj * 32 + a] = row_ptr_f(g, g.x_begin + bx - 1 + a / 9, wrapi(by + (a / 3) % 3, g.n1),
                                              wrapi(bz + a % 3, g.n2), out, ghost, T::RL);
            }
        }
        mbar_wait(bar_acc, bc & 1);
        ++bc;
        tc_fence_after();
        if (warp < 4) {  // lane quarter = warp: this slot's Z rows
            const int z = T::BPC == 4 ? lane : 32 * (warp & 1) + lane;
            float *ep = epi + pj * T::NX * T::NZ;
            const uint32_t tl = tmem + ((uint32_t)(32 * warp) << 16) + T::NB * pj;
#pragma unroll
            for (int x0 = 0; x0 < T::NX; x0 += 16) {
                float v[16];
                tmem_ld16(tl + x0, v);
                tmem_wait_ld();
                if (z < T::NZ) {
#pragma unroll
                    for (int i = 0; i < 16; ++i)
                        if (x0 + i < T::NX)
                            ep[(x0 + i) * T::NZ + z] = v[i];
                }
            }
        }
        tc_fence_before();
        asm volatile("bar.sync %0, %1;" ::"r"(1 + pj), "r"(pthreads) : "memory");
        // ---- deposit: FP32 REDs in global address order, the bin's entries split over its warps
        if (nbk > 0) {
            const float *ep = epi + pj * T::NX * T::NZ;
            if (ORDER == 1) {
                for (int i = 32 * role; i < T::NDEP; i += 32 * T::WPB) {
                    if (i + lane < T::NDEP) {
                        const int t = tab[i + lane];
                        red_add_f32(rowp[pj * 32 + (t & 7)] + ((t >> 3) & 255), ep[t >> 11]);
                    }
                }
            } else if (T::OT) {
                for (int i = 32 * role; i < T::NDEP2; i += 32 * T::WPB) {
                    const int t = tab[i + lane];
                    const int a = t & 31;
                    if (a < 27)
                        red_add_f32(rowp[pj * 32 + a] + ((t >> 5) & 127), ep[t >> 12]);
                }
            } else if (lane < 3 * NC) {
                const int4 *unit = reinterpret_cast<const int4 *>(tab);
                const int lbz = lane / NC, lc = lane - NC * lbz;
                const int noff0 = NC * lbz + lc;                        // P(0, bz) = bz
                const int noff1 = NC * (lbz + 1 + (lbz > 0)) + lc;      // P(1, bz) = 1, 3, 4
                const int noff2 = NC * (lbz == 0 ? 2 : lbz + 3) + lc;   // P(2, bz) = 2, 4, 5
                for (int u = role; u < T::NUNIT; u += T::WPB) {
                    const int4 t = unit[u];
                    const int az = t.w >> 16;
                    const int no = az == 0 ? noff0 : (az == 1 ? noff1 : noff2);
                    float *p = rowp[pj * 32 + t.x] + t.y + lane;
                    red_add_f32(p, ep[(t.z & 0xffff) + no]);
                    red_add_f32(p + 5 * NC, ep[(t.z >> 16) + no]);
                    red_add_f32(p + 10 * NC, ep[(t.w & 0xffff) + no]);
                }
            }
        }
        // (epi / rowp of this slot are rewritten only after the next bin's chunk barriers)
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(T::TMEM_COLS) : "memory");
}

template <int ORDER, int NC, bool X3>
cudaError_t launch_tf32(const Geo &geo, const AsmArgs &a, cudaStream_t s)
{
    using T = PP<ORDER, NC, X3>;
    // per call: the attribute is per device/context (a process may drive several GPUs)
    cudaError_t e = cudaFuncSetAttribute(k_asm_tf32<ORDER, NC, X3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         T::SMEM);
    if (e)
        return e;
    int dev = 0, sms = 148, smem_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_asm_tf32<ORDER, NC, X3>);
    // resident CTAs per SM from smem / threads / registers, capped by the 512 TMEM columns
    int per_sm = smem_sm / (T::SMEM + 1024);
    per_sm = min(per_sm, 2048 / T::THREADS);
    if (fa.numRegs > 0)
        per_sm = min(per_sm, 65536 / (fa.numRegs * T::THREADS));
    per_sm = min(per_sm, 512 / T::TMEM_COLS);
    if (per_sm < 1)
        per_sm = 1;
    const int64_t ngroups = (a.nbins + T::BPC - 1) / T::BPC;
    int64_t grid = (int64_t)sms * per_sm;
    if (grid > ngroups)
        grid = ngroups;
    k_asm_tf32<ORDER, NC, X3><<<(unsigned)grid, T::THREADS, T::SMEM, s>>>(
        geo, a.rec, a.seg_begin, a.nbins, a.rec_stride, a.wscale, a.sigma, reinterpret_cast<float *>(a.out),
        reinterpret_cast<float *>(a.ghost), reinterpret_cast<float *>(a.dblk));
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
