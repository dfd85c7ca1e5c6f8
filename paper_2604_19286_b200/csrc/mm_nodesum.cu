// Two-phase deposit, phase 2: node rows summed from the bins' pair-product blocks.
//
// Phase 1 (the TF32 assembly kernel with a block buffer) stores each bin's finished block
//
//   D_j[ux uy][uz c] = sum_{p in bin j} X_p[ux uy] Z_p[uz c]      (pair-product plan)
//
// with plain coalesced stores instead of adding its 27 x 27 x C node-pair entries into the
// output with global atomics.  This kernel owns the output: one warp per node row g computes
//
//   M[g][d][c] = sum over the bins j whose support window holds g and g + d of
//                D_j[P(a_x, b_x) NU + P(a_y, b_y)][P(a_z, b_z) C + c],   a = g - j, b = a + d,
//
// (eq_mass_matrix, regrouped by support window as in Algorithm 1,
// PAPER.md:386-416, and eq_D_batches, which holds in any grouping), and writes the row once:
// no zero-fill pass and no global atomics (the order-2 RED kernels issue 27 x 27 x 9 of them per
// bin, bound by the L2 atomic rate).  P(a, b) is the per-axis pair index: a + b for CIC, the
// unordered pair index a + b + (a && b) for TSC.  Phase 1 writes a zero block for an empty bin,
// so the bins around a node follow from its coordinates alone.  Slab grids: owned rows, then the ghost planes in row_ptr's
// order, from the local bins only.
#include "mm_internal.cuh"

namespace mm {

namespace {

template <int ORDER, int C>
struct NS {
    static constexpr int L = ORDER + 1;          // window nodes per axis
    static constexpr int L3 = L * L * L;
    static constexpr int NE = L3 * C;            // entries (b, c) of one window node a
    static constexpr int NU = ORDER == 1 ? 3 : 6;
    static constexpr int NZ = NU * C;
    static constexpr int BLK = NU * NU * NZ;     // block elements per bin
    static constexpr int W = 2 * ORDER + 1;
    static constexpr int RL = W * W * W * C;     // node row length
    static constexpr int WARPS = 8;
    static constexpr int TAB_BYTES = (L3 * NE * 4 + 15) / 16 * 16;
    static_assert(BLK < 65536 && RL < 65536, "16-bit table fields");
};

template <typename T, int ORDER, int C>
__global__ void __launch_bounds__(256) k_nodesum(Geo g, const T *__restrict__ D, int64_t nown, int64_t nrows,
                                                 T *__restrict__ out,
                                                 T *__restrict__ ghost, int accumulate)
{
    using N = NS<ORDER, C>;
    constexpr int NI = (N::NE + 31) / 32;             // entries per lane and bin
    constexpr int G = NI >= 8 ? 4 : (NI >= 2 ? 8 : 16);  // bins whose loads are in flight together
    constexpr int MAXL = N::L3 + N::L * N::L;         // + the periodic duplicates of one a_x
    extern __shared__ __align__(16) unsigned char ns_smem[];
    uint32_t *tab = reinterpret_cast<uint32_t *>(ns_smem);  // [a][e]: block offset | row offset << 16
    T *accs = reinterpret_cast<T *>(ns_smem + N::TAB_BYTES);
    int2 *lists = reinterpret_cast<int2 *>(ns_smem + N::TAB_BYTES + N::WARPS * N::RL * sizeof(T));
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T *acc = accs + warp * N::RL;
    int2 *list = lists + warp * MAXL;  // non-empty bins around the node: (window node a, bin j)

    for (int i = threadIdx.x; i < N::L3 * N::NE; i += blockDim.x) {
        const int a = i / N::NE, e = i - a * N::NE, b = e / C, c = e - b * C;
        const int ax = a / (N::L * N::L), ay = (a / N::L) % N::L, az = a % N::L;
        const int bx = b / (N::L * N::L), by = (b / N::L) % N::L, bz = b % N::L;
        auto P = [](int u, int v) { return ORDER == 1 ? u + v : u + v + (u && v); };
        const int doff = (P(ax, bx) * N::NU + P(ay, by)) * N::NZ + P(az, bz) * C + c;
        const int slot = ((bx - ax + ORDER) * N::W + (by - ay + ORDER)) * N::W + (bz - az + ORDER);
        tab[i] = (uint32_t)doff | ((uint32_t)(slot * C + c) << 16);
    }
    __syncthreads();

    const int plane = g.n1 * g.n2;
    for (int64_t r = (int64_t)blockIdx.x * N::WARPS + warp; r < nrows; r += (int64_t)gridDim.x * N::WARPS) {
        int X, rem;
        T *dst;
        if (r < nown) {
            const int xl = (int)(r / plane);
            rem = (int)(r - (int64_t)xl * plane);
            X = g.x_begin + xl;
            dst = out + r * N::RL;
        } else {
            const int64_t gr = r - nown;
            const int p = (int)(gr / plane);
            rem = (int)(gr - (int64_t)p * plane);
            X = ORDER == 1 ? g.x_end : (p == 0 ? g.x_begin - 1 : g.x_end + p - 1);
            dst = ghost + gr * N::RL;
        }
        const int Y = rem / g.n2, Z = rem - (rem / g.n2) * g.n2;
        // ---- the bins around the node, lane-parallel: lane = window node a, three candidate x
        //      bins (the unwrapped periodic axis has two bins for one window).  No memory access:
        //      phase 1 wrote a zero block for every empty bin.
        int n = 0;
#pragma unroll
        for (int k = -1; k <= 1; ++k) {
            bool ok = false;
            int j = 0;
            if (lane < N::L3 && (k == 0 || g.periodic_x)) {
                const int ax = lane / (N::L * N::L), ay = (lane / N::L) % N::L, az = lane % N::L;
                const int bx = X - g.x_begin + (ORDER - 1) - ax + k * g.n0;
                int by = Y - ay, bz = Z - az;
                by += by < 0 ? g.n1 : 0;
                bz += bz < 0 ? g.n2 : 0;
                ok = bx >= 0 && bx < g.nbx;
                j = (bx * g.n1 + by) * g.n2 + bz;
            }
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            if (ok)
                list[n + __popc(m & ((1u << lane) - 1))] = make_int2(lane, j);
            n += __popc(m);
        }
        for (int e = lane; e < N::RL; e += 32)
            acc[e] = accumulate ? dst[e] : T(0);
        __syncwarp();
        // ---- G bins at a time: all their loads first, then the additions bin by bin
        for (int i0 = 0; i0 < n; i0 += G) {
            T v[G][NI];
#pragma unroll
            for (int q = 0; q < G; ++q) {
                if (i0 + q < n) {
                    const int2 t2 = list[i0 + q];
                    const T *Dj = D + (int64_t)t2.y * N::BLK;
                    const uint32_t *ta = tab + t2.x * N::NE;
#pragma unroll
                    for (int ii = 0; ii < NI; ++ii) {
                        const int e = 32 * ii + lane;
                        v[q][ii] = (N::NE % 32 == 0 || e < N::NE) ? __ldg(Dj + (ta[e] & 0xffffu)) : T(0);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < G; ++q) {
                if (i0 + q < n) {
                    const uint32_t *ta = tab + list[i0 + q].x * N::NE;
#pragma unroll
                    for (int ii = 0; ii < NI; ++ii) {
                        const int e = 32 * ii + lane;
                        if (N::NE % 32 == 0 || e < N::NE)
                            acc[ta[e] >> 16] += v[q][ii];
                    }
                    __syncwarp();  // the next bin may add into the same entries
                }
            }
        }
        for (int e = lane; e < N::RL; e += 32)
            dst[e] = acc[e];
        __syncwarp();
    }
}

template <typename T, int ORDER, int C>
cudaError_t launch_ns(const Geo &g, const void *D, void *out, void *ghost, int accumulate, cudaStream_t s)
{
    using N = NS<ORDER, C>;
    const size_t smem = N::TAB_BYTES + (size_t)N::WARPS * N::RL * sizeof(T) +
                        (size_t)N::WARPS * (N::L3 + N::L * N::L) * sizeof(int2);
    auto kern = k_nodesum<T, ORDER, C>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e)
        return e;
    const int64_t plane = (int64_t)g.n1 * g.n2;
    const int64_t nown = (int64_t)(g.x_end - g.x_begin) * plane;
    const int64_t nrows = nown + (g.periodic_x ? 0 : (ORDER == 1 ? 1 : 3) * plane);
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * N::WARPS, smem);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (nrows + N::WARPS - 1) / N::WARPS;
    const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    const unsigned grid = (unsigned)(want < cap ? (want < 1 ? 1 : want) : cap);
    kern<<<grid, 32 * N::WARPS, smem, s>>>(g, static_cast<const T *>(D), nown, nrows, static_cast<T *>(out),
                                           static_cast<T *>(ghost), accumulate);
    count_launch();
    return cudaGetLastError();
}

}  // namespace

int64_t block_elems(int order, int ncomp)
{
    const int nu = order == 1 ? 3 : 6;
    return (int64_t)nu * nu * nu * ncomp;
}

cudaError_t nodesum_enqueue(const Geo &g, int ncomp, int elem_bytes, const void *D, void *out, void *ghost,
                            int accumulate, cudaStream_t s)
{
    if (elem_bytes == 4) {
        if (g.order == 1)
            return ncomp == 9 ? launch_ns<float, 1, 9>(g, D, out, ghost, accumulate, s)
                              : launch_ns<float, 1, 1>(g, D, out, ghost, accumulate, s);
        return ncomp == 9 ? launch_ns<float, 2, 9>(g, D, out, ghost, accumulate, s)
                          : launch_ns<float, 2, 1>(g, D, out, ghost, accumulate, s);
    }
    if (g.order == 1)
        return ncomp == 9 ? launch_ns<double, 1, 9>(g, D, out, ghost, accumulate, s)
                          : launch_ns<double, 1, 1>(g, D, out, ghost, accumulate, s);
    return ncomp == 9 ? launch_ns<double, 2, 9>(g, D, out, ghost, accumulate, s)
                      : launch_ns<double, 2, 1>(g, D, out, ghost, accumulate, s);
}

}  // namespace mm
