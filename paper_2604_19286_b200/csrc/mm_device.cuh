// Device helpers shared by the FP64 assembly kernels (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mm_internal.cuh"

namespace mm {
namespace dev {

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
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}

// The same with an L2 evict-first policy: data streamed exactly once (sorted records) should
// not push the output rows that the REDs revisit out of L2.
__device__ __forceinline__ double4 ld256_ef(const double *p)
{
    double4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p));
    return v;
}

// Fire-and-forget FP64 reduction into GLOBAL memory (REDG.E.ADD.F64.RN).  Explicit PTX:
// pointers that travel through shared memory are generic to the compiler, which would
// otherwise emit a generic ATOM with a shared-memory CAS fallback.
__device__ __forceinline__ void red_add(double *p, double v)
{
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}

// The same without a compiler memory clobber: shared-memory loads may be scheduled across it
// (the RED reads only registers; ordering against later global writes and flag releases is
// kept by asm volatile order and the release's own clobber).
__device__ __forceinline__ void red_add_nc(double *p, double v)
{
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v));
}

// Predicated form (one instruction, no branch around it).
__device__ __forceinline__ void red_add_if(double *p, double v, bool ok)
{
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q red.global.add.f64 [%0], %1;\n\t}" ::"l"(p),
                 "d"(v), "r"((int)ok));
}

__device__ __forceinline__ int wrapi(int i, int n)
{
    return i < 0 ? i + n : (i >= n ? i - n : i);
}

// Base address of node row (X unwrapped global, Y/Z wrapped); rowlen = S*C.
__device__ __forceinline__ double *row_ptr(const Geo &g, int X, int Y, int Z, double *out, double *ghost, int rowlen)
{
    if (g.periodic_x) {
        X = X < 0 ? X + g.n0 : (X >= g.n0 ? X - g.n0 : X);
        return out + ((int64_t)(X * g.n1 + Y) * g.n2 + Z) * rowlen;
    }
    int xl = X - g.x_begin;
    if (xl >= 0 && X < g.x_end)
        return out + ((int64_t)(xl * g.n1 + Y) * g.n2 + Z) * rowlen;
    int plane = (g.order == 1) ? 0 : (X < g.x_begin ? 0 : 1 + (X - g.x_end));
    return ghost + ((int64_t)(plane * g.n1 + Y) * g.n2 + Z) * rowlen;
}

// Flag index of a node row (same X convention as row_ptr): owned rows first, then the ghost
// planes in row_ptr's order.
__device__ __forceinline__ int64_t row_id(const Geo &g, int X, int Y, int Z)
{
    if (g.periodic_x) {
        X = X < 0 ? X + g.n0 : (X >= g.n0 ? X - g.n0 : X);
        return ((int64_t)X * g.n1 + Y) * g.n2 + Z;
    }
    const int xl = X - g.x_begin;
    if (xl >= 0 && X < g.x_end)
        return ((int64_t)xl * g.n1 + Y) * g.n2 + Z;
    const int plane = (g.order == 1) ? 0 : (X < g.x_begin ? 0 : 1 + (X - g.x_end));
    return ((int64_t)(g.x_end - g.x_begin + plane) * g.n1 + Y) * g.n2 + Z;
}

// ---- first-writer zeroing (DESIGN.md §7 "Output zeroing inside the assembly") -----------
// Bins are processed in DESCENDING index order through a ticket counter (ticket t = bin
// nbins-1-t), so the first bin to touch a node row is the toucher with the largest index.
// The holder of ticket t zeroes the rows whose first toucher is ticket t + D (and, for t < D,
// those of ticket t itself) as soon as it has the ticket (not when it processes it: a ticket
// held for later must not hold back rows others wait for), and publishes them (flag = epoch,
// release) before its next wait; a bin waits (acquire) for the flags of the rows it deposits
// into.  Every waiter's rows are zeroed by a ticket taken no later than its own, by a running
// warp that releases before it waits: no deadlock, whatever the residency.
struct ZeroPlan {
    int32_t *flags;  // [rows owned + ghost rows]; nullptr: no zeroing in the kernel
    int32_t epoch;   // this launch's flag value (the handle counts launches)
    int lookahead;   // D, in tickets
};

// Row coordinates along one axis whose first toucher (largest covering bin) is bin coordinate
// b; bins b in [0, nb) cover rows b - s + a, a = 0..R (mod n when periodic; then nb = n + s).
// Periodic: a row u < R is first touched by the last bin nb - 1 (through the wrap), any other
// row by bin u + s.  Slab (x, no wrap): row u by bin min(u + s, nb - 1).  Returns the count
// (<= R + 1); u[] holds wrapped (periodic) or local unwrapped (slab) coordinates.
__device__ __forceinline__ int first_rows(int b, int nb, int n, int R, int s, bool periodic, int u[3])
{
    if (b == nb - 1) {
        if (periodic) {
            u[0] = 0;
            u[1] = R == 1 ? n - 1 : 1;
            u[2] = n - 1;
        } else {
            u[0] = nb - 1 - s;
            u[1] = nb - s;
            u[2] = nb + 1 - s;
        }
        return R + 1;
    }
    if (periodic && b - s < R)
        return 0;
    u[0] = b - s;
    return 1;
}

// Rows whose first toucher is bin `bin` (whole-range launch: bin planes 0..nbx-1): the per-axis
// lists.  Returns the number of rows (product of the list lengths).
__device__ __forceinline__ int first_rows3(const Geo &g, int bin, int ux[3], int uy[3], int uz[3], int &nx, int &ny,
                                           int &nz)
{
    const int R = g.order, plane = g.n1 * g.n2;
    const int bxl = bin / plane, rem = bin - bxl * plane, by = rem / g.n2, bz = rem - by * g.n2;
    nx = first_rows(bxl, g.nbx, g.n0, R, R - 1, g.periodic_x != 0, ux);
    ny = first_rows(by, g.n1, g.n1, R, 0, true, uy);
    nz = first_rows(bz, g.n2, g.n2, R, 0, true, uz);
    return nx * ny * nz;
}

// Warp-cooperative zeroing of the rows first touched by `bin`; lane lbase + k (k < count) gets
// the flag index of row k in `rel` for the later release.
__device__ __forceinline__ void zero_first_rows(const Geo &g, int bin, double *out, double *ghost, int rowlen, int lane,
                                                int lbase, int64_t &rel)
{
    int ux[3], uy[3], uz[3], nx, ny, nz;
    const int cnt = first_rows3(g, bin, ux, uy, uz, nx, ny, nz);
    for (int k = 0; k < cnt; ++k) {
        const int ix = k / (ny * nz), r = k - ix * ny * nz, iy = r / nz, iz = r - iy * nz;
        const int X = g.x_begin + (ix == 0 ? ux[0] : (ix == 1 ? ux[1] : ux[2]));
        const int Y = iy == 0 ? uy[0] : (iy == 1 ? uy[1] : uy[2]);
        const int Z = iz == 0 ? uz[0] : (iz == 1 ? uz[1] : uz[2]);
        double *p = row_ptr(g, X, Y, Z, out, ghost, rowlen);
        for (int e = lane; e < rowlen; e += 32)
            p[e] = 0.0;
        if (lane == lbase + k)
            rel = row_id(g, X, Y, Z);
    }
}

__device__ __forceinline__ void flag_release(int32_t *p, int32_t v)
{
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int32_t flag_acquire(const int32_t *p)
{
    int32_t v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void flag_wait(const int32_t *p, int32_t v)
{
    while (flag_acquire(p) != v) {
    }
}

// s^{ij} = sigma q alpha^{ij}, alpha = (delta + omega omega^T + eps omega)/(1+|omega|^2)
// (eq_alpha_matrix, with -C(omega)_{ij} = eps_{ijk} omega_k).  FP64 SIMT work
// shares the FP64 pipe with the DMMAs, so this is written for few instructions: f = sigma q / d
// by a Newton-refined reciprocal, then one FMA per component with f*omega.
__device__ __forceinline__ void coeff9(double q, double Bx, double By, double Bz, double wscale, double sigma,
                                       double s[9])
{
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

__device__ __forceinline__ double2 lds128(const double *p)
{
    return *reinterpret_cast<const double2 *>(p);
}

// Work ticket: atom.inc with limit 2^31-1 (== +1 for any reachable count); ptxas does not
// warp-aggregate inc, so the ticket can be requested a whole bin ahead.
__device__ __forceinline__ int ticket(int *p)
{
    unsigned r;
    asm volatile("atom.global.inc.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(0x7fffffffu) : "memory");
    return (int)r;
}

}  // namespace dev

}  // namespace mm
