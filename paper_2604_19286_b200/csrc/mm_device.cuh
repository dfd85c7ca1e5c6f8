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
