// Internal declarations of libmm (not part of the ABI).  See include/mm.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/mm.h"

namespace mm {

// Node rows of a handle's output (owned rows + ghost planes): the size of the flag array of
// the first-writer zeroing.
inline int64_t flag_rows(const mm_grid &g, int order)
{
    const bool whole = g.x_begin == 0 && g.x_end == g.n[0];
    const int planes = (g.x_end - g.x_begin) + (whole ? 0 : (order == 1 ? 1 : 3));
    return (int64_t)planes * g.n[1] * g.n[2];
}

// Kernel-side grid/slab geometry.
struct Geo {
    int n0, n1, n2;
    double h0, h1, h2;
    int x_begin, x_end;
    int order;
    int periodic_x;  // whole axis 0 owned -> wrap, else slab with ghost planes
    int nbx;         // bins along axis 0 = x_end - x_begin + order - 1
    double ih0, ih1, ih2;  // 1/h, exact when the spacing is a power of two
    int h_pow2;            // all three spacings powers of two: x/h == x * (1/h) bit for bit
    int bx0;               // assembly launches over a range of bin planes: bin 0 of the launch
                           // is bin plane bx0 (seg_begin is offset by the caller)
};

Geo make_geo(const mm_grid &g, int order);

// Status words in device memory (read back once per sort).
// ST_STICKY: OR of the error bits of every sort since the last check (mm_sort_wait / the
// synchronous sort); words [0, ST_PER_SORT) are cleared at the start of each sort.
enum { ST_ERR = 0, ST_NPAD = 1, ST_NMID = 2, ST_NHUGE = 3, ST_PER_SORT = 4, ST_STICKY = 4, ST_WORDS = 8 };
enum { ERR_DOMAIN = 1, ERR_NONFINITE = 2 };

// Bins larger than these go to the CTA / huge fix-up paths.
constexpr int WARP_BIN_MAX = 1024;
constexpr int CTA_BIN_MAX = 16384;

void count_launch(int n = 1);

// ---- sort (mm_sort.cu) ---------------------------------------------------
struct SortBufs {
    int64_t np, nbins;
    int k_pad;
    const double *pos, *q, *B;
    int f32;             // 1: pos and B point to FP32 arrays (widened exactly on load)
    uint32_t *key;
    int32_t *rank;       // atomic rank, later reused as dest (inverse permutation)
    int32_t *count;      // [nbins]
    int32_t *seg_begin;  // [nbins + 1]
    int32_t *perm;       // [capacity]
    double *rec;         // [capacity][8]
    int32_t *scan_tmp;   // [>= nblocks + 1]
    int32_t *mid_list;   // [nbins]
    int32_t *huge_list;  // [nbins]
    int32_t *status;     // [ST_WORDS]
    int64_t capacity;
    double *rec_tmp = nullptr;  // [capacity][8] scratch: the record-first path (inputs beyond L2),
                                // which leaves rank as the atomic rank (no inverse permutation)
};
int64_t scan_tmp_elems(int64_t nbins);
cudaError_t sort_enqueue(const Geo &geo, const SortBufs &b, cudaStream_t s);
// dest[perm[i]] = i for the padded slots i < *seg_end (perm -1 = pad)
cudaError_t inverse_enqueue(const int32_t *perm, const int32_t *seg_end, int64_t capacity, int32_t *dest,
                            cudaStream_t s);
// incremental re-binning (mm_resort_by_cell): SortBufs of the handle (perm = the NEW permutation
// buffer) plus the previous sort's permutation and scratch
struct IncBufs {
    int32_t *perm_old;        // [capacity] the previous sort's permutation (leavers get marked)
    int32_t *seg_old;         // [nbins + 1] scratch: the previous seg_begin
    int32_t *arr_count;       // [nbins]
    int32_t *arr_begin;       // [nbins + 1]
    int32_t *arr;             // [np] arrivals by bin
};
cudaError_t resort_enqueue(const Geo &geo, const SortBufs &b, const IncBufs &ib, cudaStream_t s);

// ---- assembly (mm_assemble_fp64.cu) ----------------------------------------
struct AsmArgs {
    const double *rec;
    int rec_stride;       // doubles per record: 8 {xi, q, B, 0} | 4 {xi, q} (handle sorted without B)
    const int32_t *seg_begin;
    int64_t nbins;
    int ncomp;            // 1 | 9
    double wscale;        // omega = wscale * B   (= qom*dt/(2c))
    double sigma;
    double *out;          // owned rows (FP64; FP32 for the TF32 paths, reinterpreted)
    double *ghost;        // ghost planes (slab only)
    int *work;            // device work counter, zeroed before the launch
    int32_t *zflags;      // first-writer zeroing (dev::ZeroPlan): row flags, nullptr = output pre-zeroed
    int32_t zepoch;       //   flag value of this launch
    void *dblk = nullptr; // two-phase deposit: per-bin pair-product blocks [nbins][block_elems]
                          //   (the kernel stores them; nodesum_enqueue writes the output), else REDs
};
cudaError_t assemble_fp64_enqueue(const Geo &geo, const AsmArgs &a, cudaStream_t s);
// true when the kernel for (order, ncomp, tf32) zeroes its output rows itself (AsmArgs::zflags)
bool zeroes_inside(int order, int ncomp, int tf32);

// ---- TF32 / 3xTF32 on tcgen05 (mm_assemble_tf32.cu); out/ghost hold FP32 ----------
cudaError_t assemble_tf32_enqueue(const Geo &geo, const AsmArgs &a, int x3, cudaStream_t s);

// ---- two-phase deposit, phase 2 (mm_nodesum.cu) -------------------------------
// elements of one bin's pair-product block: (NU^2) x (NU C), NU = 3 | 6
int64_t block_elems(int order, int ncomp);
// every owned (and, on a slab, ghost) node row = (accumulate ? row : 0) + the sum of the blocks of
// the bins around it; D holds elem_bytes-wide blocks of every bin (zero for an empty bin)
cudaError_t nodesum_enqueue(const Geo &g, int ncomp, int elem_bytes, const void *D, void *out, void *ghost,
                            int accumulate, cudaStream_t s);

// ---- operator apply (mm_apply.cu) -------------------------------------------
cudaError_t apply_enqueue(const Geo &geo, int ncomp, const double *M, const double *E, double *y, int accumulate,
                          cudaStream_t s);

// ---- NEXT-4: moments and field gather (mm_moments.cu) -------------------------
cudaError_t moments_enqueue(const Geo &g, int nq, const double *rec, int rs, const int32_t *perm,
                            const int32_t *seg_begin, int64_t nbins, const double *v, double sigma, double *out,
                            double *ghost, cudaStream_t s);
cudaError_t gather_enqueue(const Geo &g, double *rec, const int32_t *perm, const int32_t *seg_begin, int64_t nbins,
                           const double *F, double *Fp, cudaStream_t s);

// ---- communicator (mm_comm.cu) -----------------------------------------------
mm_status api_fail(mm_status st, const char *fmt, ...);  // sets mm_last_error (mm_api.cu)
const char *nccl_error(int r);
int comm_nranks(const mm_comm *c);
int comm_rank(const mm_comm *c);
cudaError_t ghost_exchange_enqueue(mm_comm *c, int order, int width, int64_t plane_elems, int elem_bytes, void *out,
                                   void *ghost, cudaStream_t s, int *nccl_rc, cudaError_t (*between)(void *),
                                   void *between_ctx);

// ---- halo (mm_halo.cu) -----------------------------------------------------
cudaError_t ghost_add_enqueue(double *out, const double *recv, int64_t n, cudaStream_t s);
int64_t partition_tmp_elems(int64_t np);
// tmp: [partition_tmp_elems(np)] int32; the class ends are left in tmp[3 ntiles .. +2]
cudaError_t partition_enqueue(const Geo &g, int64_t np, const double *pos, const double *q, const double *B,
                              double *pos_o, double *q_o, double *B_o, int32_t *tmp, cudaStream_t s);

}  // namespace mm
