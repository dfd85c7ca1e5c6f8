// C ABI of libmm (include/mm.h): argument validation, handle lifetime, stream
// plumbing and error strings.  All arithmetic lives in the kernels of
// mm_sort.cu, mm_assemble_fp64.cu and mm_halo.cu.
#include <atomic>
#include <cmath>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "mm_internal.cuh"

struct mm_sorted {
    mm_grid g;
    int order;
    int k_pad;
    int has_B;
    int valid;
    int device;
    int64_t np, np_padded, nbins;
    int64_t cap_np;   // particle-indexed arrays
    int64_t cap_rec;  // record slots
    uint32_t *key;
    int32_t *rank;
    int32_t *count;
    int32_t *seg_begin;
    int32_t *perm;
    double *rec;
    int32_t *scan_tmp;
    int32_t *mid_list;
    int32_t *huge_list;
    int32_t *d_status;
    int32_t *h_status;  // pinned
    int32_t *d_work;    // assembly work counter
    int32_t *d_flags;   // first-writer zeroing: one flag per output node row (lazily allocated)
    int pending;        // an asynchronous sort whose status has not been checked (mm_sort_wait)
    void *sort_stream;  // the stream of the last asynchronous sort
    // incremental re-binning (mm_resort_by_cell), lazily allocated
    int32_t *perm2;     // [cap_rec] the other permutation buffer
    int32_t *inc_seg_old, *inc_arr_count, *inc_arr_begin, *inc_arr;
    int64_t inc_np;     // np the incremental buffers were sized for
    int32_t epoch;      // flag value of the last zeroing launch
    double *rec_tmp;    // record-first sort scratch [cap_rec][8] (inputs beyond L2, lazily allocated)
    int64_t cap_tmp;
    int dest_valid;     // rank[] holds the inverse permutation (classic path); else the atomic ranks
    void *d_dblk;       // two-phase deposit: per-bin pair-product blocks (lazily allocated)
    size_t dblk_bytes;
};

namespace {

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};

mm_status fail(mm_status st, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}

mm_status cuda_fail(cudaError_t e, const char *where)
{
    if (e == cudaErrorMemoryAllocation)
        return fail(MM_ERR_OUT_OF_MEMORY, "%s: %s", where, cudaGetErrorString(e));
    return fail(MM_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

mm_status check_grid(const mm_grid *g, int order)
{
    if (!g)
        return fail(MM_ERR_INVALID_ARG, "grid is NULL");
    if (order != 1 && order != 2)
        return fail(MM_ERR_INVALID_ARG, "order must be 1 or 2 (got %d)", order);
    for (int a = 0; a < 3; ++a) {
        if (g->n[a] < 2 * order + 1)
            return fail(MM_ERR_INVALID_ARG, "n[%d] = %d < 2*order+1 (stencil offsets would alias)", a, g->n[a]);
        if (!(g->h[a] > 0.0) || !std::isfinite(g->h[a]))
            return fail(MM_ERR_INVALID_ARG, "h[%d] must be finite and > 0", a);
    }
    if (g->x_begin < 0 || g->x_end > g->n[0] || g->x_end <= g->x_begin)
        return fail(MM_ERR_INVALID_ARG, "bad slab [%d, %d) for n[0] = %d", g->x_begin, g->x_end, g->n[0]);
    const bool whole = g->x_begin == 0 && g->x_end == g->n[0];
    if (!whole && g->x_end - g->x_begin < order)
        return fail(MM_ERR_INVALID_ARG, "slab width %d < order %d", g->x_end - g->x_begin, order);
    int64_t nbins = (int64_t)(g->x_end - g->x_begin + order - 1) * g->n[1] * g->n[2];
    if (nbins >= INT32_MAX)
        return fail(MM_ERR_INVALID_ARG, "too many bins (%lld)", (long long)nbins);
    return MM_OK;
}

void release(mm_sorted *h)
{
    if (!h)
        return;
    cudaFree(h->key);
    cudaFree(h->rank);
    cudaFree(h->count);
    cudaFree(h->seg_begin);
    cudaFree(h->perm);
    cudaFree(h->rec);
    cudaFree(h->scan_tmp);
    cudaFree(h->mid_list);
    cudaFree(h->huge_list);
    cudaFree(h->d_status);
    cudaFree(h->d_work);
    cudaFree(h->d_flags);
    cudaFree(h->d_dblk);
    cudaFree(h->rec_tmp);
    cudaFree(h->perm2);
    cudaFree(h->inc_seg_old);
    cudaFree(h->inc_arr_count);
    cudaFree(h->inc_arr_begin);
    cudaFree(h->inc_arr);
    if (h->h_status)
        cudaFreeHost(h->h_status);
    delete h;
}

}  // namespace

namespace mm {

void count_launch(int n)
{
    g_launches.fetch_add(n, std::memory_order_relaxed);
}

Geo make_geo(const mm_grid &g, int order)
{
    Geo o;
    o.n0 = g.n[0];
    o.n1 = g.n[1];
    o.n2 = g.n[2];
    o.h0 = g.h[0];
    o.h1 = g.h[1];
    o.h2 = g.h[2];
    o.x_begin = g.x_begin;
    o.x_end = g.x_end;
    o.order = order;
    o.periodic_x = (g.x_begin == 0 && g.x_end == g.n[0]) ? 1 : 0;
    o.nbx = g.x_end - g.x_begin + order - 1;
    // Division by a power of two is the exact product with its (exact) reciprocal, so the
    // IEEE-RN quotient x/h equals RN(x * (1/h)) bit for bit (R5).
    auto pow2 = [](double h) {
        int ex;
        return std::frexp(h, &ex) == 0.5 && ex > -1000 && ex < 1000;
    };
    o.ih0 = 1.0 / g.h[0];
    o.ih1 = 1.0 / g.h[1];
    o.ih2 = 1.0 / g.h[2];
    o.h_pow2 = pow2(g.h[0]) && pow2(g.h[1]) && pow2(g.h[2]);
    o.bx0 = 0;
    return o;
}

}  // namespace mm

extern "C" {

const char *mm_last_error(void)
{
    return g_err.c_str();
}

const char *mm_version(void)
{
    return "mm-b200 0.1 sm_100a (FP64 DMMA 8x8x4)";
}

int64_t mm_launch_count(void)
{
    return g_launches.load();
}

int mm_ghost_planes(int order)
{
    return order == 1 ? 1 : (order == 2 ? 3 : -1);
}

int64_t mm_out_elems(const mm_grid *g, int order, mm_kind kind)
{
    if (check_grid(g, order) != MM_OK || (kind != MM_SCALAR && kind != MM_TENSOR))
        return -1;
    int64_t S = (2 * order + 1) * (2 * order + 1) * (2 * order + 1);
    return (int64_t)(g->x_end - g->x_begin) * g->n[1] * g->n[2] * S * (int64_t)kind;
}

namespace {
// pos / B point to FP64 arrays (f32 = 0) or FP32 arrays (f32 = 1, widened exactly on load)
mm_status sort_common(const mm_grid *g, int order, int k_pad, int64_t np, const void *pos, const double *q,
                      const void *B, int f32, void *stream, mm_sorted **inout, bool async = false)
{
    try {
        mm_status st = check_grid(g, order);
        if (st)
            return st;
        if (!inout)
            return fail(MM_ERR_INVALID_ARG, "inout is NULL");
        if (k_pad < 4 || k_pad % 4 != 0 || k_pad > 1024)
            return fail(MM_ERR_INVALID_ARG, "k_pad must be a positive multiple of 4 (got %d)", k_pad);
        if (np < 0 || np >= INT32_MAX)
            return fail(MM_ERR_INVALID_ARG, "np out of range (%lld)", (long long)np);
        if (np > 0 && (!pos || !q))
            return fail(MM_ERR_INVALID_ARG, "pos/q must not be NULL");
        const int64_t nbins = (int64_t)(g->x_end - g->x_begin + order - 1) * g->n[1] * g->n[2];
        const int64_t cap_rec = np + nbins * (k_pad - 1);
        if (cap_rec >= INT32_MAX)
            return fail(MM_ERR_INVALID_ARG, "np + nbins*(k_pad-1) exceeds 2^31");
        mm_sorted *h = *inout;
        const bool fresh = (h == nullptr);
        if (!fresh) {
            if (h->order != order || memcmp(h->g.n, g->n, sizeof(g->n)) || h->g.x_begin != g->x_begin ||
                h->g.x_end != g->x_end || memcmp(h->g.h, g->h, sizeof(g->h)))
                return fail(MM_ERR_INCOMPATIBLE, "handle was created for another grid/order");
        } else {
            h = new (std::nothrow) mm_sorted;
            if (!h)
                return fail(MM_ERR_OUT_OF_MEMORY, "host allocation failed");
            memset(h, 0, sizeof(*h));
            h->g = *g;
            h->order = order;
            cudaGetDevice(&h->device);
        }
        cudaStream_t s = (cudaStream_t)stream;
        cudaError_t e = cudaSuccess;
        if (np > h->cap_np || !h->key) {
            cudaFree(h->key);
            cudaFree(h->rank);
            h->key = nullptr;
            h->rank = nullptr;
            h->cap_np = 0;
            const size_t n = (size_t)(np > 0 ? np : 1);
            e = cudaMalloc((void **)&h->key, sizeof(uint32_t) * n);
            if (!e) e = cudaMalloc((void **)&h->rank, sizeof(int32_t) * n);
            if (!e) h->cap_np = (int64_t)n;
        }
        if (!e && (cap_rec > h->cap_rec || !h->perm)) {
            cudaFree(h->perm);
            cudaFree(h->rec);
            h->perm = nullptr;
            h->rec = nullptr;
            h->cap_rec = 0;
            const size_t n = (size_t)(cap_rec > 0 ? cap_rec : 1);
            e = cudaMalloc((void **)&h->perm, sizeof(int32_t) * n);
            if (!e) e = cudaMalloc((void **)&h->rec, sizeof(double) * 8 * n);
            if (!e) h->cap_rec = (int64_t)n;
        }
        if (!e && !h->count) {
            const size_t nb = (size_t)(nbins > 0 ? nbins : 1);
            e = cudaMalloc((void **)&h->count, sizeof(int32_t) * nb);
            if (!e) e = cudaMalloc((void **)&h->seg_begin, sizeof(int32_t) * (nb + 1));
            if (!e) e = cudaMalloc((void **)&h->mid_list, sizeof(int32_t) * nb);
            if (!e) e = cudaMalloc((void **)&h->huge_list, sizeof(int32_t) * nb);
            if (!e) e = cudaMalloc((void **)&h->scan_tmp, sizeof(int32_t) * (size_t)mm::scan_tmp_elems(nbins));
            if (!e) e = cudaMalloc((void **)&h->d_status, sizeof(int32_t) * mm::ST_WORDS);
            if (!e) e = cudaMalloc((void **)&h->d_work, sizeof(int32_t) * 4);
            if (!e) e = cudaMallocHost((void **)&h->h_status, sizeof(int32_t) * mm::ST_WORDS);
            if (!e) e = cudaMemsetAsync(h->d_status, 0, sizeof(int32_t) * mm::ST_WORDS, (cudaStream_t)stream);
        }
        if (e) {
            if (fresh)
                release(h);
            return cuda_fail(e, "mm_sort_by_cell allocation");
        }
        h->k_pad = k_pad;
        h->has_B = B ? 1 : 0;
        h->nbins = nbins;
        h->np = np;
        h->valid = 0;
        mm::SortBufs b;
        b.np = np;
        b.nbins = nbins;
        b.k_pad = k_pad;
        b.pos = static_cast<const double *>(pos);
        b.q = q;
        b.B = static_cast<const double *>(B);
        b.f32 = f32;
        b.key = h->key;
        b.rank = h->rank;
        b.count = h->count;
        b.seg_begin = h->seg_begin;
        b.perm = h->perm;
        b.rec = h->rec;
        b.scan_tmp = h->scan_tmp;
        b.mid_list = h->mid_list;
        b.huge_list = h->huge_list;
        b.status = h->d_status;
        b.capacity = h->cap_rec;
        // record-first path from MM_SORT_RECFIRST_MIN particles on (default 48 M: beyond L2 the
        // classic path's random 4-B passes dominate)
        const char *rfm = getenv("MM_SORT_RECFIRST_MIN");  // read per call (tests, A/B)
        const int64_t recfirst_min = rfm ? (int64_t)atoll(rfm) : (int64_t)48 * 1000 * 1000;
        if (np >= recfirst_min && np > 0) {
            if (h->cap_tmp < h->cap_rec) {
                cudaFree(h->rec_tmp);
                h->rec_tmp = nullptr;
                h->cap_tmp = 0;
                e = cudaMalloc((void **)&h->rec_tmp, sizeof(double) * 8 * (size_t)h->cap_rec);
                if (e) {
                    if (fresh)
                        release(h);
                    return cuda_fail(e, "mm_sort_by_cell allocation");
                }
                h->cap_tmp = h->cap_rec;
            }
            b.rec_tmp = h->rec_tmp;
        }
        h->dest_valid = b.rec_tmp ? 0 : 1;
        e = mm::sort_enqueue(mm::make_geo(*g, order), b, s);
        if (async) {
            // no host round trip: the status stays on the device (sticky error word) until
            // mm_sort_wait; np_padded is read there too
            if (e) {
                if (fresh)
                    release(h);
                return cuda_fail(e, "mm_sort_by_cell_async");
            }
            h->valid = 1;
            h->pending = 1;
            h->sort_stream = stream;
            *inout = h;
            return MM_OK;
        }
        if (!e)
            e = cudaMemcpyAsync(h->h_status, h->d_status, sizeof(int32_t) * mm::ST_WORDS, cudaMemcpyDeviceToHost, s);
        if (!e)  // this sort's errors are reported now: clear the sticky word
            e = cudaMemsetAsync(h->d_status + mm::ST_STICKY, 0, sizeof(int32_t), s);
        if (!e)
            e = cudaStreamSynchronize(s);
        if (e) {
            if (fresh)
                release(h);
            return cuda_fail(e, "mm_sort_by_cell");
        }
        const int err = h->h_status[mm::ST_ERR];
        if (err) {
            if (fresh)
                release(h);
            if (err & mm::ERR_NONFINITE)
                return fail(MM_ERR_NONFINITE, "NaN/Inf in particle positions, charges or B");
            return fail(MM_ERR_DOMAIN, "particle outside the owned cell slab [%d,%d)x[0,%d)x[0,%d)", g->x_begin,
                        g->x_end, g->n[1], g->n[2]);
        }
        h->np_padded = h->h_status[mm::ST_NPAD];
        h->valid = 1;
        *inout = h;
        return MM_OK;
    } catch (...) {
        return fail(MM_ERR_CUDA, "unexpected exception in mm_sort_by_cell");
    }
}

}  // namespace

mm_status mm_sort_by_cell(const mm_grid *g, int order, int k_pad, int64_t np, const double *pos, const double *q,
                          const double *B, void *stream, mm_sorted **inout)
{
    return sort_common(g, order, k_pad, np, pos, q, B, 0, stream, inout);
}

mm_status mm_sort_by_cell_mixed(const mm_grid *g, int order, int k_pad, int64_t np, const float *pos,
                                const double *q, const float *B, void *stream, mm_sorted **inout)
{
    return sort_common(g, order, k_pad, np, pos, q, B, 1, stream, inout);
}

mm_status mm_sort_by_cell_async(const mm_grid *g, int order, int k_pad, int64_t np, const double *pos,
                                const double *q, const double *B, void *stream, mm_sorted **inout)
{
    return sort_common(g, order, k_pad, np, pos, q, B, 0, stream, inout, true);
}

mm_status mm_resort_by_cell(mm_sorted *h, int64_t np, const double *pos, const double *q, const double *B,
                            void *stream, int wait)
{
    try {
        if (!h)
            return fail(MM_ERR_INVALID_ARG, "NULL handle");
        if (h->pending) {  // the previous sort must be known good: its bins are the starting point
            mm_status st = mm_sort_wait(h, h->sort_stream);
            if (st)
                return st;
        }
        if (!h->valid)
            return fail(MM_ERR_INCOMPATIBLE, "handle holds no valid sort to update");
        if (np != h->np)
            return fail(MM_ERR_INCOMPATIBLE, "np (%lld) differs from the handle's sort (%lld)", (long long)np,
                        (long long)h->np);
        if ((B != nullptr) != (h->has_B != 0))
            return fail(MM_ERR_INCOMPATIBLE, "B must be given iff the handle was sorted with B");
        if (np > 0 && (!pos || !q))
            return fail(MM_ERR_INVALID_ARG, "pos/q must not be NULL");
        cudaStream_t s = (cudaStream_t)stream;
        cudaError_t e = cudaSuccess;
        if (!h->perm2 || h->inc_np < np) {
            cudaFree(h->perm2);
            cudaFree(h->inc_seg_old);
            cudaFree(h->inc_arr_count);
            cudaFree(h->inc_arr_begin);
            cudaFree(h->inc_arr);
            h->perm2 = h->inc_seg_old = h->inc_arr_count = h->inc_arr_begin = h->inc_arr = nullptr;
            h->inc_np = 0;
            const size_t nb = (size_t)(h->nbins > 0 ? h->nbins : 1), n = (size_t)(np > 0 ? np : 1);
            e = cudaMalloc((void **)&h->perm2, sizeof(int32_t) * (size_t)h->cap_rec);
            if (!e) e = cudaMalloc((void **)&h->inc_seg_old, sizeof(int32_t) * (nb + 1));
            if (!e) e = cudaMalloc((void **)&h->inc_arr_count, sizeof(int32_t) * nb);
            if (!e) e = cudaMalloc((void **)&h->inc_arr_begin, sizeof(int32_t) * (nb + 1));
            if (!e) e = cudaMalloc((void **)&h->inc_arr, sizeof(int32_t) * n);
            if (e)
                return cuda_fail(e, "mm_resort_by_cell allocation");
            h->inc_np = np;
        }
        mm::SortBufs b;
        b.np = np;
        b.nbins = h->nbins;
        b.k_pad = h->k_pad;
        b.pos = pos;
        b.q = q;
        b.B = B;
        b.f32 = 0;
        b.key = h->key;
        b.rank = h->rank;
        b.count = h->count;
        b.seg_begin = h->seg_begin;
        b.perm = h->perm2;  // the new permutation
        b.rec = h->rec;
        b.scan_tmp = h->scan_tmp;
        b.mid_list = h->mid_list;
        b.huge_list = h->huge_list;
        b.status = h->d_status;
        b.capacity = h->cap_rec;
        mm::IncBufs ib;
        ib.perm_old = h->perm;
        ib.seg_old = h->inc_seg_old;
        ib.arr_count = h->inc_arr_count;
        ib.arr_begin = h->inc_arr_begin;
        ib.arr = h->inc_arr;
        h->valid = 0;
        if (!h->dest_valid) {  // the record-first sort left the atomic ranks in rank[]
            e = mm::inverse_enqueue(h->perm, h->seg_begin + h->nbins, h->cap_rec, h->rank, s);
            if (e)
                return cuda_fail(e, "mm_resort_by_cell");
            h->dest_valid = 1;
        }
        e = mm::resort_enqueue(mm::make_geo(h->g, h->order), b, ib, s);
        if (e)
            return cuda_fail(e, "mm_resort_by_cell");
        int32_t *t = h->perm;  // stream order: later work sees the new buffer
        h->perm = h->perm2;
        h->perm2 = t;
        h->valid = 1;
        if (!wait) {
            h->pending = 1;
            h->sort_stream = stream;
            return MM_OK;
        }
        e = cudaMemcpyAsync(h->h_status, h->d_status, sizeof(int32_t) * mm::ST_WORDS, cudaMemcpyDeviceToHost, s);
        if (!e)
            e = cudaMemsetAsync(h->d_status + mm::ST_STICKY, 0, sizeof(int32_t), s);
        if (!e)
            e = cudaStreamSynchronize(s);
        if (e)
            return cuda_fail(e, "mm_resort_by_cell");
        const int err = h->h_status[mm::ST_ERR];
        if (err) {
            h->valid = 0;
            if (err & mm::ERR_NONFINITE)
                return fail(MM_ERR_NONFINITE, "NaN/Inf in particle positions, charges or B");
            return fail(MM_ERR_DOMAIN, "particle outside the owned cell slab");
        }
        h->np_padded = h->h_status[mm::ST_NPAD];
        return MM_OK;
    } catch (...) {
        return fail(MM_ERR_CUDA, "unexpected exception in mm_resort_by_cell");
    }
}

mm_status mm_sort_wait(mm_sorted *h, void *stream)
{
    try {
        if (!h)
            return fail(MM_ERR_INVALID_ARG, "NULL handle");
        if (!h->pending)
            return MM_OK;
        cudaStream_t s = (cudaStream_t)stream;
        cudaError_t e = cudaMemcpyAsync(h->h_status, h->d_status, sizeof(int32_t) * mm::ST_WORDS,
                                        cudaMemcpyDeviceToHost, s);
        if (!e)
            e = cudaMemsetAsync(h->d_status + mm::ST_STICKY, 0, sizeof(int32_t), s);
        if (!e)
            e = cudaStreamSynchronize(s);
        if (e)
            return cuda_fail(e, "mm_sort_wait");
        h->pending = 0;
        h->np_padded = h->h_status[mm::ST_NPAD];
        const int err = h->h_status[mm::ST_STICKY];
        if (err) {
            h->valid = 0;
            if (err & mm::ERR_NONFINITE)
                return fail(MM_ERR_NONFINITE, "NaN/Inf in particle positions, charges or B (asynchronous sort)");
            return fail(MM_ERR_DOMAIN, "particle outside the owned cell slab (asynchronous sort)");
        }
        return MM_OK;
    } catch (...) {
        return fail(MM_ERR_CUDA, "unexpected exception in mm_sort_wait");
    }
}

mm_status mm_sorted_view(const mm_sorted *h, mm_sorted_info *out)
{
    if (!h || !out)
        return fail(MM_ERR_INVALID_ARG, "NULL argument");
    if (h->pending) {
        mm_status st = mm_sort_wait(const_cast<mm_sorted *>(h), h->sort_stream);
        if (st)
            return st;
    }
    if (!h->valid)
        return fail(MM_ERR_INCOMPATIBLE, "handle holds no valid sort");
    out->np = h->np;
    out->np_padded = h->np_padded;
    out->nbins = h->nbins;
    out->capacity = h->cap_rec;
    out->order = h->order;
    out->k_pad = h->k_pad;
    out->has_B = h->has_B;
    out->rec_stride = h->has_B ? 8 : 4;
    out->perm = h->perm;
    out->seg_begin = h->seg_begin;
    out->seg_count = h->count;
    out->rec = h->rec;
    return MM_OK;
}

}  // extern "C"

namespace {

mm_status check_assemble(const mm_sorted *h, mm_kind kind, mm_precision prec, const mm_species *sp, const void *out)
{
    if (!h || !sp || !out)
        return fail(MM_ERR_INVALID_ARG, "NULL handle, species or out");
    if (!h->valid)
        return fail(MM_ERR_INCOMPATIBLE, "handle holds no valid sort");
    if (kind != MM_SCALAR && kind != MM_TENSOR)
        return fail(MM_ERR_INVALID_ARG, "kind must be MM_SCALAR or MM_TENSOR");
    if (prec != MM_FP64 && prec != MM_TF32 && prec != MM_TF32X3)
        return fail(MM_ERR_INVALID_ARG, "precision must be MM_FP64, MM_TF32 or MM_TF32X3");
    if (kind == MM_TENSOR && !h->has_B && h->np > 0)
        return fail(MM_ERR_INCOMPATIBLE, "MM_TENSOR needs a handle sorted with B");
    if (!(sp->c > 0.0) || !std::isfinite(sp->qom) || !std::isfinite(sp->dt) || !std::isfinite(sp->sigma) ||
        !std::isfinite(sp->c))
        return fail(MM_ERR_INVALID_ARG, "species constants must be finite with c > 0");
    return MM_OK;
}

// The assembly kernels over the bin planes [bx_lo, bx_hi) of a handle (the whole range for
// mm_assemble; boundary / interior ranges for mm_assemble_slab).  work_idx selects the launch's
// work counter (zeroed by the caller).
cudaError_t enqueue_range(const mm_sorted *h, mm::Geo geo, mm_kind kind, mm_precision prec, const mm_species *sp,
                          void *out, void *ghost, int bx_lo, int bx_hi, int work_idx, cudaStream_t s,
                          int32_t *zflags = nullptr, int32_t zepoch = 0, void *dblk = nullptr)
{
    const int64_t plane = (int64_t)h->g.n[1] * h->g.n[2];
    if (bx_hi <= bx_lo)
        return cudaSuccess;
    geo.bx0 = bx_lo;
    mm::AsmArgs a;
    a.work = h->d_work + work_idx;
    a.rec = h->rec;
    a.rec_stride = h->has_B ? 8 : 4;
    a.seg_begin = h->seg_begin + plane * bx_lo;
    a.nbins = plane * (bx_hi - bx_lo);
    a.ncomp = (int)kind;
    a.wscale = sp->qom * sp->dt / 2.0 / sp->c;
    a.sigma = sp->sigma;
    a.out = static_cast<double *>(out);
    a.ghost = geo.periodic_x ? nullptr : static_cast<double *>(ghost);
    a.zflags = zflags;
    a.zepoch = zepoch;
    a.dblk = dblk ? static_cast<char *>(dblk) + (prec == MM_FP64 ? 8 : 4) * plane * bx_lo *
                                                     mm::block_elems(h->order, (int)kind)
                  : nullptr;
    if (prec == MM_FP64)
        return mm::assemble_fp64_enqueue(geo, a, s);
    return mm::assemble_tf32_enqueue(geo, a, prec == MM_TF32X3 ? 1 : 0, s);
}

// Two-phase deposit (mm_nodesum.cu) over the whole bin range: the assembly kernel stores one
// pair-product block per bin, a node-row kernel sums them (no REDs, no zero-fill).  Measured
// slower than the RED deposit on every config (the node kernel is L1-bound), so
// it is off unless MM_TWO_PHASE (read per call) selects it: bit 0 TF32 order 2, bit 1 TF32
// order 1, bit 2 FP64 order 2, bit 3 (diagnostics) phase 1 alone.  tests/test_gpu_twophase.py.
bool two_phase(const mm_sorted *h, mm_precision prec)
{
    const char *v = getenv("MM_TWO_PHASE");
    const int mode = v ? atoi(v) : 0;
    if (prec == MM_FP64)
        return h->order == 2 && (mode & 4);
    return h->order == 2 ? (mode & 1) : (mode & 2);
}

int64_t row_elems(const mm_sorted *h, mm_kind kind)
{
    const int64_t S = (2 * h->order + 1) * (2 * h->order + 1) * (2 * h->order + 1);
    return S * (int64_t)kind;
}

}  // namespace

namespace mm {
mm_status api_fail(mm_status st, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return st;
}
}  // namespace mm

extern "C" {

mm_status mm_assemble(const mm_sorted *h, mm_kind kind, mm_precision prec, const mm_species *sp, int accumulate,
                      void *out, void *ghost, void *stream)
{
    try {
        mm_status st = check_assemble(h, kind, prec, sp, out);
        if (st)
            return st;
        mm::Geo geo = mm::make_geo(h->g, h->order);
        if (!geo.periodic_x && !ghost)
            return fail(MM_ERR_INVALID_ARG, "slab grid needs a ghost buffer");
        const size_t esz = prec == MM_FP64 ? sizeof(double) : sizeof(float);
        cudaStream_t s = (cudaStream_t)stream;
        const int64_t rowlen = row_elems(h, kind);
        const int64_t nout = (int64_t)(h->g.x_end - h->g.x_begin) * h->g.n[1] * h->g.n[2] * rowlen;
        const int64_t nghost = geo.periodic_x ? 0 : (int64_t)mm_ghost_planes(h->order) * h->g.n[1] * h->g.n[2] * rowlen;
        cudaError_t e = cudaSuccess;
        // kernels that zero their output rows themselves (first-writer flags)
        int32_t *zflags = nullptr;
        if (!accumulate && mm::zeroes_inside(h->order, (int)kind, prec == MM_FP64 ? 0 : 1)) {
            mm_sorted *hm = const_cast<mm_sorted *>(h);
            if (!hm->d_flags) {
                e = cudaMalloc((void **)&hm->d_flags, sizeof(int32_t) * (size_t)mm::flag_rows(h->g, h->order));
                if (!e)
                    e = cudaMemsetAsync(hm->d_flags, 0, sizeof(int32_t) * (size_t)mm::flag_rows(h->g, h->order), s);
                if (e)
                    return cuda_fail(e, "mm_assemble flags");
                hm->epoch = 0;
            }
            if (++hm->epoch == INT32_MAX) {  // flags restart from 0 after 2^31 launches
                e = cudaMemsetAsync(hm->d_flags, 0, sizeof(int32_t) * (size_t)mm::flag_rows(h->g, h->order), s);
                if (e)
                    return cuda_fail(e, "mm_assemble flags");
                hm->epoch = 1;
            }
            zflags = hm->d_flags;
        }
        if (two_phase(h, prec)) {
            mm_sorted *hm = const_cast<mm_sorted *>(h);
            const size_t need = esz * (size_t)h->nbins * (size_t)mm::block_elems(h->order, (int)kind);
            if (hm->dblk_bytes < need) {
                cudaFree(hm->d_dblk);
                hm->d_dblk = nullptr;
                hm->dblk_bytes = 0;
                e = cudaMalloc(&hm->d_dblk, need);
                if (e)
                    return cuda_fail(e, "mm_assemble block buffer");
                hm->dblk_bytes = need;
            }
            e = cudaMemsetAsync(h->d_work, 0, sizeof(int32_t) * 4, s);
            if (!e)
                e = enqueue_range(h, geo, kind, prec, sp, out, ghost, 0, geo.nbx, 0, s, nullptr, 0, hm->d_dblk);
            const char *v = getenv("MM_TWO_PHASE");  // bit 3: phase 1 alone (timing diagnostics)
            if (!e && !(v && (atoi(v) & 8)))
                e = mm::nodesum_enqueue(geo, (int)kind, (int)esz, hm->d_dblk, out,
                                        geo.periodic_x ? nullptr : ghost, accumulate, s);
            if (e)
                return cuda_fail(e, "mm_assemble launch");
            return MM_OK;
        }
        if (!accumulate && !zflags) {
            e = cudaMemsetAsync(out, 0, esz * (size_t)nout, s);
            if (!e && nghost)
                e = cudaMemsetAsync(ghost, 0, esz * (size_t)nghost, s);
            if (e)
                return cuda_fail(e, "mm_assemble memset");
        }
        // the work counter is read by the ticket-scheduled FP64 kernels (runs of bins per atomic);
        // the TF32 kernels use a static schedule
        if (zflags || prec == MM_FP64) {
            e = cudaMemsetAsync(h->d_work, 0, sizeof(int32_t) * 4, s);
            if (e)
                return cuda_fail(e, "mm_assemble memset");
        }
        e = enqueue_range(h, geo, kind, prec, sp, out, ghost, 0, geo.nbx, 0, s, zflags, zflags ? h->epoch : 0);
        if (e)
            return cuda_fail(e, "mm_assemble launch");
        return MM_OK;
    } catch (...) {
        return fail(MM_ERR_CUDA, "unexpected exception in mm_assemble");
    }
}

mm_status mm_ghost_exchange(mm_comm *comm, const mm_grid *g, int order, mm_kind kind, mm_precision prec, void *out,
                            void *ghost, void *stream)
{
    try {
        mm_status st = check_grid(g, order);
        if (st)
            return st;
        if (!comm || !out || !ghost)
            return fail(MM_ERR_INVALID_ARG, "NULL comm, out or ghost");
        if (kind != MM_SCALAR && kind != MM_TENSOR)
            return fail(MM_ERR_INVALID_ARG, "kind must be MM_SCALAR or MM_TENSOR");
        const bool whole = g->x_begin == 0 && g->x_end == g->n[0];
        if (whole != (mm::comm_nranks(comm) == 1))
            return fail(MM_ERR_INCOMPATIBLE, "a slab grid needs a communicator of >= 2 ranks, a whole grid one rank");
        const int64_t S = (2 * order + 1) * (2 * order + 1) * (2 * order + 1);
        int rc = 0;
        cudaError_t e = mm::ghost_exchange_enqueue(comm, order, g->x_end - g->x_begin,
                                                   (int64_t)g->n[1] * g->n[2] * S * (int64_t)kind,
                                                   prec == MM_FP64 ? 8 : 4, out, ghost, (cudaStream_t)stream, &rc,
                                                   nullptr, nullptr);
        if (rc)
            return fail(MM_ERR_NCCL, "ghost exchange: %s", mm::nccl_error(rc));
        if (e)
            return cuda_fail(e, "ghost exchange");
        return MM_OK;
    } catch (...) {
        return fail(MM_ERR_CUDA, "unexpected exception in mm_ghost_exchange");
    }
}

mm_status mm_assemble_slab(const mm_sorted *h, mm_kind kind, mm_precision prec, const mm_species *sp, int accumulate,
                           void *out, void *ghost, mm_comm *comm, void *stream)
{
    try {
        mm_status st = check_assemble(h, kind, prec, sp, out);
        if (st)
            return st;
        if (!comm || !ghost)
            return fail(MM_ERR_INVALID_ARG, "NULL comm or ghost");
        const bool whole = h->g.x_begin == 0 && h->g.x_end == h->g.n[0];
        if (whole != (mm::comm_nranks(comm) == 1))
            return fail(MM_ERR_INCOMPATIBLE, "a slab grid needs a communicator of >= 2 ranks, a whole grid one rank");
        mm::Geo geo = mm::make_geo(h->g, h->order);
        geo.periodic_x = 0;  // one rank: its own ring neighbour (self ring), same path as N ranks
        const int o = h->order, w = h->g.x_end - h->g.x_begin, nbx = geo.nbx;
        const size_t esz = prec == MM_FP64 ? sizeof(double) : sizeof(float);
        cudaStream_t s = (cudaStream_t)stream;
        const int64_t rowlen = row_elems(h, kind);
        const int64_t plane_elems = (int64_t)h->g.n[1] * h->g.n[2] * rowlen;
        cudaError_t e = cudaMemsetAsync(ghost, 0, esz * (size_t)(mm_ghost_planes(o) * plane_elems), s);
        if (!e && !accumulate)
            e = cudaMemsetAsync(out, 0, esz * (size_t)(w * plane_elems), s);
        if (!e)
            e = cudaMemsetAsync(h->d_work, 0, sizeof(int32_t) * 4, s);
        if (e)
            return cuda_fail(e, "mm_assemble_slab memset");
        // boundary bin planes (their windows reach a ghost plane) first, then the exchange on the
        // comm stream overlapped with the interior bins, then the received planes are added
        // order 1: boundary bx = nbx-1 (node plane x_end); order 2: bx = 0 (x_begin-1) and
        // bx = nbx-2, nbx-1 (x_end, x_end+1)
        int lo_hi = 0, hi_lo = nbx - 1;
        if (o == 2) {
            lo_hi = 1;
            hi_lo = nbx - 2;
            if (hi_lo < lo_hi)
                hi_lo = lo_hi;
        }
        e = enqueue_range(h, geo, kind, prec, sp, out, ghost, 0, lo_hi, 0, s);
        if (!e)
            e = enqueue_range(h, geo, kind, prec, sp, out, ghost, hi_lo, nbx, 1, s);
        if (e)
            return cuda_fail(e, "mm_assemble_slab launch");
        int rc = 0;
        // the interior launch is enqueued between the event the comm stream waits for and the
        // wait for the received planes: ghost_exchange_enqueue records ev_ready first
        struct Interior {
            const mm_sorted *h;
            mm::Geo geo;
            mm_kind kind;
            mm_precision prec;
            const mm_species *sp;
            void *out, *ghost;
            int lo, hi;
            cudaStream_t s;
        } in = {h, geo, kind, prec, sp, out, ghost, lo_hi, hi_lo, s};
        e = mm::ghost_exchange_enqueue(
            comm, o, w, plane_elems, (int)esz, out, ghost, s, &rc,
            [](void *p) {
                const Interior *q = static_cast<const Interior *>(p);
                return enqueue_range(q->h, q->geo, q->kind, q->prec, q->sp, q->out, q->ghost, q->lo, q->hi, 2, q->s);
            },
            &in);
        if (rc)
            return fail(MM_ERR_NCCL, "ghost exchange: %s", mm::nccl_error(rc));
        if (e)
            return cuda_fail(e, "mm_assemble_slab");
        return MM_OK;
    } catch (...) {
        return fail(MM_ERR_CUDA, "unexpected exception in mm_assemble_slab");
    }
}

mm_status mm_deposit_moments(const mm_sorted *h, int nq, const mm_species *sp, const double *v, int accumulate,
                             double *out, double *ghost, void *stream)
{
    try {
        if (!h || !sp || !out || (h->np > 0 && !v))
            return fail(MM_ERR_INVALID_ARG, "NULL handle, species, v or out");
        if (!h->valid)
            return fail(MM_ERR_INCOMPATIBLE, "handle holds no valid sort");
        if (nq != 4 && nq != 10)
            return fail(MM_ERR_INVALID_ARG, "nq must be 4 (rho, J) or 10 (implicit moments)");
        if (!std::isfinite(sp->sigma))
            return fail(MM_ERR_INVALID_ARG, "sigma must be finite");
        mm::Geo geo = mm::make_geo(h->g, h->order);
        if (!geo.periodic_x && !ghost)
            return fail(MM_ERR_INVALID_ARG, "slab grid needs a ghost buffer");
        cudaStream_t s = (cudaStream_t)stream;
        const int64_t plane = (int64_t)h->g.n[1] * h->g.n[2] * nq;
        cudaError_t e = cudaSuccess;
        if (!accumulate) {
            e = cudaMemsetAsync(out, 0, sizeof(double) * (size_t)((h->g.x_end - h->g.x_begin) * plane), s);
            if (!e && !geo.periodic_x)
                e = cudaMemsetAsync(ghost, 0, sizeof(double) * (size_t)(mm_ghost_planes(h->order) * plane), s);
        }
        if (!e)
            e = mm::moments_enqueue(geo, nq, h->rec, h->has_B ? 8 : 4, h->perm, h->seg_begin, h->nbins, v, sp->sigma,
                                    out, geo.periodic_x ? nullptr : ghost, s);
        if (e)
            return cuda_fail(e, "mm_deposit_moments");
        return MM_OK;
    } catch (...) {
        return fail(MM_ERR_CUDA, "unexpected exception in mm_deposit_moments");
    }
}

mm_status mm_gather_field(mm_sorted *h, const double *F, double *Fp, void *stream)
{
    try {
        if (!h || !F)
            return fail(MM_ERR_INVALID_ARG, "NULL handle or field");
        if (!h->valid)
            return fail(MM_ERR_INCOMPATIBLE, "handle holds no valid sort");
        if (!h->has_B && h->np > 0)
            return fail(MM_ERR_INCOMPATIBLE, "the gather writes B into the records: sort with B");
        mm::Geo geo = mm::make_geo(h->g, h->order);
        cudaError_t e = mm::gather_enqueue(geo, h->rec, h->perm, h->seg_begin, h->nbins, F, Fp, (cudaStream_t)stream);
        if (e)
            return cuda_fail(e, "mm_gather_field");
        return MM_OK;
    } catch (...) {
        return fail(MM_ERR_CUDA, "unexpected exception in mm_gather_field");
    }
}

mm_status mm_apply(const mm_grid *g, int order, mm_kind kind, const double *M, const double *E, double *y,
                   int accumulate, void *stream)
{
    try {
        mm_status st = check_grid(g, order);
        if (st)
            return st;
        if (kind != MM_SCALAR && kind != MM_TENSOR)
            return fail(MM_ERR_INVALID_ARG, "kind must be MM_SCALAR or MM_TENSOR");
        if (!M || !E || !y)
            return fail(MM_ERR_INVALID_ARG, "NULL M, E or y");
        if (g->x_begin != 0 || g->x_end != g->n[0])
            return fail(MM_ERR_INCOMPATIBLE, "mm_apply supports the whole periodic domain only in this version");
        mm::Geo geo = mm::make_geo(*g, order);
        cudaError_t e = mm::apply_enqueue(geo, (int)kind, M, E, y, accumulate ? 1 : 0, (cudaStream_t)stream);
        if (e)
            return cuda_fail(e, "mm_apply launch");
        return MM_OK;
    } catch (...) {
        return fail(MM_ERR_CUDA, "unexpected exception in mm_apply");
    }
}

mm_status mm_slab_partition(const mm_grid *g, int64_t np, const double *pos, const double *q, const double *B,
                            double *pos_out, double *q_out, double *B_out, int64_t counts[3], void *stream)
{
    try {
        mm_status st = check_grid(g, 1);
        if (st)
            return st;
        if (!counts || np < 0 || np >= INT32_MAX)
            return fail(MM_ERR_INVALID_ARG, "counts NULL or np out of range");
        if (np > 0 && (!pos || !q || !pos_out || !q_out || (B && !B_out)))
            return fail(MM_ERR_INVALID_ARG, "NULL particle arrays");
        cudaStream_t s = (cudaStream_t)stream;
        const mm::Geo geo = mm::make_geo(*g, 1);
        int32_t *tmp = nullptr;
        const int64_t nt = mm::partition_tmp_elems(np);
        cudaError_t e = cudaMallocAsync((void **)&tmp, sizeof(int32_t) * (size_t)nt, s);
        if (!e)
            e = mm::partition_enqueue(geo, np, pos, q, B, pos_out, q_out, B_out, tmp, s);
        int32_t ends[3] = {0, 0, 0};
        if (!e)
            e = cudaMemcpyAsync(ends, tmp + nt - 3, sizeof(ends), cudaMemcpyDeviceToHost, s);
        if (tmp)
            cudaFreeAsync(tmp, s);
        if (!e)
            e = cudaStreamSynchronize(s);
        if (e)
            return cuda_fail(e, "mm_slab_partition");
        counts[0] = ends[0];
        counts[1] = ends[1] - ends[0];
        counts[2] = ends[2] - ends[1];
        return MM_OK;
    } catch (...) {
        return fail(MM_ERR_CUDA, "unexpected exception in mm_slab_partition");
    }
}

mm_status mm_ghost_add(const mm_grid *g, int order, mm_kind kind, double *out, const double *recv, int first_plane,
                       int nplanes, void *stream)
{
    mm_status st = check_grid(g, order);
    if (st)
        return st;
    if (kind != MM_SCALAR && kind != MM_TENSOR)
        return fail(MM_ERR_INVALID_ARG, "bad kind");
    const int w = g->x_end - g->x_begin;
    if (!out || !recv || nplanes < 0 || first_plane < 0 || first_plane + nplanes > w)
        return fail(MM_ERR_INVALID_ARG, "bad ghost_add arguments (planes [%d,%d) of %d)", first_plane,
                    first_plane + nplanes, w);
    const int64_t S = (2 * order + 1) * (2 * order + 1) * (2 * order + 1);
    const int64_t plane = (int64_t)g->n[1] * g->n[2] * S * (int64_t)kind;
    cudaError_t e = mm::ghost_add_enqueue(out + first_plane * plane, recv, nplanes * plane, (cudaStream_t)stream);
    if (e)
        return cuda_fail(e, "mm_ghost_add");
    return MM_OK;
}

void mm_free(mm_sorted *h)
{
    if (!h)
        return;
    cudaDeviceSynchronize();
    release(h);
}

}  // extern "C"
