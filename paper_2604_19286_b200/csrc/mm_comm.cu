// Multi-GPU boundary of libmm: an NCCL communicator
// owned by the library, the ghost-plane reduction over NCCL send/recv, and the slab assembly
// that overlaps that exchange with the interior bins.
//
// x-slab decomposition with particles owned by cell (north_star): rank r owns node planes
// [x_begin, x_end).  mm_assemble writes the rows of nodes outside the slab into ghost planes
// (order 1: plane x_end; order 2: x_begin - 1, x_end, x_end + 1), and only those planes are
// exchanged, on a periodic ring:
//   order 1: ghost 0 (node plane x_end)       -> r + 1, added into its owned plane 0
//   order 2: ghost 0 (x_begin - 1)             -> r - 1, added into its last owned plane
//            ghosts 1, 2 (x_end, x_end + 1)    -> r + 1, added into its owned planes 0, 1
// (slab width >= order, so a ghost plane never skips a rank).  Every rank posts, inside one
// ncclGroupStart/End, send(next), recv(prev), send(prev), recv(next): between two ranks the
// messages of one direction match in posting order even when next == prev (world 2), and a
// world of one rank sends to itself (the "self ring", the same code path on one GPU).
//
// NCCL is loaded at run time (dlopen of libnccl.so.2: inside a PyTorch process this is the
// library torch already loaded), so libmm links and loads on hosts without NCCL and the
// communicator calls report MM_ERR_NCCL there.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <new>

#include "mm_internal.cuh"

namespace mm {
namespace {

struct NcclApi {
    bool ok = false;
    const char *why = "NCCL not loaded";
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl()
{
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = "libnccl.so.2 not found";
            return;
        }
        auto sym = [&](const char *n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
        api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
        api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
        api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd &&
                 api.Send && api.Recv && api.GetErrorString;
        if (!api.ok)
            api.why = "libnccl.so.2 lacks a required symbol";
    });
    return api;
}

// elementwise add of received FP32 ghost planes (the FP64 kernel lives in mm_halo.cu)
__global__ void k_ghost_add_f32(float *__restrict__ out, const float *__restrict__ recv, int64_t n)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] += __ldg(recv + i);
}

}  // namespace
}  // namespace mm

struct mm_comm {
    ncclComm_t nc;
    int nranks, rank, device;
    cudaStream_t cs;        // communication stream
    cudaEvent_t ev_ready;   // ghost planes complete (main stream)
    cudaEvent_t ev_done;    // received planes available (comm stream)
    void *recv;             // receive buffers (grown on demand)
    size_t recv_bytes;
};

namespace mm {

const char *nccl_error(int r)
{
    const NcclApi &a = nccl();
    return a.ok ? a.GetErrorString((ncclResult_t)r) : a.why;
}

bool nccl_available(const char **why)
{
    const NcclApi &a = nccl();
    if (why)
        *why = a.why;
    return a.ok;
}

cudaError_t ghost_add_f32_enqueue(float *out, const float *recv, int64_t n, cudaStream_t s)
{
    if (n <= 0)
        return cudaSuccess;
    int blocks = (int)((n + 255) / 256);
    if (blocks > 148 * 8)
        blocks = 148 * 8;
    k_ghost_add_f32<<<blocks, 256, 0, s>>>(out, recv, n);
    count_launch();
    return cudaGetLastError();
}

// Exchange of the ghost planes over the communicator and their addition into the owned rows
// (see the routing table at the top of the file).  Everything is asynchronous on `s`: the comm
// stream waits for `s`, runs the NCCL group, `between` (if any) enqueues more work on `s` that
// overlaps the transfer, and `s` waits for the comm stream before the add kernels.
// elem_bytes = 8 (FP64 output) | 4 (FP32 output of the TF32 paths).  Returns 0 or a
// (negated) ncclResult_t / a positive cudaError_t through *nccl_rc / the return value.
cudaError_t ghost_exchange_enqueue(mm_comm *c, int order, int width, int64_t plane_elems, int elem_bytes, void *out,
                                   void *ghost, cudaStream_t s, int *nccl_rc, cudaError_t (*between)(void *),
                                   void *between_ctx)
{
    const NcclApi &a = nccl();
    *nccl_rc = 0;
    const int np_next = order == 1 ? 1 : 2;  // planes to r+1 (ghost planes 0 | 1, 2)
    const int np_prev = order == 1 ? 0 : 1;  // planes to r-1 (ghost plane 0)
    const size_t pb = (size_t)plane_elems * elem_bytes;
    const size_t need = pb * (np_next + np_prev);
    if (c->recv_bytes < need) {
        cudaError_t e = cudaStreamSynchronize(c->cs);
        if (!e) {
            cudaFree(c->recv);
            c->recv = nullptr;
            c->recv_bytes = 0;
            e = cudaMalloc(&c->recv, need);
        }
        if (e)
            return e;
        c->recv_bytes = need;
    }
    char *g = static_cast<char *>(ghost);
    char *r_prev = static_cast<char *>(c->recv);          // np_next planes from r-1
    char *r_next = r_prev + pb * np_next;                  // np_prev planes from r+1
    const int nxt = (c->rank + 1) % c->nranks, prv = (c->rank + c->nranks - 1) % c->nranks;
    const ncclDataType_t dt = elem_bytes == 8 ? ncclFloat64 : ncclFloat32;
    const size_t cnt_next = (size_t)plane_elems * np_next, cnt_prev = (size_t)plane_elems * np_prev;
    cudaError_t e = cudaEventRecord(c->ev_ready, s);
    if (!e)
        e = cudaStreamWaitEvent(c->cs, c->ev_ready, 0);
    if (e)
        return e;
    ncclResult_t r = a.GroupStart();
    const char *send_next = g + (order == 1 ? 0 : pb);     // ghost plane 0 | planes 1, 2
    if (r == ncclSuccess)
        r = a.Send(send_next, cnt_next, dt, nxt, c->nc, c->cs);
    if (r == ncclSuccess)
        r = a.Recv(r_prev, cnt_next, dt, prv, c->nc, c->cs);
    if (r == ncclSuccess && np_prev) {
        r = a.Send(g, cnt_prev, dt, prv, c->nc, c->cs);
        if (r == ncclSuccess)
            r = a.Recv(r_next, cnt_prev, dt, nxt, c->nc, c->cs);
    }
    const ncclResult_t r2 = a.GroupEnd();
    if (r == ncclSuccess)
        r = r2;
    if (r != ncclSuccess) {
        *nccl_rc = (int)r;
        return cudaSuccess;
    }
    e = cudaEventRecord(c->ev_done, c->cs);
    // work enqueued on s here (the interior bins of mm_assemble_slab) overlaps the exchange
    if (!e && between)
        e = between(between_ctx);
    if (!e)
        e = cudaStreamWaitEvent(s, c->ev_done, 0);
    if (e)
        return e;
    // planes from r-1 (its x_end, x_end+1) are owned planes 0, 1; the plane from r+1 (its
    // x_begin - 1) is the last owned plane
    char *o = static_cast<char *>(out);
    for (int k = 0; k < np_next && !e; ++k)
        e = elem_bytes == 8 ? ghost_add_enqueue(reinterpret_cast<double *>(o + pb * k),
                                                reinterpret_cast<const double *>(r_prev + pb * k), plane_elems, s)
                            : ghost_add_f32_enqueue(reinterpret_cast<float *>(o + pb * k),
                                                    reinterpret_cast<const float *>(r_prev + pb * k), plane_elems, s);
    if (np_prev && !e)
        e = elem_bytes == 8 ? ghost_add_enqueue(reinterpret_cast<double *>(o + pb * (width - 1)),
                                                reinterpret_cast<const double *>(r_next), plane_elems, s)
                            : ghost_add_f32_enqueue(reinterpret_cast<float *>(o + pb * (width - 1)),
                                                    reinterpret_cast<const float *>(r_next), plane_elems, s);
    return e;
}

int comm_nranks(const mm_comm *c) { return c->nranks; }
int comm_rank(const mm_comm *c) { return c->rank; }

}  // namespace mm

extern "C" {

mm_status mm_comm_unique_id(void *uid)
{
    const mm::NcclApi &a = mm::nccl();
    if (!uid)
        return mm::api_fail(MM_ERR_INVALID_ARG, "uid is NULL");
    if (!a.ok)
        return mm::api_fail(MM_ERR_NCCL, a.why);
    ncclUniqueId id;
    const ncclResult_t r = a.GetUniqueId(&id);
    if (r != ncclSuccess)
        return mm::api_fail(MM_ERR_NCCL, a.GetErrorString(r));
    memcpy(uid, id.internal, NCCL_UNIQUE_ID_BYTES);
    return MM_OK;
}

mm_status mm_comm_create(int nranks, int rank, const void *uid, mm_comm **out)
{
    const mm::NcclApi &a = mm::nccl();
    if (!uid || !out || nranks < 1 || rank < 0 || rank >= nranks)
        return mm::api_fail(MM_ERR_INVALID_ARG, "bad communicator arguments (nranks %d, rank %d)", nranks, rank);
    if (!a.ok)
        return mm::api_fail(MM_ERR_NCCL, a.why);
    mm_comm *c = new (std::nothrow) mm_comm;
    if (!c)
        return mm::api_fail(MM_ERR_OUT_OF_MEMORY, "host allocation failed");
    memset(c, 0, sizeof(*c));
    c->nranks = nranks;
    c->rank = rank;
    cudaGetDevice(&c->device);
    cudaError_t e = cudaStreamCreateWithFlags(&c->cs, cudaStreamNonBlocking);
    if (!e)
        e = cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming);
    if (!e)
        e = cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming);
    if (e) {
        mm_comm_free(c);
        return mm::api_fail(MM_ERR_CUDA, "mm_comm_create: %s", cudaGetErrorString(e));
    }
    ncclUniqueId id;
    memcpy(id.internal, uid, NCCL_UNIQUE_ID_BYTES);
    const ncclResult_t r = a.CommInitRank(&c->nc, nranks, id, rank);
    if (r != ncclSuccess) {
        c->nc = nullptr;
        mm_comm_free(c);
        return mm::api_fail(MM_ERR_NCCL, "ncclCommInitRank: %s", a.GetErrorString(r));
    }
    *out = c;
    return MM_OK;
}

void mm_comm_free(mm_comm *c)
{
    if (!c)
        return;
    if (c->cs)
        cudaStreamSynchronize(c->cs);
    if (c->nc && mm::nccl().ok)
        mm::nccl().CommDestroy(c->nc);
    cudaFree(c->recv);
    if (c->ev_ready)
        cudaEventDestroy(c->ev_ready);
    if (c->ev_done)
        cudaEventDestroy(c->ev_done);
    if (c->cs)
        cudaStreamDestroy(c->cs);
    delete c;
}

}  // extern "C"
