// Ghost-plane reduction of the slab decomposition:
// received ghost node rows are added into the owned rows they belong to.
// HBM-bound streaming add: 24 B moved per element.
#include "mm_internal.cuh"

namespace mm {

namespace {

__global__ void k_ghost_add(double *__restrict__ out, const double *__restrict__ recv, int64_t n)
{
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        out[i] += __ldg(recv + i);
}

}  // namespace

cudaError_t ghost_add_enqueue(double *out, const double *recv, int64_t n, cudaStream_t s)
{
    if (n <= 0)
        return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16)
        blocks = 148 * 16;
    k_ghost_add<<<(unsigned)blocks, 256, 0, s>>>(out, recv, n);
    count_launch();
    return cudaGetLastError();
}

}  // namespace mm
