// merge.cu -- modulo-2 addition of partial hashes (Eq. (7)):
// r = sum_i K_i mod 2, i.e. the XOR of G packed m-bit vectors.  Used by the
// multi-GPU input-column split after NCCL moves the partials (NCCL has no XOR
// reduction operator).  128-bit coalesced loads, grid-stride.
#include <string.h>

#include "pa_internal.h"

namespace pa {
namespace {

__global__ void k_xor_fold(uint32_t *__restrict__ dst, const uint32_t *__restrict__ src, uint64_t words,
                           uint32_t count, uint64_t stride)
{
    const uint64_t nv = words / 4;
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv; i += step) {
        uint4 a = make_uint4(0, 0, 0, 0);
        for (uint32_t g = 0; g < count; ++g) {
            const uint4 b = __ldg(reinterpret_cast<const uint4 *>(src + g * stride) + i);
            a.x ^= b.x;
            a.y ^= b.y;
            a.z ^= b.z;
            a.w ^= b.w;
        }
        reinterpret_cast<uint4 *>(dst)[i] = a;
    }
    for (uint64_t i = 4 * nv + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words; i += step) {
        uint32_t a = 0;
        for (uint32_t g = 0; g < count; ++g) a ^= __ldg(src + g * stride + i);
        dst[i] = a;
    }
}

}  // namespace
}  // namespace pa

using namespace pa;

extern "C" pa_status pa_xor_fold(uint32_t *dst, const uint32_t *src, uint64_t words, uint32_t count,
                                 uint64_t src_stride_words, void *stream)
{
    if (!dst || !src || count == 0 || src_stride_words < words || (src_stride_words & 3) ||
        ((uintptr_t)dst & 15) || ((uintptr_t)src & 15)) {
        set_error("pa_xor_fold: need non-NULL 16-byte aligned dst/src, count >= 1, src_stride_words >= words "
                  "and a multiple of 4 (words = %llu, count = %u, stride = %llu)",
                  (unsigned long long)words, count, (unsigned long long)src_stride_words);
        return PA_ERR_INVALID_ARG;
    }
    if (words == 0) return PA_OK;
    const uint64_t blocks = (words / 4 + 255) / 256;
    k_xor_fold<<<(unsigned)(blocks < 148 * 8 ? (blocks ? blocks : 1) : 148 * 8), 256, 0, (cudaStream_t)stream>>>(
        dst, src, words, count, src_stride_words);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "pa_xor_fold launch");
    return PA_OK;
}

// ---------------------------------------------------------------- Eq. (7) over peer memory
// The multi-GPU column split's merge without a data collective: every rank's K3 leaves its
// partial hash in a buffer the other ranks have mapped (CUDA IPC over NVLink / NVSwitch), and
// rank r reads word w of every partial straight from the peers' memory -- the reduce-scatter
// and the XOR fold as one kernel (NVLink loads, 16 bytes per lane per peer).
namespace pa {
namespace {

__global__ void k_xor_fold_peers(uint32_t *__restrict__ dst, const uint32_t *const *__restrict__ srcs,
                                 uint32_t count, uint64_t w0, uint64_t words)
{
    const uint64_t nv = words / 4;  // w0 is a multiple of 4 (16-byte aligned slice)
    const uint64_t step = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv; i += step) {
        uint4 a = make_uint4(0, 0, 0, 0);
        for (uint32_t g = 0; g < count; ++g) {
            const uint4 b = __ldcv(reinterpret_cast<const uint4 *>(srcs[g] + w0) + i);  // peer memory: no caching
            a.x ^= b.x;
            a.y ^= b.y;
            a.z ^= b.z;
            a.w ^= b.w;
        }
        reinterpret_cast<uint4 *>(dst)[i] = a;
    }
    for (uint64_t i = 4 * nv + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words; i += step) {
        uint32_t a = 0;
        for (uint32_t g = 0; g < count; ++g) a ^= __ldcv(srcs[g] + w0 + i);
        dst[i] = a;
    }
}

}  // namespace
}  // namespace pa

extern "C" pa_status pa_xor_fold_peers(uint32_t *dst, const uint32_t *const *srcs, uint32_t count,
                                       uint64_t first_word, uint64_t words, void *stream)
{
    if (!dst || !srcs || count == 0 || (first_word & 3) || ((uintptr_t)dst & 15) || ((uintptr_t)srcs & 7)) {
        set_error("pa_xor_fold_peers: need non-NULL dst (16-byte aligned) and srcs, count >= 1, first_word a "
                  "multiple of 4 (count = %u, first_word = %llu)", count, (unsigned long long)first_word);
        return PA_ERR_INVALID_ARG;
    }
    if (words == 0) return PA_OK;
    const uint64_t blocks = (words / 4 + 255) / 256;
    k_xor_fold_peers<<<(unsigned)(blocks < 148 * 4 ? (blocks ? blocks : 1) : 148 * 4), 256, 0,
                       (cudaStream_t)stream>>>(dst, srcs, count, first_word, words);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "pa_xor_fold_peers launch");
    return PA_OK;
}

// Peer-mappable device buffers for the fused merge (a whole cudaMalloc allocation, so its IPC
// handle opens at its base on the peers).
extern "C" pa_status pa_peer_alloc(uint64_t bytes, void **dev_ptr)
{
    if (!dev_ptr || bytes == 0) {
        set_error("pa_peer_alloc: need bytes > 0 and a non-NULL dev_ptr");
        return PA_ERR_INVALID_ARG;
    }
    *dev_ptr = nullptr;
    cudaError_t e = cudaMalloc(dev_ptr, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *dev_ptr = nullptr;
        set_error("pa_peer_alloc: cudaMalloc of %llu bytes failed: %s", (unsigned long long)bytes,
                  cudaGetErrorString(e));
        return PA_ERR_NOMEM;
    }
    return PA_OK;
}

extern "C" pa_status pa_peer_free(void *dev_ptr)
{
    if (dev_ptr) cudaFree(dev_ptr);
    return PA_OK;
}

extern "C" pa_status pa_peer_export(const void *dev_ptr, pa_peer_handle *handle)
{
    if (!dev_ptr || !handle) {
        set_error("pa_peer_export: NULL argument");
        return PA_ERR_INVALID_ARG;
    }
    static_assert(sizeof(cudaIpcMemHandle_t) <= sizeof(handle->bytes), "IPC handle size");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void *>(dev_ptr));
    if (e != cudaSuccess) return cuda_fail(e, "pa_peer_export (cudaIpcGetMemHandle)");
    memset(handle->bytes, 0, sizeof handle->bytes);
    memcpy(handle->bytes, &h, sizeof h);
    return PA_OK;
}

extern "C" pa_status pa_peer_open(const pa_peer_handle *handle, void **dev_ptr)
{
    if (!handle || !dev_ptr) {
        set_error("pa_peer_open: NULL argument");
        return PA_ERR_INVALID_ARG;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle->bytes, sizeof h);
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "pa_peer_open (cudaIpcOpenMemHandle)");
    return PA_OK;
}

extern "C" pa_status pa_peer_close(void *dev_ptr)
{
    if (!dev_ptr) return PA_OK;
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) return cuda_fail(e, "pa_peer_close");
    return PA_OK;
}
