// merge.cu -- modulo-2 addition of partial hashes (Eq. (7)):
// r = sum_i K_i mod 2, i.e. the XOR of G packed m-bit vectors.  Used by the
// multi-GPU input-column split after NCCL moves the partials (NCCL has no XOR
// reduction operator).  128-bit coalesced loads, grid-stride.
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
