// seed_layout.cu -- pa_seed_from_paper_eq1: the paper's Eq. (1) seed order -> this
// library's diagonal order (reading R2).
//
// Eq. (1) fills T's first column with t_0 .. t_{n-1} top-down and its
// first row with t_0, t_n, .., t_{n+l-2}: T_{i,j} = t_{i-j} (i >= j), t_{j-i+n-1} (j > i),
// with the hash r = u T.  As y = T' x with T'[a][b] = T_{b,a} = s[a-b+n-1]:
//   b >= a:  t_{b-a}      = s[n-1-(b-a)]   -> s[u] = t_{n-1-u}  for u <  n
//   a >  b:  t_{a-b+n-1}  = s[a-b+n-1]     -> s[u] = t_u        for u >= n
// so the conversion reverses the first n seed bits and keeps the rest.
#include "pa_internal.h"

namespace pa {
namespace {

// 32 bits of src starting at bit p (p may be negative); bits outside [0, 32 nw) read 0
__device__ __forceinline__ uint32_t window32(const uint32_t *__restrict__ src, int64_t p, uint64_t nw)
{
    const int64_t w = p >= 0 ? p / 32 : -((31 - p) / 32);
    const int sh = (int)(p - 32 * w);
    const uint32_t lo = (w >= 0 && (uint64_t)w < nw) ? __ldg(src + w) : 0u;
    const uint32_t hi = (w + 1 >= 0 && (uint64_t)(w + 1) < nw) ? __ldg(src + w + 1) : 0u;
    return sh ? (lo >> sh) | (hi << (32 - sh)) : lo;
}

__global__ void k_seed_from_eq1(uint32_t *__restrict__ s, const uint32_t *__restrict__ t, uint64_t n, uint64_t L,
                                uint64_t nw)
{
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nw; w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t u0 = 32 * w;
        const uint32_t direct = window32(t, (int64_t)u0, nw);                 // bit j = t[u0 + j]
        const uint32_t rev = __brev(window32(t, (int64_t)n - 32 - (int64_t)u0, nw));  // bit j = t[n-1-u0-j]
        const uint32_t low = n <= u0 ? 0u : (n - u0 >= 32 ? ~0u : (1u << (n - u0)) - 1u);  // u0 + j < n
        uint32_t v = (rev & low) | (direct & ~low);
        if (L - u0 < 32) v &= (1u << (L - u0)) - 1u;  // bits >= n+m-1 written 0
        s[w] = v;
    }
}

}  // namespace
}  // namespace pa

using namespace pa;

extern "C" pa_status pa_seed_from_paper_eq1(uint32_t *s_bits, const uint32_t *t_bits, uint64_t n, uint64_t m,
                                            void *stream)
{
    if (!s_bits || !t_bits || n == 0 || m == 0 || ((uintptr_t)s_bits & 15) || ((uintptr_t)t_bits & 15)) {
        set_error("pa_seed_from_paper_eq1: need non-NULL 16-byte aligned s_bits/t_bits and n, m >= 1 "
                  "(n = %llu, m = %llu)", (unsigned long long)n, (unsigned long long)m);
        return PA_ERR_INVALID_ARG;
    }
    const uint64_t L = n + m - 1, nw = (L + 31) / 32;
    const uintptr_t a0 = (uintptr_t)s_bits, b0 = (uintptr_t)t_bits;
    if (a0 < b0 + 4 * nw && b0 < a0 + 4 * nw) {
        set_error("pa_seed_from_paper_eq1: s_bits and t_bits overlap");
        return PA_ERR_INVALID_ARG;
    }
    const uint64_t blocks = (nw + 255) / 256;
    k_seed_from_eq1<<<(unsigned)(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, (cudaStream_t)stream>>>(
        s_bits, t_bits, n, L, nw);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "pa_seed_from_paper_eq1 launch");
    return PA_OK;
}
