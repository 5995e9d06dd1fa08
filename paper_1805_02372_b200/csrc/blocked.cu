// blocked.cu -- length-compatible hashing (Sec. 3, Fig. 1, Eq. (4)-(7),
// P:103-141): when one transform of n+m-1 points is too long (memory, or the
// planner's two-pass limit), split T into row blocks [r0, r1) and column (key)
// blocks [c0, c1).  Block (r, c) is itself a Toeplitz hash:
//     T[r0+i][c0+j] = s[(r0+i) - (c0+j) + n - 1] = s'[i - j + n_b - 1],
//     s' = s[r0 + n - c1 ...],  n_b = c1 - c0,
// and the row block's output is the XOR of its column blocks' outputs (Eq. (7):
// "modulo-2 addition among all the intermediate keys").  SURVEY NEXT-3.
#include "bits.cuh"
#include "pa_internal.h"

namespace pa {
namespace {

// dst word w = bits [off + 32w, off + 32w + 32) of src, bits at or past off + nbits zero
__global__ void k_shift_copy(const uint32_t *__restrict__ src, uint64_t off, uint64_t nbits,
                             uint32_t *__restrict__ dst, uint64_t words)
{
    const int64_t lo = (int64_t)off, hi = (int64_t)(off + nbits);
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
         w += (uint64_t)gridDim.x * blockDim.x)
        dst[w] = bits32(src, lo + 32 * (int64_t)w, lo, hi);
}

__global__ void k_xor_into(uint32_t *__restrict__ dst, const uint32_t *__restrict__ src, uint64_t words, int first)
{
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
         w += (uint64_t)gridDim.x * blockDim.x)
        dst[w] = first ? src[w] : (dst[w] ^ src[w]);
}

unsigned grid_for(uint64_t words)
{
    uint64_t b = (words + 255) / 256;
    return (unsigned)(b == 0 ? 1 : (b < 4096 ? b : 4096));
}

}  // namespace
}  // namespace pa

using namespace pa;

extern "C" pa_status pa_hash_blocked(uint64_t n, uint64_t m, const uint32_t *seed_bits,
                                     const uint32_t *key_bits, uint32_t *out_bits,
                                     uint64_t max_block_bits, void *stream)
{
    if (n == 0 || m == 0 || m > n || !seed_bits || !key_bits || !out_bits) {
        set_error("pa_hash_blocked: need 1 <= m <= n and non-NULL pointers (n = %llu, m = %llu)",
                  (unsigned long long)n, (unsigned long long)m);
        return PA_ERR_INVALID_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    // default block limit: the whole product if one handle can plan it, else the
    // longest transform the planner accepts (binary search over n' + m' - 1)
    uint64_t lim = max_block_bits;
    if (lim == 0) {
        pa_info info;
        if (pa_plan(n, m, &info) == PA_OK) {
            lim = n + m - 1;
        } else {
            uint64_t lo = 64, hi = n + m - 1;
            while (lo + 1 < hi) {
                const uint64_t mid = lo + (hi - lo) / 2;
                if (pa_plan(mid, 1, &info) == PA_OK) lo = mid;
                else hi = mid;
            }
            lim = lo;
        }
    }
    if (lim < 64) {
        set_error("pa_hash_blocked: max_block_bits = %llu is too small (>= 64)", (unsigned long long)lim);
        return PA_ERR_INVALID_ARG;
    }
    // row blocks of m_b bits (whole uint32 words when there is more than one), column
    // blocks of n_b key bits, n_b + m_b - 1 <= lim (Eq. (4): blocks of the key; the rows
    // too "if the length of final secret keys is long")
    uint64_t mb = m, nb;
    if (m + 31 > lim / 2) mb = ((lim / 2) / 32) * 32;
    if (mb == 0) mb = 32;
    nb = lim + 1 - mb;
    if (nb > n) nb = n;
    const uint64_t kwords = (nb + 31) / 32 + 4;
    const uint64_t owords = (mb + 31) / 32 + 4;
    uint32_t *tkey = nullptr, *tout = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&tkey, kwords * 4)) != cudaSuccess || (e = cudaMalloc(&tout, owords * 4)) != cudaSuccess) {
        if (tkey) cudaFree(tkey);
        set_error("pa_hash_blocked: scratch allocation failed: %s", cudaGetErrorString(e));
        return PA_ERR_NOMEM;
    }
    pa_status st = PA_OK;
    for (uint64_t r0 = 0; r0 < m && st == PA_OK; r0 += mb) {
        const uint64_t r1 = (r0 + mb < m) ? r0 + mb : m;
        const uint64_t rw = (r1 - r0 + 31) / 32;
        bool first = true;
        for (uint64_t c0 = 0; c0 < n && st == PA_OK; c0 += nb) {
            const uint64_t c1 = (c0 + nb < n) ? c0 + nb : n;
            const uint64_t ng = c1 - c0;
            k_shift_copy<<<grid_for((ng + 31) / 32), 256, 0, s>>>(key_bits, c0, ng, tkey, (ng + 31) / 32);
            pa_options o;
            pa_options_init(&o);
            o.seed_bit_offset = r0 + n - c1;
            o.allow_wide = 1;
            pa_handle hb = nullptr;
            st = pa_create_ex(&hb, ng, r1 - r0, seed_bits, &o, stream);
            if (st != PA_OK) break;
            st = pa_hash(hb, tkey, tout, stream);
            if (st == PA_OK) {
                k_xor_into<<<grid_for(rw), 256, 0, s>>>(out_bits + r0 / 32, tout, rw, first ? 1 : 0);
                first = false;
            }
            pa_destroy(hb);
        }
    }
    if (st == PA_OK && (e = cudaGetLastError()) != cudaSuccess) st = cuda_fail(e, "pa_hash_blocked launches");
    cudaStreamSynchronize(s);
    cudaFree(tkey);
    cudaFree(tout);
    return st;
}
