// bits.cuh -- LSB-first bit-string access for libpa kernels (product code).
#pragma once
#include <stdint.h>

namespace pa {

// Bits [P, P+32) of the LSB-first string held in uint32 words `w`, where only
// positions in [lo, hi) are valid (others read as 0 and their words are never
// touched).  P may be negative.
__device__ __forceinline__ uint32_t bits32(const uint32_t *__restrict__ w, int64_t P,
                                           int64_t lo, int64_t hi)
{
    if (P >= hi || P + 32 <= lo) return 0u;
    int64_t q = (P >= 0) ? (P >> 5) : -((-P + 31) >> 5);  // floor(P / 32)
    int r = (int)(P - q * 32);
    int64_t wlo = lo >> 5, whi = (hi - 1) >> 5;           // readable word range
    uint32_t w0 = (q >= wlo && q <= whi) ? __ldg(w + q) : 0u;
    uint32_t w1 = (q + 1 >= wlo && q + 1 <= whi) ? __ldg(w + q + 1) : 0u;
    uint32_t v = __funnelshift_r(w0, w1, r);
    // mask positions < lo and >= hi
    if (P < lo) {
        int64_t d = lo - P;                 // 1..31
        v &= 0xFFFFFFFFu << d;
    }
    if (P + 32 > hi) {
        int64_t k = hi - P;                 // 1..31
        v &= (k >= 32) ? 0xFFFFFFFFu : ((1u << k) - 1u);
    }
    return v;
}

}  // namespace pa
