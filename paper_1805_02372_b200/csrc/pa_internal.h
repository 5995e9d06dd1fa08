// pa_internal.h -- shared declarations of libpa's CUDA translation units.
// Product code only; nothing here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pa.h"

namespace pa {

// ---------------------------------------------------------------- route (a)
// FP64 negacyclic ("right-angle") convolution of length N = 2M real points
// via a complex DFT of length M = N1 * N2 (four-step split), DESIGN.md Sec. 4.
constexpr int kMaxStages = 24;

struct RadixPlan {
    int S;                  // number of stages
    int R[kMaxStages];      // radix of stage i (DIF order; DIT runs them reversed)
};

struct Geometry {
    uint64_t M;             // complex transform length
    uint64_t M4;            // 4*M (exponent modulus of the twist/twiddle table)
    uint32_t N1, N2, C;     // rows are N1 long (contiguous), N2 rows, C columns per CTA
    uint32_t taus;          // tau_lo table size B; tau(e) = tau_hi[e / B] * tau_lo[e % B]
    RadixPlan p1, p2;       // radix plans of N1 and N2
    uint32_t t1, t2;        // threads per CTA: strided passes (K1/K3), row pass (K2)
    uint32_t smem1, smem2;  // dynamic shared bytes: K1/K3, K2
};

struct RouteA {
    Geometry g;
    double2 *buf = nullptr;    // [N2][N1] working array (also the seed's scratch)
    double2 *spec = nullptr;   // [N2][N1] seed spectrum / M, in K2's position order
    double2 *W1 = nullptr;     // omega_N1^e, e < N1
    double2 *W2 = nullptr;     // omega_N2^e, e < N2
    double2 *theta = nullptr;  // exp(i pi b / (2 N2)), b < N2
    double2 *tau_lo = nullptr; // exp(2 pi i e / 4M), e < B
    double2 *tau_hi = nullptr; // exp(2 pi i h B / 4M), h < ceil(4M/B)
    int *rev2 = nullptr;       // DIF output position -> frequency index, N2 entries
    unsigned long long *resid = nullptr; // max |v - rint v| (as double bits)
};

// ---------------------------------------------------------------- route (b)
struct RouteB {
    uint32_t *sr = nullptr;    // reversed seed, zero padded
    uint64_t srw = 0;          // words in sr
};

}  // namespace pa

struct pa_ctx {
    int device = 0;
    uint64_t n = 0, m = 0, L = 0, off = 0;
    int route = 0;
    pa::RouteA a;
    pa::RouteB b;
    size_t ws_bytes = 0;
    uint64_t kernels_per_hash = 0;
    // pointer-validation cache (pa_hash called repeatedly with the same buffers)
    const void *ok_key = nullptr, *ok_out = nullptr;
    // staging for pa_hash_host
    uint32_t *stage_key = nullptr, *stage_out = nullptr;
};

namespace pa {

// route (a)
pa_status ra_plan(uint64_t n, uint64_t m, Geometry *g, char *err, size_t errlen);
pa_status ra_create(pa_ctx *h, const uint32_t *seed, cudaStream_t s);
pa_status ra_hash(pa_ctx *h, const uint32_t *key, uint32_t *out, uint64_t zero_words,
                  cudaStream_t s);
void ra_destroy(pa_ctx *h);

// route (b)
pa_status rb_create(pa_ctx *h, const uint32_t *seed, cudaStream_t s);
pa_status rb_hash(pa_ctx *h, const uint32_t *key, uint32_t *out, uint64_t zero_words,
                  cudaStream_t s);
void rb_destroy(pa_ctx *h);

void set_error(const char *fmt, ...);
pa_status cuda_fail(cudaError_t e, const char *what);

}  // namespace pa
