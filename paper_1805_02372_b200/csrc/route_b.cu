// route_b.cu -- route (b): bit-packed direct GF(2) Toeplitz product.
//
// y[i] = XOR_j s[i-j+n-1] AND x[j]   (Eq. (1), r = uT P:88-92)
//
// With the reversed seed sr[u] = s[L-1-u] (L = n+m-1) the row i reads a forward
// window:  s[i+n-1-j] = sr[(m-1-i) + j], so
//     y[i] = parity( OR-free XOR_k  X_k AND window32(sr, o_i + 32k) ),  o_i = m-1-i,
// where X_k is key word k.  A thread owns a group of 32 consecutive offsets
// o = 32q + b (b = 0..31): for key word k every one of its 32 windows lies in
// the word pair (sr[q+k], sr[q+k+1]) and is one funnel shift (SHF) away, so the
// inner loop is SHF + LOP3 per 32 bit-products, register resident.  Threads of a
// CTA take consecutive q (coalesced seed loads), the key word is a warp-uniform
// broadcast load, and CTAs along y take disjoint key-word chunks whose partial
// parities are merged with atomicXor (order-independent, hence deterministic).
#include <algorithm>

#include "bits.cuh"
#include "pa_internal.h"

namespace pa {
namespace {

// sr word w = bits [32w, 32w+32) of reverse(s), zero past L.
__global__ void k_reverse_seed(const uint32_t *__restrict__ seed, uint64_t off, uint64_t L,
                               uint32_t *__restrict__ sr, uint64_t srw)
{
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < srw;
         w += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        if (32 * w < L) {
            // source positions off+L-1-32w-b, b = 0..31: a window starting at P0
            int64_t P0 = (int64_t)(off + L) - 32 - 32 * (int64_t)w;
            v = __brev(bits32(seed, P0, (int64_t)off, (int64_t)(off + L)));
            uint64_t valid = L - 32 * w;            // bits b < valid are real
            if (valid < 32) v &= (1u << valid) - 1u;
        }
        sr[w] = v;
    }
}

constexpr int kThreadsB = 128;

// Threads of a CTA: qb consecutive offsets q (qb = 32, 64 or 128: all of them when
// m is small) times 128/qb key-word chunks.  blockIdx.z = key of the batch.
__global__ void __launch_bounds__(kThreadsB)
k_toeplitz_bitpacked(const uint32_t *__restrict__ key, uint64_t n, uint64_t m,
                     const uint32_t *__restrict__ sr, uint32_t *__restrict__ out,
                     uint64_t Q, uint64_t KW, uint64_t KC, uint32_t qb, uint64_t key_stride,
                     uint64_t out_stride)
{
    key += blockIdx.z * key_stride;
    out += blockIdx.z * out_stride;
    const uint32_t cb = kThreadsB / qb;
    uint64_t q = blockIdx.x * (uint64_t)qb + threadIdx.x % qb;
    uint64_t k0 = (blockIdx.y * (uint64_t)cb + threadIdx.x / qb) * KC;
    uint64_t k1 = min(KW, k0 + KC);
    if (q >= Q || k0 >= k1) return;
    uint32_t acc[32];
#pragma unroll
    for (int b = 0; b < 32; ++b) acc[b] = 0u;
    const uint32_t lastmask = (n & 31) ? ((1u << (n & 31)) - 1u) : 0xFFFFFFFFu;
    uint32_t A = __ldg(sr + q + k0);
    for (uint64_t k = k0; k < k1; ++k) {
        uint32_t X = __ldg(key + k);
        if (k == KW - 1) X &= lastmask;
        uint32_t B = __ldg(sr + q + k + 1);
#pragma unroll
        for (int b = 0; b < 32; ++b) acc[b] ^= X & __funnelshift_r(A, B, b);
        A = B;
    }
    uint32_t P = 0;
#pragma unroll
    for (int b = 0; b < 32; ++b) P |= (uint32_t)(__popc(acc[b]) & 1) << b;
    // offset o = 32q + b is row i = m-1-o; valid only for o <= m-1
    uint64_t o0 = 32 * q;
    uint64_t nvalid = m - o0;                // >= 1 since q < Q = ceil(m/32)
    if (nvalid < 32) P &= (1u << nvalid) - 1u;
    // rows m-32-32q .. m-1-32q in increasing order <-> b = 31 .. 0
    uint32_t R = __brev(P);
    int64_t base = (int64_t)m - 32 - (int64_t)o0;
    if (base < 0) {
        R >>= (int)(-base);                  // dropped bits were masked rows
        if (R) atomicXor(out, R);
        return;
    }
    uint64_t wd = (uint64_t)base >> 5;
    int sh = (int)(base & 31);
    if (R << sh) atomicXor(out + wd, R << sh);
    if (sh && (R >> (32 - sh))) atomicXor(out + wd + 1, R >> (32 - sh));
}

}  // namespace

size_t rb_bytes(uint64_t n, uint64_t m) { return al256(((m + 31) / 32 + (n + 31) / 32 + 4) * 4); }

pa_status rb_create(pa_ctx *h, const uint32_t *seed, cudaStream_t s)
{
    uint64_t Q = (h->m + 31) / 32, KW = (h->n + 31) / 32;
    h->b.srw = Q + KW + 4;
    pa_status st = dev_alloc(h, (void **)&h->b.sr, rb_bytes(h->n, h->m), "route (b) reversed seed");
    if (st != PA_OK) return st;
    h->kernels_per_hash = 1;
    return rb_seed(h, seed, s);
}

pa_status rb_seed(pa_ctx *h, const uint32_t *seed, cudaStream_t s)
{
    uint64_t gw = (h->b.srw + 255) / 256;
    int grid = (int)(gw < 4096 ? gw : 4096);
    k_reverse_seed<<<grid, 256, 0, s>>>(seed, h->off, h->L, h->b.sr, h->b.srw);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "route (b) seed reversal launch");
    return PA_OK;
}

pa_status rb_hash_batch(pa_ctx *h, const uint32_t *keys, uint64_t key_stride, uint32_t *outs, uint64_t out_stride,
                        uint32_t count, uint64_t zero_words, cudaStream_t s)
{
    uint64_t Q = (h->m + 31) / 32, KW = (h->n + 31) / 32;
    cudaError_t e = cudaSuccess;
    if (zero_words)
        e = count == 1 ? cudaMemsetAsync(outs, 0, zero_words * 4, s)
                       : cudaMemset2DAsync(outs, out_stride * 4, 0, zero_words * 4, count, s);
    if (e != cudaSuccess) return cuda_fail(e, "route (b) output memset");
    const uint32_t qb = Q <= 32 ? 32 : Q <= 64 ? 64 : kThreadsB;
    const uint32_t cb = kThreadsB / qb;
    // key-word chunk so that ~8 CTAs per SM worth of (q, chunk) items exist (over the batch)
    uint64_t gx = (Q + qb - 1) / qb;
    uint64_t want_y = std::max<uint64_t>(1, (148ull * 8 * cb + gx * count - 1) / (gx * count));
    uint64_t KC = (KW + want_y - 1) / want_y;
    if (KC < 16) KC = 16;
    uint64_t gy = ((KW + KC - 1) / KC + cb - 1) / cb;
    if (gy > 65535) {
        KC = (KW + 65535 * cb - 1) / (65535 * cb);
        gy = ((KW + KC - 1) / KC + cb - 1) / cb;
    }
    prof_begin(h, 3, s);
    for (uint32_t k0 = 0; k0 < count; k0 += 65535) {
        const uint32_t c = count - k0 < 65535 ? count - k0 : 65535;
        dim3 grid((unsigned)gx, (unsigned)gy, c);
        k_toeplitz_bitpacked<<<grid, kThreadsB, 0, s>>>(keys + k0 * key_stride, h->n, h->m, h->b.sr,
                                                        outs + k0 * out_stride, Q, KW, KC, qb, key_stride,
                                                        out_stride);
    }
    prof_end(h, s);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "route (b) kernel launch");
    return PA_OK;
}

pa_status rb_hash(pa_ctx *h, const uint32_t *key, uint32_t *out, uint64_t zero_words, cudaStream_t s)
{
    return rb_hash_batch(h, key, 0, out, 0, 1, zero_words, s);
}

void rb_destroy(pa_ctx *h)
{
    dev_free(h, h->b.sr);
    h->b.sr = nullptr;
}

}  // namespace pa
