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
#include <atomic>

#include "bits.cuh"
#include "bulk.cuh"
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

// A CTA owns qb consecutive row words q (32 offsets o = 32q + b each, one thread per q and key
// chunk) times cb key-word chunks of KC words: its key words [k_lo, k_hi) and the seed words
// they meet, sr[q0 + k_lo, q0 + qb + k_hi + 1) -- a contiguous 16-byte-aligned superset -- are
// staged into shared memory by the bulk-copy engine (cp.async.bulk, one elected thread, an
// mbarrier transaction count), so the inner loop reads both from shared memory: the seed word of
// lane q is conflict-free (consecutive lanes, consecutive words) and the key word a broadcast.
// Per key word: two LDS, then 32 x (SHF + LOP3) on 32 register-resident accumulators.  The
// cb partial parities of a row word are XOR-reduced in shared memory; when one CTA covers all
// row words and all key words of a key (C1 and its batches: direct = 1) it writes every output
// word itself (no memset, no atomics), otherwise it atomicXors the reduced word into the
// zeroed output (order-free, deterministic).  blockIdx.z = key of the batch.
__global__ void __launch_bounds__(1024)
k_toeplitz_bitpacked(const uint32_t *__restrict__ key, uint64_t n, uint64_t m,
                     const uint32_t *__restrict__ sr, uint64_t srw4, uint32_t *__restrict__ out,
                     uint64_t Q, uint64_t KW, uint32_t KC, uint32_t qb, uint64_t key_stride,
                     uint64_t out_stride, uint32_t direct, uint64_t out_words)
{
    extern __shared__ __align__(16) uint32_t smb[];
    __shared__ __align__(8) uint64_t bar;
    key += blockIdx.z * key_stride;
    out += blockIdx.z * out_stride;
    const uint32_t T = blockDim.x, cb = T / qb, tid = threadIdx.x;
    const uint32_t qi = tid % qb, ci = tid / qb;
    const uint64_t q0 = blockIdx.x * (uint64_t)qb;
    const uint64_t k_lo = blockIdx.y * (uint64_t)cb * KC;              // multiple of 4
    const uint64_t k_hi = min((uint64_t)KW, (uint64_t)(k_lo + (uint64_t)cb * KC));
    const uint32_t kwords = (uint32_t)(k_hi - k_lo);                   // > 0
    const uint32_t kcap = (uint32_t)(((uint64_t)cb * KC + 3) / 4 * 4);
    uint32_t *skey = smb;                                              // [kcap]
    uint32_t *sseed = smb + kcap;                                      // seed superset
    const uint64_t s_lo = (q0 + k_lo) & ~3ull;
    const uint32_t sofs = (uint32_t)(q0 + k_lo - s_lo);
    const uint64_t s_hi = min((uint64_t)srw4, (uint64_t)((q0 + qb + k_hi + 1 + 3) & ~3ull));
    const uint32_t swords = (uint32_t)(s_hi - s_lo);
    uint32_t *sP = sseed + (((uint64_t)qb + kcap + 8 + 3) & ~3ull);    // [cb][qb] partial parities
    const uint32_t kbulk = kwords & ~3u;                               // the rest: plain loads (the
    if (tid == 0) {                                                    // key buffer ends at ceil(n/32))
        mbar_init(&bar, 1);
        mbar_arrive_expect_tx(&bar, 4u * (swords + kbulk));
        bulk_g2s(sseed, sr + s_lo, 4u * swords, &bar);
        if (kbulk) bulk_g2s(skey, key + k_lo, 4u * kbulk, &bar);
    }
    if (tid < kwords - kbulk) skey[kbulk + tid] = __ldg(key + k_lo + kbulk + tid);
    __syncthreads();  // barrier initialised, key tail stored
    mbar_wait(&bar, 0);
    const uint64_t q = q0 + qi;
    const uint64_t c0 = k_lo + (uint64_t)ci * KC, c1 = min((uint64_t)k_hi, (uint64_t)(c0 + KC));
    uint32_t P = 0;
    if (q < Q && c0 < c1) {
        uint32_t acc[32];
#pragma unroll
        for (int b = 0; b < 32; ++b) acc[b] = 0u;
        const uint32_t lastmask = (n & 31) ? ((1u << (n & 31)) - 1u) : 0xFFFFFFFFu;
        const uint32_t *sp = sseed + qi + sofs;  // sr[q + k] = sp[k - k_lo]
        uint32_t A = sp[c0 - k_lo];
        for (uint64_t k = c0; k < c1; ++k) {
            uint32_t X = skey[k - k_lo];
            if (k == KW - 1) X &= lastmask;
            const uint32_t B = sp[k - k_lo + 1];
#pragma unroll
            for (int b = 0; b < 32; ++b) acc[b] ^= X & __funnelshift_r(A, B, b);
            A = B;
        }
#pragma unroll
        for (int b = 0; b < 32; ++b) P |= (uint32_t)(__popc(acc[b]) & 1) << b;
        // offset o = 32q + b is row i = m-1-o; valid only for o <= m-1
        const uint64_t nvalid = m - 32 * q;  // >= 1 since q < Q = ceil(m/32)
        if (nvalid < 32) P &= (1u << nvalid) - 1u;
    }
    sP[ci * qb + qi] = P;
    __syncthreads();
    // reduce the cb chunks; Rs[qi] = brev(word): bit j <-> row m - 32 - 32q + j
    uint32_t *Rs = sP;  // in place: row 0 of sP
    if (ci == 0) {
        uint32_t R = P;
        for (uint32_t c = 1; c < cb; ++c) R ^= sP[c * qb + qi];
        R = __brev(R);
        if (!direct) {
            if (q < Q && R) {
                const int64_t base = (int64_t)m - 32 - 32 * (int64_t)q;
                if (base < 0) {
                    R >>= (int)(-base);  // dropped bits were masked rows
                    if (R) atomicXor(out, R);
                } else {
                    const uint64_t wd = (uint64_t)base >> 5;
                    const int sh = (int)(base & 31);
                    if (R << sh) atomicXor(out + wd, R << sh);
                    if (sh && (R >> (32 - sh))) atomicXor(out + wd + 1, R >> (32 - sh));
                }
            }
            return;
        }
        Rs[qi] = R;
    } else if (!direct) {
        return;
    }
    __syncthreads();
    // direct: this CTA holds every row word of the key (q0 = 0, Q <= qb) -- write out all words
    for (uint64_t w = tid; w < out_words; w += T) {
        const int64_t i0 = 32 * (int64_t)w;
        uint32_t word = 0;
        if (i0 < (int64_t)m) {
            const int64_t olo = (int64_t)m - 32 - i0, ohi = (int64_t)m - 1 - i0;  // o of rows i0+31, i0
            const int64_t qa = olo >> 5, qz = ohi >> 5;                             // floor
            for (int64_t qq = qa; qq <= qz; ++qq) {
                if (qq < 0 || qq >= (int64_t)Q) continue;
                const int64_t sh = (int64_t)m - 32 - 32 * qq - i0;                  // in (-32, 32)
                const uint32_t R = Rs[qq];
                word |= sh >= 0 ? (R << sh) : (R >> -sh);
            }
            const int64_t rem = (int64_t)m - i0;
            if (rem < 32) word &= (1u << rem) - 1u;
        }
        out[w] = word;
    }
}

}  // namespace

// reversed seed, padded to a multiple of 4 words plus 4 (the bulk copies read 16-byte supersets)
static uint64_t rb_srw4(uint64_t n, uint64_t m) { return ((m + 31) / 32 + (n + 31) / 32 + 8 + 3) / 4 * 4; }
size_t rb_bytes(uint64_t n, uint64_t m) { return al256(rb_srw4(n, m) * 4); }

pa_status rb_create(pa_ctx *h, const uint32_t *seed, cudaStream_t s)
{
    h->b.srw = rb_srw4(h->n, h->m);
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

// shared bytes of a CTA: key words, seed superset, partial parities
static size_t rb_smem(uint32_t T, uint32_t qb, uint32_t KC)
{
    const uint64_t cb = T / qb, kcap = (cb * KC + 3) / 4 * 4;
    return 4 * (kcap + ((qb + kcap + 8 + 3) & ~3ull) + cb * qb) + 16;
}

pa_status rb_hash_batch(pa_ctx *h, const uint32_t *keys, uint64_t key_stride, uint32_t *outs, uint64_t out_stride,
                        uint32_t count, uint64_t zero_words, cudaStream_t s)
{
    const uint64_t Q = (h->m + 31) / 32, KW = (h->n + 31) / 32;
    // CTA shape: qb row words (all of them when m <= 8192) x cb key-word chunks of KC words
    const uint32_t qb = Q <= 32 ? 32 : Q <= 64 ? 64 : Q <= 128 ? 128 : 256;
    const uint64_t gx = (Q + qb - 1) / qb;
    // many keys: 128 threads and >= 32 words per chunk (the loop dominates); one key: 256
    // threads and short chunks (latency).  Chunks so that ~4 CTAs per SM exist; at most 8192
    // key words staged per CTA (32 KB).
    uint32_t T = (count * gx >= 4 * 148 && qb <= 128) ? 128 : 256;
    if (count * gx < 148 && gx == 1) {
        // one (or a few) keys whose row words fit one CTA: as many chunks of >= 4 key words as
        // 1024 threads hold, so the whole hash is one short CTA (C1: 10.2 -> see DESIGN Sec. 6)
        uint32_t c = 1;
        while (c * 2 * qb <= 1024 && (uint64_t)c * 2 * 4 <= KW) c *= 2;
        T = std::max<uint32_t>(T, c * qb);
    }
    const uint32_t cb = T / qb;
    const uint64_t want_ctas = 4 * 148;
    uint64_t gy = std::max<uint64_t>(1, (want_ctas + gx * count - 1) / (gx * count));
    const uint64_t min_kc = T == 128 ? 32 : T > 256 ? 4 : 16;
    uint64_t KC = (KW + gy * cb - 1) / (gy * cb);
    if (KC < min_kc) KC = min_kc;
    KC = (KC + 3) / 4 * 4;
    if (cb * KC > 8192) KC = std::max<uint64_t>(4, 8192 / cb / 4 * 4);
    gy = (KW + cb * KC - 1) / (cb * KC);
    if (gy > 65535) return (set_error("route (b): n = %llu is beyond the bit-packed route's grid",
                                      (unsigned long long)h->n), PA_ERR_UNSUPPORTED);
    // (zero_words = 0: accumulate into the caller's output -- atomics, never plain stores)
    const uint32_t direct = gx == 1 && gy == 1 && zero_words > 0;
    const size_t smem = rb_smem(T, qb, (uint32_t)KC);
    cudaError_t e = cudaSuccess;
    if (!direct && zero_words)
        e = count == 1 ? cudaMemsetAsync(outs, 0, zero_words * 4, s)
                       : cudaMemset2DAsync(outs, out_stride * 4, 0, zero_words * 4, count, s);
    if (e != cudaSuccess) return cuda_fail(e, "route (b) output memset");
    // the shared-memory attribute is per device (a process may drive several): set once per device
    static std::atomic<uint64_t> attr_done{0};
    const uint64_t bit = h->device < 64 ? 1ull << h->device : 0;
    if (!bit || !(attr_done.load() & bit)) {
        if ((e = cudaFuncSetAttribute(k_toeplitz_bitpacked, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024)) !=
            cudaSuccess)
            return cuda_fail(e, "route (b) cudaFuncSetAttribute");
        attr_done.fetch_or(bit);
    }
    prof_begin(h, 3, s);
    for (uint32_t k0 = 0; k0 < count; k0 += 65535) {
        const uint32_t c = count - k0 < 65535 ? count - k0 : 65535;
        dim3 grid((unsigned)gx, (unsigned)gy, c);
        k_toeplitz_bitpacked<<<grid, T, smem, s>>>(keys + k0 * key_stride, h->n, h->m, h->b.sr, h->b.srw,
                                                   outs + k0 * out_stride, Q, KW, (uint32_t)KC, qb, key_stride,
                                                   out_stride, direct, zero_words);
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
