// blocked.cu -- length-compatible hashing (Sec. 3, Fig. 1, Eq. (4)-(7),
// P:103-141): when one transform of n+m-1 points is too long (device memory, or the
// planner's two-pass limit), split T into row blocks [r0, r0 + mb) and column (key)
// blocks [c0, c0 + nb).  Block (r, c) is itself a Toeplitz hash:
//     T[r0+i][c0+j] = s[(r0+i) - (c0+j) + n - 1] = s'[i - j + nb - 1],
//     s' = s[r0 + n - c0 - nb ...],
// and the row block's output is the XOR of its column blocks' outputs (Eq. (7):
// "modulo-2 addition among all the intermediate keys").  SURVEY NEXT-3.
//
// Every block has the same shape (nb, mb), both multiples of 32: the last column block's key
// bits past n are zero-padded (any seed bits may meet them, so its window is zero-padded
// where it starts before s[0]), and the last row block's rows past m are computed and
// dropped.  One handle of that shape serves all blocks: pa_set_seed rebinds it to each block's
// seed window (P:90 -- the seed is an input like the key), so nothing is created or destroyed
// per block.  The seed window of block (r0, c0) starts at bit r0 + n - c0 - nb, which is
// congruent to n mod 32 for every block: it is staged as whole words with the handle's fixed
// seed_bit_offset = n mod 32.
//
// pa_hash_blocked_host streams the key and seed from HOST memory (the paper's keys of
// 10^9-10^10 bits at 50-100 km, beyond one device's memory): block i+1's key and
// seed words move host->device on a copy stream (two staging slots) while block i is hashed,
// and every finished row block's output moves device->host the same way.
#include <stdio.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>

#include "bits.cuh"
#include "pa_internal.h"

namespace pa {
namespace {

__global__ void k_xor_into(uint32_t *__restrict__ dst, const uint32_t *__restrict__ src, uint64_t words, int first)
{
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < words;
         w += (uint64_t)gridDim.x * blockDim.x)
        dst[w] = first ? src[w] : (dst[w] ^ src[w]);
}

// zero every bit at or past `bits` of a words-long array (tail masking of staged blocks)
__global__ void k_mask_from(uint32_t *__restrict__ w, uint64_t words, uint64_t bits)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < words;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t lo = 32 * i;
        if (lo >= bits) w[i] = 0u;
        else if (bits - lo < 32) w[i] &= (1u << (bits - lo)) - 1u;
    }
}

unsigned grid_for(uint64_t words)
{
    uint64_t b = (words + 255) / 256;
    return (unsigned)(b == 0 ? 1 : (b < 4096 ? b : 4096));
}

// Block shape for a transform-length limit: (nb, mb) multiples of 32 with nb + mb - 1 <= lim,
// the one with the least transform work: k row blocks of mb = m / k rows and the longest key
// blocks that fit, work = k * ceil(n / nb) * (nb + mb), over k = 1 .. 64 (one row block whenever
// m fits with room for key blocks -- e.g. m = 10^8, lim = 1.6 * 10^8: 17 blocks of 1.6 * 10^8
// against 26 for square 8 * 10^7 blocks).
bool block_shape(uint64_t n, uint64_t m, uint64_t lim, uint64_t *nb, uint64_t *mb)
{
    const uint64_t nr = (n + 31) / 32 * 32;
    double best = 0.0;
    bool found = false;
    for (uint64_t k = 0; k <= 64; ++k) {
        // k >= 1: m split into k row blocks; k = 0: square blocks of half the limit (the only
        // shape once the limit is far below m)
        const uint64_t mbk = k ? ((m + k - 1) / k + 31) / 32 * 32 : std::min((lim / 2) / 32 * 32, (m + 31) / 32 * 32);
        if (mbk < 32 || mbk + 31 > lim) continue;
        const uint64_t nbk = std::min((lim + 1 - mbk) / 32 * 32, nr);
        if (nbk < 32) continue;
        const double work = (double)((m + mbk - 1) / mbk) * (double)((nr + nbk - 1) / nbk) * (double)(nbk + mbk);
        if (!found || work < best) {
            best = work;
            *nb = nbk;
            *mb = mbk;
            found = true;
        }
        if (k && mbk == 32) break;
    }
    return found;
}

struct Staging {
    uint64_t sw = 0, kw = 0;     // words per slot: seed window, key block
    uint32_t *seed[2] = {}, *key[2] = {};
};

}  // namespace
}  // namespace pa

using namespace pa;

// The block handle is kept between calls of the same block shape on the same device (creating a
// multi-GB handle and freeing it costs more than hashing a block); pa_hash_blocked_release frees
// it.  Calls are serialised on this cache.
static std::mutex g_bmutex;
static struct BlockCache {
    pa_handle h = nullptr;
    uint64_t nb = 0, mb = 0, off = 0;
    int device = -1;
    uint32_t *stage = nullptr;  // staging slots + accumulators (reused when large enough)
    size_t stage_bytes = 0;
    int stage_device = -1;
} g_bcache;

// The block shape for a limit and an optional device budget: the largest limit <= lim whose
// block handle + staging fit the budget (when one is given), then block_shape.
static pa_status blocked_shape_for(uint64_t n, uint64_t m, uint64_t lim, uint64_t budget, const char *who,
                                   uint64_t *nb_out, uint64_t *mb_out)
{
    auto device_bytes = [&](uint64_t L, uint64_t *nb, uint64_t *mb) -> uint64_t {
        if (!block_shape(n, m, L, nb, mb)) return ~0ull;
        pa_options o;
        pa_options_init(&o);
        o.allow_wide = 1;
        o.seed_bit_offset = n % 32;
        uint64_t ws = 0;
        if (pa_workspace_size(*nb, *mb, &o, &ws) != PA_OK) return ~0ull;
        const uint64_t sw = (n % 32 + *nb + *mb + 31) / 32 + 4, kw = *nb / 32 + 4, ow = *mb / 32 + 4;
        return ws + 2 * 4 * (sw + kw) + 3 * 4 * ow + (8u << 20);  // + headroom for the graph / tables
    };
    uint64_t nb = 0, mb = 0;
    if (budget) {
        uint64_t lo = 64, hi = std::max<uint64_t>(lim, 65);
        if (device_bytes(lo, &nb, &mb) > budget) {
            set_error("%s: device_budget_bytes = %llu cannot hold even the smallest block", who,
                      (unsigned long long)budget);
            return PA_ERR_NOMEM;
        }
        if (device_bytes(hi, &nb, &mb) <= budget) lo = hi;
        while (lo + 1 < hi) {
            const uint64_t mid = lo + (hi - lo) / 2;
            if (device_bytes(mid, &nb, &mb) <= budget) lo = mid;
            else hi = mid;
        }
        lim = lo;
    }
    if (!block_shape(n, m, lim, &nb, &mb)) {
        set_error("%s: max_block_bits = %llu is too small for 32-bit aligned blocks", who, (unsigned long long)lim);
        return PA_ERR_INVALID_ARG;
    }
    *nb_out = nb;
    *mb_out = mb;
    return PA_OK;
}

// The block loop shared by the device- and host-resident entry points.
static pa_status blocked_impl(uint64_t n, uint64_t m, const uint32_t *seed_bits, const uint32_t *key_bits,
                              uint32_t *out_bits, uint64_t lim, bool host, uint64_t budget, cudaStream_t s,
                              const char *who)
{
    uint64_t nb = 0, mb = 0;
    if (pa_status st0 = blocked_shape_for(n, m, lim, budget, who, &nb, &mb); st0 != PA_OK) return st0;
    const uint64_t KW = (n + 31) / 32, SW = (n + m - 1 + 31) / 32, OW = (m + 31) / 32;
    const uint64_t off = n % 32;
    Staging st;
    // every slot / buffer starts 16-byte aligned (multiples of 4 words)
    st.sw = ((off + nb + mb - 1 + 31) / 32 + 4 + 3) / 4 * 4;
    st.kw = (nb / 32 + 4 + 3) / 4 * 4;
    const uint64_t ow = (mb / 32 + 4 + 3) / 4 * 4;
    std::lock_guard<std::mutex> lock(g_bmutex);
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t need = 4 * (2 * (st.sw + st.kw) + 3 * ow);
    cudaError_t e = cudaSuccess;
    if (!g_bcache.stage || g_bcache.stage_device != dev || g_bcache.stage_bytes < need) {
        if (g_bcache.stage) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(g_bcache.stage_device);
            cudaFree(g_bcache.stage);  // synchronous: no earlier call's copies still use it
            cudaSetDevice(prev);
            g_bcache.stage = nullptr;
            g_bcache.stage_bytes = 0;
        }
        if ((e = cudaMalloc(&g_bcache.stage, need)) != cudaSuccess) {
            cudaGetLastError();
            g_bcache.stage = nullptr;
            set_error("%s: staging allocation failed: %s", who, cudaGetErrorString(e));
            return PA_ERR_NOMEM;
        }
        g_bcache.stage_bytes = need;
        g_bcache.stage_device = dev;
    }
    uint32_t *blk = g_bcache.stage;
    for (int i = 0; i < 2; ++i) {
        st.seed[i] = blk + i * (st.sw + st.kw);
        st.key[i] = st.seed[i] + st.sw;
    }
    uint32_t *tpart = blk + 2 * (st.sw + st.kw), *tacc[2] = {tpart + ow, tpart + 2 * ow};
    cudaStream_t cs = nullptr;
    cudaEvent_t ev_in[2] = {}, ev_free[2] = {}, ev_acc[2] = {}, ev_out[2] = {};
    pa_handle hb = nullptr;
    if (g_bcache.h && g_bcache.nb == nb && g_bcache.mb == mb && g_bcache.off == off && g_bcache.device == dev) {
        hb = g_bcache.h;
    } else if (g_bcache.h) {
        pa_destroy(g_bcache.h);
        g_bcache.h = nullptr;
        g_bcache.device = -1;
    }
    const bool fresh = hb == nullptr;
    pa_status res = PA_OK;
    auto fail = [&](pa_status r) {
        if (res == PA_OK) res = r;
        return r;
    };
    if ((e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)) != cudaSuccess) {
        fail(cuda_fail(e, who));
    } else {
        for (int i = 0; i < 2; ++i)
            if (cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_free[i], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_acc[i], cudaEventDisableTiming) != cudaSuccess ||
                cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming) != cudaSuccess)
                fail(cuda_fail(cudaGetLastError(), who));
    }
    const cudaMemcpyKind kin = host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const cudaMemcpyKind kout = host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    // stage block (r0, c0) into slot i on the copy stream: seed words from bit r0 + n - c0 - nb
    // (congruent to off mod 32; words before s[0] or past s[n+m-2] are zero) and the key words
    // [c0/32, c0/32 + nb/32) (past n zero)
    auto stage = [&](uint64_t r0, uint64_t c0, int i) -> pa_status {
        cudaError_t x = cudaSuccess;
        const int64_t w0 = ((int64_t)(r0 + n) - (int64_t)c0 - (int64_t)nb - (int64_t)off) / 32;  // exact
        const int64_t wa = std::max<int64_t>(w0, 0), wb = std::min<int64_t>(w0 + (int64_t)st.sw, (int64_t)SW);
        if (wa > w0 || wb < w0 + (int64_t)st.sw)
            x = cudaMemsetAsync(st.seed[i], 0, 4 * st.sw, cs);
        if (x == cudaSuccess && wb > wa)
            x = cudaMemcpyAsync(st.seed[i] + (wa - w0), seed_bits + wa, 4 * (wb - wa), kin, cs);
        if (x == cudaSuccess && wb > wa && (uint64_t)wb == SW) {  // bits past n+m-1 of the last seed word
            // only the words from the one holding bit n+m-1 on (masking the whole window with one
            // warp cost ~7 ms per 3 * 10^8-bit block)
            const uint64_t rel = (n + m - 1) - 32 * (uint64_t)wa, q = rel / 32;
            if (q < (uint64_t)(wb - wa))
                k_mask_from<<<1, 32, 0, cs>>>(st.seed[i] + (wa - w0) + q, (uint64_t)(wb - wa) - q, rel - 32 * q);
        }
        const uint64_t ka = c0 / 32, kb = std::min<uint64_t>(KW, ka + nb / 32);
        if (x == cudaSuccess && kb - ka < nb / 32) x = cudaMemsetAsync(st.key[i], 0, 4 * st.kw, cs);
        if (x == cudaSuccess) x = cudaMemcpyAsync(st.key[i], key_bits + ka, 4 * (kb - ka), kin, cs);
        if (x == cudaSuccess && kb == KW) {  // key bits past n: the words from the one holding bit n on
            const uint64_t q = (n - c0) / 32;
            if (q < kb - ka) k_mask_from<<<1, 32, 0, cs>>>(st.key[i] + q, kb - ka - q, n - c0 - 32 * q);
        }
        if (x == cudaSuccess) x = cudaGetLastError();
        if (x == cudaSuccess) x = cudaEventRecord(ev_in[i], cs);
        return x == cudaSuccess ? PA_OK : cuda_fail(x, who);
    };
    const uint64_t R = (m + mb - 1) / mb, Cb = (n + nb - 1) / nb;
    uint64_t b = 0;  // block counter: slot = b & 1
    if (res == PA_OK) {
        // the copy stream starts after whatever `s` already holds (the caller's inputs)
        cudaEventRecord(ev_free[0], s);
        cudaStreamWaitEvent(cs, ev_free[0], 0);
        cudaEventRecord(ev_free[1], s);
        fail(stage(0, 0, 0));
    }
    for (uint64_t r = 0; r < R && res == PA_OK; ++r) {
        const uint64_t r0 = r * mb;
        const int a = (int)(r & 1);
        if (r >= 2) cudaStreamWaitEvent(s, ev_out[a], 0);  // row block r-2's output has left tacc[a]
        for (uint64_t c = 0; c < Cb && res == PA_OK; ++c, ++b) {
            const int i = (int)(b & 1);
            // prefetch the next block into the other slot once the block that used it is done
            const uint64_t nr = c + 1 < Cb ? r : r + 1, nc = c + 1 < Cb ? c + 1 : 0;
            if (nr < R) {
                cudaStreamWaitEvent(cs, ev_free[i ^ 1], 0);
                if (fail(stage(nr * mb, nc * nb, i ^ 1)) != PA_OK) break;
            }
            cudaStreamWaitEvent(s, ev_in[i], 0);
            if (!hb) {
                pa_options o;
                pa_options_init(&o);
                o.seed_bit_offset = off;
                o.allow_wide = 1;
                if (fail(pa_create_ex(&hb, nb, mb, st.seed[i], &o, s)) != PA_OK) break;
                g_bcache.h = hb;
                g_bcache.nb = nb;
                g_bcache.mb = mb;
                g_bcache.off = off;
                g_bcache.device = dev;
            } else if (fail(pa_set_seed(hb, st.seed[i], s)) != PA_OK) {
                break;
            }
            if (fail(pa_hash(hb, st.key[i], tpart, s)) != PA_OK) break;
            cudaEventRecord(ev_free[i], s);  // slot i may be restaged
#ifdef PA_DEV
            if (dev_env("PA_BLOCKED_DEBUG")) {
                size_t fr = 0, tot = 0;
                cudaStreamSynchronize(s);
                cudaMemGetInfo(&fr, &tot);
                pa_info inf;
                pa_get_info(hb, &inf);
                fprintf(stderr, "block r=%llu/%llu c=%llu/%llu nb=%llu mb=%llu free %.3f GiB ws %.3f GiB plan %llux%llu\n",
                        (unsigned long long)r, (unsigned long long)R, (unsigned long long)c, (unsigned long long)Cb,
                        (unsigned long long)nb, (unsigned long long)mb, fr / 1073741824.0,
                        inf.workspace_bytes / 1073741824.0, (unsigned long long)inf.n1, (unsigned long long)inf.n2);
            }
#endif
            k_xor_into<<<grid_for(mb / 32), 256, 0, s>>>(tacc[a], tpart, mb / 32, c == 0 ? 1 : 0);
        }
        if (res != PA_OK) break;
        // row block r: rows [r0, r0 + mb) -> output words [r0/32, ...), the rows past m dropped
        const uint64_t words = std::min<uint64_t>(mb / 32, OW - r0 / 32);
        if (r0 + 32 * words > m) k_mask_from<<<1, 32, 0, s>>>(tacc[a] + words - 1, 1, m - (r0 + 32 * (words - 1)));
        cudaEventRecord(ev_acc[a], s);
        cudaStreamWaitEvent(cs, ev_acc[a], 0);
        if ((e = cudaMemcpyAsync(out_bits + r0 / 32, tacc[a], 4 * words, kout, cs)) != cudaSuccess) {
            fail(cuda_fail(e, who));
            break;
        }
        cudaEventRecord(ev_out[a], cs);
    }
    if (res == PA_OK && (e = cudaGetLastError()) != cudaSuccess) fail(cuda_fail(e, who));
    if (cs) {
        cudaStreamSynchronize(cs);
        cudaStreamDestroy(cs);
    }
    cudaStreamSynchronize(s);
    if (res != PA_OK && g_bcache.h) {  // a failed call does not leave a handle in an unknown state
        pa_destroy(g_bcache.h);
        g_bcache.h = nullptr;
        g_bcache.nb = g_bcache.mb = g_bcache.off = 0;
        g_bcache.device = -1;
    }
    (void)fresh;
    for (int i = 0; i < 2; ++i)
        for (cudaEvent_t ev : {ev_in[i], ev_free[i], ev_acc[i], ev_out[i]})
            if (ev) cudaEventDestroy(ev);
    return res;
}

// A block shape route (a) plans as ONE transform (a block that itself needed the in-handle
// Eq. (4) split would transform its seed windows twice).
static bool one_plan(uint64_t n, uint64_t m, uint64_t lim)
{
    uint64_t nb, mb;
    if (!block_shape(n, m, lim, &nb, &mb)) return false;
    Geometry g;
    char err[256];
    return ra_plan(nb, mb, &g, err, sizeof err, 0) == PA_OK;
}
// default block limit: among limits from the longest block route (a) plans as one transform down
// to a third of it, the one whose blocks the cost model prices cheapest in total -- blocks x
// (hash + seed transform ~ 0.57 hash, measured at C4) + a per-block fixed cost (launches, copy
// latency).  The longest block is not always the fastest: its plans tend to general kernels.
static uint64_t default_limit_search(uint64_t n, uint64_t m);
// the search plans ~80 shapes (~20 ms of host time): remembered per (n, m) for the process
static uint64_t default_limit(uint64_t n, uint64_t m)
{
    static std::mutex mu;
    static std::map<std::pair<uint64_t, uint64_t>, uint64_t> memo;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = memo.find({n, m});
        if (it != memo.end()) return it->second;
    }
    const uint64_t lim = default_limit_search(n, m);
    std::lock_guard<std::mutex> lock(mu);
    memo[{n, m}] = lim;
    return lim;
}
static uint64_t default_limit_search(uint64_t n, uint64_t m)
{
    if (one_plan(n, m, n + m - 1)) return n + m - 1;
    uint64_t lo = 64, hi = n + m - 1;
    while (lo + 1 < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (one_plan(n, m, mid)) lo = mid;
        else hi = mid;
    }
    uint64_t pick = lo;
    double best = 1e300;
    auto price = [&](uint64_t L, Geometry *g) -> bool {
        uint64_t nb, mb;
        if (L < 64 || L > lo || !block_shape(n, m, L, &nb, &mb)) return false;
        char err[256];
        if (ra_plan(nb, mb, g, err, sizeof err, 0) != PA_OK) return false;
        const double blocks = (double)((m + mb - 1) / mb) * (double)((n + nb - 1) / nb);
        const double t = blocks * (1.57 * ra_last_plan_cost() * (ra_plan_specialised(*g) ? 1.0 : 1.2) + 30e-6);
        if (const char *e = dev_env("PA_BLOCKED_DEBUG"); e && atoi(e))
            fprintf(stderr, "blocked: model %8.2f ms lim %llu -> nb %llu mb %llu plan %ux%u C=%u spec %d blocks %.0f\n",
                    t * 1e3, (unsigned long long)L, (unsigned long long)nb, (unsigned long long)mb, g->N1, g->N2, g->C,
                    (int)ra_plan_specialised(*g), blocks);
        if (t < best) {
            best = t;
            pick = L;
        }
        return true;
    };
    for (int i = 0; i < 48; ++i) {
        const uint64_t L = (uint64_t)((double)lo * std::pow(0.977, i));
        Geometry g;
        if (L < 64) break;
        if (!price(L, &g)) continue;
        // and the longest block the same plan holds (2 N1 N2 points): fewer blocks at no cost
        Geometry g2;
        price(2ull * g.N1 * g.N2, &g2);
    }
    if (const char *e = dev_env("PA_BLOCKED_DEBUG"); e && atoi(e))
        fprintf(stderr, "blocked: pick lim %llu (longest %llu)\n", (unsigned long long)pick, (unsigned long long)lo);
    return pick;
}

extern "C" pa_status pa_hash_blocked(uint64_t n, uint64_t m, const uint32_t *seed_bits,
                                     const uint32_t *key_bits, uint32_t *out_bits,
                                     uint64_t max_block_bits, void *stream)
{
    if (n == 0 || m == 0 || m > n || !seed_bits || !key_bits || !out_bits) {
        set_error("pa_hash_blocked: need 1 <= m <= n and non-NULL pointers (n = %llu, m = %llu)",
                  (unsigned long long)n, (unsigned long long)m);
        return PA_ERR_INVALID_ARG;
    }
    const uint64_t lim = max_block_bits ? max_block_bits : default_limit(n, m);
    if (lim < 64) {
        set_error("pa_hash_blocked: max_block_bits = %llu is too small (>= 64)", (unsigned long long)lim);
        return PA_ERR_INVALID_ARG;
    }
    return blocked_impl(n, m, seed_bits, key_bits, out_bits, lim, false, 0, (cudaStream_t)stream,
                        "pa_hash_blocked");
}

extern "C" pa_status pa_hash_blocked_host(uint64_t n, uint64_t m, const uint32_t *seed_host, const uint32_t *key_host,
                                          uint32_t *out_host, uint64_t max_block_bits,
                                          uint64_t device_budget_bytes, void *stream)
{
    if (n == 0 || m == 0 || m > n || !seed_host || !key_host || !out_host) {
        set_error("pa_hash_blocked_host: need 1 <= m <= n and non-NULL pointers (n = %llu, m = %llu)",
                  (unsigned long long)n, (unsigned long long)m);
        return PA_ERR_INVALID_ARG;
    }
    uint64_t lim = max_block_bits ? max_block_bits : default_limit(n, m);
    if (lim < 64) {
        set_error("pa_hash_blocked_host: max_block_bits = %llu is too small (>= 64)", (unsigned long long)lim);
        return PA_ERR_INVALID_ARG;
    }
    return blocked_impl(n, m, seed_host, key_host, out_host, lim, true, device_budget_bytes, (cudaStream_t)stream,
                        "pa_hash_blocked_host");
}

extern "C" pa_status pa_blocked_plan(uint64_t n, uint64_t m, uint64_t max_block_bits, uint64_t device_budget_bytes,
                                     uint64_t *nb, uint64_t *mb, uint64_t *blocks)
{
    if (n == 0 || m == 0 || m > n || !nb || !mb || !blocks) {
        set_error("pa_blocked_plan: need 1 <= m <= n and non-NULL outputs (n = %llu, m = %llu)",
                  (unsigned long long)n, (unsigned long long)m);
        return PA_ERR_INVALID_ARG;
    }
    const uint64_t lim = max_block_bits ? max_block_bits : default_limit(n, m);
    if (lim < 64) {
        set_error("pa_blocked_plan: max_block_bits = %llu is too small (>= 64)", (unsigned long long)lim);
        return PA_ERR_INVALID_ARG;
    }
    pa_status st = blocked_shape_for(n, m, lim, device_budget_bytes, "pa_blocked_plan", nb, mb);
    if (st != PA_OK) return st;
    *blocks = ((m + *mb - 1) / *mb) * ((n + *nb - 1) / *nb);
    return PA_OK;
}

extern "C" void pa_hash_blocked_release(void)
{
    std::lock_guard<std::mutex> lock(g_bmutex);
    int prev = 0;
    cudaGetDevice(&prev);
    if (g_bcache.h) pa_destroy(g_bcache.h);  // switches to the handle's device itself
    if (g_bcache.stage) {
        cudaSetDevice(g_bcache.stage_device);
        cudaFree(g_bcache.stage);
    }
    cudaSetDevice(prev);
    g_bcache = BlockCache{};
}
