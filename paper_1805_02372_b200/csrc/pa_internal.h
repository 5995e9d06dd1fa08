// pa_internal.h -- shared declarations of libpa's CUDA translation units.
// Product code only; nothing here is shared with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "../../include/pa.h"
#include "fft_core.cuh"

namespace pa {

// Developer overrides (plan / kernel-variant experiments, tools/dev/) exist only in a PA_DEV
// build (PA_DEV=1 python paper_1805_02372_b200/build.py); the product library ignores the
// environment.
#ifdef PA_DEV
inline const char *dev_env(const char *k) { return getenv(k); }
#else
inline const char *dev_env(const char *) { return nullptr; }
#endif

// ---------------------------------------------------------------- route (a)
// FP64 negacyclic ("right-angle") convolution of length N = 2M real points
// via a complex DFT of length M = N1 * N2 (four-step split), DESIGN.md Sec. 4.
struct Geometry {
    uint64_t M;             // complex transform length
    uint32_t N1, N2;        // rows are N1 long (contiguous), N2 rows
    uint32_t C, logC;       // columns per CTA in the strided passes (power of two <= 16)
    uint32_t C3, logC3;     // K3's column groups (C, or C / 2 when that fits two CTAs per SM)
    uint32_t t3, tile3, smem3;  // K3's threads / tile / shared bytes for C3
    uint32_t pfs;           // K2: L2 prefetch of the CTA's own spectrum row (one CTA per SM)
    uint32_t k1gout;        // K1's last stage stores to global directly when C >= k1gout
    uint32_t ntb;           // K1's first stage from the key bits: 2^R0 x R0 table entries (0 = off)
    uint32_t k0rb, k0cb;    // K0 tile: rows x columns per CTA
    FftPlan f1, f2;         // stage plans of N1 (row pass) and N2 (strided passes)
    uint32_t t1, t2;        // threads per CTA: strided passes (K1/K3), row pass (K2)
    uint32_t t2one;         // K2's threads when its grid is at most one CTA per SM (route_a.cu k2_threads)
    uint32_t tile1, tile2;  // padded tile sizes in double2 (tables follow the tile)
    uint32_t smem1, smem2;  // dynamic shared bytes: K1/K3, K2
    uint32_t kbw;           // K0 bit-stream words per column group
    uint32_t pf2;           // K2: L2 prefetch distance in rows (0 = off)
    uint32_t lr;            // K2 -> K3 array: rows in blocks of 2^lr (route_a.cu wrow / wcol)
    bool k3t;               // K3 as the persistent TMEM-staged k3t_inv_columns (opt-in)
    uint32_t k1p_kmax;      // K1 as the persistent TMEM write-behind k1p_fwd_columns: last-stage
                            // butterflies per thread (1 or 2); 0 = plain k1_fwd_columns
    uint32_t smem1p;        // K1P dynamic shared bytes (K1's + a second key-bit buffer)
    uint32_t k1p_t;         // K1P threads per CTA
    uint32_t k1p_tcols;     // K1P TMEM columns per CTA (512: one CTA per SM, 256: two)
    uint32_t k1p_piece;     // K1P drain piece: outputs per TMEM load (2, 4, 8)
    uint32_t k3parts;       // K3 staged tile loaded in parts, the first inverse stage per part
    bool k2fresh;           // pa_hash_fresh_batch fuses the seeds' forward half into K2 (k2_rows_t kFresh)
    double2 *fout;          // kFresh launches: key fkey's spectrum row also goes to fout (the handle's)
    uint32_t fkey;
    int k2shape;            // K2 as k2_rows_t<R0, R1, NS> (index into route_a.cu kK2), 0: general k2_rows
    int k13;                // K1/K3 instantiation (route_a.cu kK13), 0: general
};

// a route-(a) plan: rows of N1 points, N2 rows, C columns per K1 CTA
struct PlanChoice {
    uint32_t N1 = 0, N2 = 0, C = 0;
};

struct RouteTables {
    double2 *W1lo, *W1hi;   // omega_N1^e = W1hi[e >> 6] * W1lo[e & 63]
    double2 *W2lo, *W2hi;   // omega_N2^e
    double2 *thlo, *thhi;   // theta_b = exp(i pi b / (2 N2)) = zeta^{N1 b}, two-level
    uint32_t *rev2;         // K1 DIF output position p -> frequency index k_b
    double2 *rho;           // [N2][64 + N1/64]: row p's two-level table of rho = e^{2 pi i (1-4k_b)/4M}
    double2 *tb;            // [2^R0][R0]: T[p][k] = sum_{r in p} e^{i pi r (1 - 4k) / 2R0} (K1 first stage)
};

struct RouteA {
    Geometry g;
    char *pblk = nullptr;      // persistent block: spec, tables, rev2, resid
    char *wblk = nullptr;      // work block: buf, kb for `cap` keys
    double2 *buf = nullptr;    // [N2][N1] working array, row-major (also the seed's scratch)
    double2 *buf2 = nullptr;   // K2's output for K3: == buf, or the row-block layout (g.lr > 0)
    double2 *spec = nullptr;   // [N2][N1] seed spectrum / M, in K2's position order
    double2 *tables = nullptr; // backing store of T's double2 tables
    RouteTables T{};
    unsigned long long *resid = nullptr; // max |v - rint v| (as double bits)
    uint32_t *kb = nullptr;    // K0 output: per-column-group bit streams of the input
    uint32_t cap = 0;          // keys the work buffers (buf, kb) hold
    uint64_t wgen = 0;         // bumped whenever the work buffers move (cached host graphs check it)
    bool shared_w = false;     // work block borrowed from the first column block (not owned)
    double2 *fspec = nullptr;  // pa_hash_fresh_batch: one spectrum per key of a chunk
    uint32_t fcap = 0;         // keys fspec holds
};

// ---------------------------------------------------------------- route (b)
struct RouteB {
    uint32_t *sr = nullptr;    // reversed seed, zero padded
    uint64_t srw = 0;          // words in sr
};

}  // namespace pa

namespace pa {
// Caller-owned device memory (pa_create_ws): a bump allocator shared by a handle
// and its column-block sub-handles.  Without one, libpa cudaMallocs.
struct Arena {
    char *base = nullptr;
    size_t size = 0, used = 0;
};
inline size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

// launch-bracketing CUDA events for pa_profile_* (kernel k = index into names)
struct Profiler {
    bool on = false;
    static constexpr int kKernels = 8;
    const char *names[kKernels] = {"k1_fwd_columns", "k2_rows", "k3_inv_columns",
                                   "k_toeplitz_bitpacked", "k0_bits_transpose", "", "", ""};
    struct Pending { int k; cudaEvent_t e0, e1; };
    Pending *pend = nullptr;
    int npend = 0, cap = 0;
    cudaEvent_t *pool = nullptr;
    int npool = 0, poolcap = 0;
    uint64_t launches[kKernels] = {};
    double total_ms[kKernels] = {};
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
    pa::Profiler prof;
    // staging for pa_hash_host (one block: key words, then output words)
    char *stage_blk = nullptr;
    uint32_t *stage_key = nullptr, *stage_out = nullptr;
    // staging for pa_hash_host_batch (cudaMalloc, grown on demand; never in a workspace)
    char *bstage = nullptr;
    size_t bstage_bytes = 0;
    // pa_hash_host_batch pipeline: copies on their own stream, overlapped with the hashes
    cudaStream_t cstream = nullptr;
    cudaEvent_t pev[5] = {};  // h2d[2], comp[2], start/done
    // device memory: the caller's workspace (nullptr: cudaMalloc)
    pa::Arena *arena = nullptr;
    bool own_arena = false;
    uint32_t batch_opt = 0;  // pa_options.batch_keys
    // Eq. (4) column split (pa_options.max_transform_len): one sub-handle per key block
    pa_ctx *parent = nullptr;
    pa_ctx **sub = nullptr;
    uint64_t *sub_c0 = nullptr;  // first key bit of each block (multiple of 128)
    uint32_t nsub = 0;
    uint64_t max_len = 0;        // pa_options.max_transform_len (route (a) planning cap)
    pa::PlanChoice force;        // a measured plan (PA_PLAN_MEASURE) replacing the model's
    bool has_force = false;
    char *share_w = nullptr;     // column blocks 1..: the first block's work block, if large enough
    size_t share_w_bytes = 0;
    // pa_hash_host as one CUDA graph (H2D, kernels, D2H); host pointers patched per call
    cudaGraph_t host_graph = nullptr;
    cudaGraphExec_t host_exec = nullptr;
    cudaGraphNode_t h2d_node = nullptr, d2h_node = nullptr;
    int host_copy = 0;  // how the graph moves the key / output: 1 copy engines, 2 copy kernels (mapped pages)
    const void *g_key_host = nullptr;
    void *g_out_host = nullptr;
    const void *g_key_dev = nullptr;  // mapped device addresses the graph's copy kernels use
    void *g_out_dev = nullptr;
    uint64_t g_wgen = 0;              // work-buffer generation the graph was captured with
    // replaced device blocks, freed once the stream that last used them passes an event
    // (stream-ordered reallocation instead of a device-wide synchronisation)
    static constexpr int kGrave = 8;
    void *grave[kGrave] = {};
    cudaEvent_t grave_ev[kGrave] = {};
    int ngrave = 0;
};

namespace pa {

// route (a)
// max_len: cap on the real transform length 2 M (0 = none), pa_options.max_transform_len
pa_status ra_plan(uint64_t n, uint64_t m, Geometry *g, char *err, size_t errlen, uint64_t max_len = 0,
                  const PlanChoice *force = nullptr);
// the cost model's distinct candidate plans, cheapest first (PA_PLAN_MEASURE)
double ra_last_plan_cost();
bool ra_plan_specialised(const Geometry &g);
int ra_plan_candidates(uint64_t n, uint64_t m, uint64_t max_len, PlanChoice *out, int max);
pa_status ra_create(pa_ctx *h, const uint32_t *seed, cudaStream_t s);
pa_status ra_seed(pa_ctx *h, const uint32_t *seed, cudaStream_t s);
pa_status ra_hash(pa_ctx *h, const uint32_t *key, uint32_t *out, uint64_t zero_words,
                  cudaStream_t s);
pa_status ra_hash_batch(pa_ctx *h, const uint32_t *keys, uint64_t key_stride, uint32_t *outs,
                        uint64_t out_stride, uint32_t count, uint64_t zero_words, cudaStream_t s,
                        const double2 *spec = nullptr, uint64_t spec_stride = 0, bool fresh = false);
pa_status ra_fresh_batch(pa_ctx *h, const uint32_t *seeds, uint64_t seed_stride, const uint32_t *keys,
                         uint64_t key_stride, uint32_t *outs, uint64_t out_stride, uint32_t count,
                         uint64_t zero_words, cudaStream_t s);
uint32_t ra_batch_keys(const pa_ctx *h);
void ra_destroy(pa_ctx *h);

// route (b)
pa_status rb_create(pa_ctx *h, const uint32_t *seed, cudaStream_t s);
pa_status rb_seed(pa_ctx *h, const uint32_t *seed, cudaStream_t s);
pa_status rb_hash(pa_ctx *h, const uint32_t *key, uint32_t *out, uint64_t zero_words,
                  cudaStream_t s);
pa_status rb_hash_batch(pa_ctx *h, const uint32_t *keys, uint64_t key_stride, uint32_t *outs, uint64_t out_stride,
                        uint32_t count, uint64_t zero_words, cudaStream_t s);
void rb_destroy(pa_ctx *h);

size_t ra_persist_bytes(const Geometry &g);
size_t ra_work_bytes(const Geometry &g, uint32_t cap);
size_t rb_bytes(uint64_t n, uint64_t m);

// device memory from the handle's arena or cudaMalloc (dev_free is a no-op for arena memory)
pa_status dev_alloc(pa_ctx *h, void **p, size_t bytes, const char *what);
void dev_free(pa_ctx *h, void *p);
// free p (cudaMalloc'ed) after the work enqueued on s so far; reap frees what has passed
void defer_free(pa_ctx *h, void *p, cudaStream_t s);
void reap(pa_ctx *h, bool wait);

void set_error(const char *fmt, ...);
// bracket one kernel launch with profiling events (no-ops unless enabled)
void prof_begin(pa_ctx *h, int k, cudaStream_t s);
void prof_end(pa_ctx *h, cudaStream_t s);
pa_status cuda_fail(cudaError_t e, const char *what);

}  // namespace pa
