/*
 * pa.h -- C ABI of libpa: bit-exact Toeplitz-hash privacy amplification on
 * NVIDIA B200 (sm_100a).
 *
 * The operation (PAPER.md = arXiv 1805.02372, lines cited as P:L):
 *   Alice draws a uniform seed of n+l-1 bits, builds the Toeplitz matrix T
 *   from it and computes r = u T; Bob computes the same with his copy of the
 *   corrected key (Sec. 2.3 Steps 1-2).  T is diagonal-constant
 *   (Sec. 2.1, Eq. (1)) and need not be square.  Written as a
 *   matrix-vector product over GF(2) with m = l output bits:
 *
 *       y[i] = XOR_{j=0}^{n-1} s[i - j + n - 1] AND x[j],   0 <= i < m,
 *
 *   i.e. T[i][j] = s[i-j+n-1] (readings R1, R2).  Equivalently y
 *   is the window [n-1, n+m-1) of the integer convolution x * s reduced
 *   mod 2 -- the paper's Sec. 3 Step 3 "results of IFFT from the nth to
 *   (n+k-1)th".
 *
 * Bit strings: LSB-first.  Bit b of a string lives in uint32 word b/32 at
 * bit position b%32 (identical bits to uint64 word b/64, bit b%64, and to
 * bytes, on little-endian).  Lengths are always in bits.
 *
 * Memory: every key/seed/out pointer of pa_create... and pa_hash... is a DEVICE
 * pointer on the handle's device (e.g. a torch CUDA tensor's data_ptr()),
 * 16-byte aligned.  Host pointers are rejected with PA_ERR_INVALID_ARG.
 * pa_hash_host is the one entry point that takes HOST buffers.
 *
 * Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default
 * stream).  pa_create... and pa_hash... only enqueue work; results are ready
 * when the stream reaches them.  One hash in flight per handle (the handle
 * owns scratch); use one handle per stream for concurrency.
 *
 * Errors: every call returns a pa_status; no C++ exception crosses the ABI.
 * pa_last_error() returns a thread-local message naming the offending field
 * and values of the most recent failing call on this thread.
 */
#ifndef PA_H
#define PA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PA_VERSION 100u /* 1.0.0 */

typedef struct pa_ctx *pa_handle;

typedef enum pa_status {
    PA_OK = 0,
    PA_ERR_INVALID_ARG = 1, /* n == 0, m == 0, m > n, NULL/unaligned/host pointer, bad option */
    PA_ERR_UNSUPPORTED = 2, /* lengths beyond what the chosen route can plan */
    PA_ERR_NOMEM = 3,       /* device allocation failed */
    PA_ERR_CUDA = 4,        /* a CUDA runtime call or launch failed (message has the CUDA error) */
    PA_ERR_PRECISION = 5    /* FP64 route: max |v - rint(v)| over the output window exceeded
                               PA_RESIDUAL_LIMIT (never expected; see DESIGN.md error bound) */
} pa_status;

/* Route (a): exact convolution by an FP64 transform of length N >= n+m-1
 * with a proven < 0.5 rounding bound.
 * Route (b): bit-packed direct GF(2) product (AND/XOR/popcount), O(n m).
 * AUTO picks (b) for small n*m and (a) otherwise. */
typedef enum pa_route {
    PA_ROUTE_AUTO = 0,
    PA_ROUTE_TRANSFORM = 1,
    PA_ROUTE_BITPACKED = 2
} pa_route;

/* Arithmetic of route (a)'s transform (SURVEY 8(b) "Create").  FP64 is the one built: an
 * FP64 complex transform with a proven < 0.5 rounding bound.  The
 * number-theoretic transforms are not built -- an NTT over a 32-bit prime costs ~190 integer
 * operations per real point and does not beat FP64 on B200 -- and are
 * rejected with PA_ERR_UNSUPPORTED naming the field. */
typedef enum pa_arith {
    PA_ARITH_AUTO = 0,
    PA_ARITH_FP64 = 1,
    PA_ARITH_NTT32 = 2,
    PA_ARITH_NTT64 = 3
} pa_arith;

/* How route (a) picks its transform plan (N1 x N2 split, column-group width).  MODEL: the
 * planner's cost model (host-only, what pa_plan reports).  MEASURE: the model's best few
 * candidates are built and timed on the device at create (FFTW-style), the fastest kept and
 * remembered per (n, m, max_transform_len, device) for the life of the process; create then
 * synchronises `stream`.  Ignored by route (b), split handles and caller workspaces. */
typedef enum pa_plan_mode {
    PA_PLAN_MODEL = 0,
    PA_PLAN_MEASURE = 1
} pa_plan_mode;

#define PA_RESIDUAL_LIMIT 0.25

typedef struct pa_options {
    uint32_t struct_size;     /* sizeof(pa_options); set by pa_options_init */
    int32_t route;            /* pa_route */
    uint64_t seed_bit_offset; /* the handle uses seed bits [off, off+n+m-1) of the
                                 caller's seed buffer (row/column shards) */
    uint32_t allow_wide;      /* 1 = accept m > n (column shards of the Eq. (4) split,
                                 P:107-110, have n_g < m); default 0 keeps 1 <= m <= n */
    uint32_t batch_keys;      /* keys per launch in pa_hash_batch (0 = library choice).  With
                                 a caller workspace (pa_create_ws), and for the column blocks of
                                 a split handle, it fixes the per-key work buffers: 0 means 1 */
    uint64_t max_transform_len; /* route (a): 0 = no limit.  Otherwise the key is cut into
                                 column blocks (Eq. (4)) so that no block's real
                                 transform length exceeds this; each block is hashed on its
                                 own seed window (offset n - n_g - c0) and the partial outputs
                                 are XOR-merged in place (Eq. (7)).  Blocks start at
                                 multiples of 128 key bits.  PA_ERR_UNSUPPORTED if even a
                                 128-bit block's transform (>= 128 + m - 1) exceeds it.  Ignored
                                 by route (b).  With 0, pa_create splits by itself when n + m is
                                 beyond one transform (~3.3e8 bits; pa_plan reports the blocks),
                                 at the block length the cost model prices cheapest */
    int32_t arith;            /* pa_arith: AUTO or FP64 (route (a)); NTT32 / NTT64 -> PA_ERR_UNSUPPORTED */
    int32_t device;           /* CUDA device of the handle: -1 (pa_options_init's default) = the
                                 caller's current device at create; >= 0 = that device.  Every
                                 later call on the handle runs on it (the library switches to it
                                 for the call and back); seed, keys, outputs and workspace must
                                 live there and `stream` must belong to it */
    uint32_t plan_mode;       /* pa_plan_mode: MODEL (default) or MEASURE */
} pa_options;

/* Runtime facts about a handle (all lengths in bits or elements). */
typedef struct pa_info {
    uint64_t n, m;            /* key bits, output bits */
    int32_t route;            /* PA_ROUTE_TRANSFORM or PA_ROUTE_BITPACKED */
    int32_t device;
    uint64_t transform_len;   /* route (a): real transform length N = 2*M (0 for route b) */
    uint64_t n1, n2;          /* route (a): complex length M = n1 * n2 (row x column split) */
    uint64_t cols_per_cta;    /* route (a): columns per CTA in the strided passes */
    uint64_t workspace_bytes; /* device bytes owned by the handle */
    uint64_t kernels_per_hash;/* kernel launches enqueued by one pa_hash */
    uint64_t column_blocks;   /* key blocks of the Eq. (4) split (1 = unsplit) */
    uint64_t k3_cols_per_cta; /* route (a): columns per CTA of the inverse column pass (K3):
                                 cols_per_cta, or half of it when that fits two CTAs per SM */
} pa_info;

/* Fill *opt with defaults (route AUTO, arith AUTO, device -1 = current, offset 0, library
 * batch width, no split). */
pa_status pa_options_init(pa_options *opt);

/* Create a hashing context for n-bit keys and m-bit outputs with the
 * (n+m-1)-bit seed at `seed_bits` (device, ceil((off+n+m-1)/32) uint32 words
 * readable).  Requires 1 <= m <= n (reading R7) unless opt->allow_wide.  The seed is consumed
 * on `stream` during create (route (a) transforms it once into a cached
 * spectrum; route (b) stores it bit-reversed); the caller may free it after
 * the stream passes this call.  On success *h owns all device memory it
 * needs; on failure *h is NULL. */
pa_status pa_create(pa_handle *h, uint64_t n, uint64_t m, const uint32_t *seed_bits,
                    void *stream);
pa_status pa_create_ex(pa_handle *h, uint64_t n, uint64_t m, const uint32_t *seed_bits,
                       const pa_options *opt, void *stream);

/* Caller-owned device memory (torch allocates, libpa carves): pa_workspace_size
 * returns the exact bytes pa_create_ws needs for (n, m, *opt) (opt may be NULL =
 * defaults) -- host-only, no device work.  pa_create_ws is pa_create_ex with every
 * device buffer of the handle (seed spectrum, tables, per-key work buffers for
 * opt->batch_keys keys, pa_hash_host staging) placed in `workspace` (device pointer
 * on the current device, 256-byte aligned, >= the size, PA_ERR_NOMEM naming both
 * numbers if smaller).  The caller keeps ownership: the workspace must outlive the
 * handle and not be touched while it lives; pa_destroy does not free it. */
pa_status pa_workspace_size(uint64_t n, uint64_t m, const pa_options *opt, uint64_t *bytes);
pa_status pa_create_ws(pa_handle *h, uint64_t n, uint64_t m, const uint32_t *seed_bits,
                       const pa_options *opt, void *workspace, uint64_t workspace_bytes,
                       void *stream);

/* Rebind the handle to a new seed (same n, m, seed_bit_offset): the paper's
 * protocol draws a fresh uniform seed for every privacy-amplification round
 * (Sec. 2.3 Step 1).  Stream-ordered: hashes enqueued before this call use
 * the old seed, hashes after it the new one.  Route (a) recomputes the cached
 * spectrum (one forward transform, ~half a hash); route (b) re-reverses the seed. */
pa_status pa_set_seed(pa_handle h, const uint32_t *seed_bits, void *stream);

/* Fresh seed per key (Sec. 2.3 Step 1: every privacy-amplification round draws a
 * new uniform seed): for k < count, rebind the handle to seed k (seeds +
 * k*seed_stride_words, n+m-1 bits at the handle's seed_bit_offset) and hash key k into
 * output k -- the result of pa_set_seed + pa_hash per key, i.e. three transforms per key on
 * route (a).  An unsplit route-(a) handle without a workspace, given two keys or more, runs the
 * seeds of a chunk of keys through K0/K1 as one batch into a second work array (extra device
 * memory: chunk x 16 M bytes, grown on demand) and hashes the chunk's keys as one batch whose K2
 * runs each seed's forward half itself, the spectrum row held in tensor memory (where that K2
 * does not apply, the chunk's seeds are transformed into per-key spectra first); otherwise (or
 * if the memory is not available) one key at a time.  Strides in uint32 words, multiples of 4.
 * Afterwards the handle holds the last seed. */
pa_status pa_hash_fresh_batch(pa_handle h, const uint32_t *seeds, uint64_t seed_stride_words,
                              const uint32_t *keys, uint64_t key_stride_words, uint32_t *outs,
                              uint64_t out_stride_words, uint32_t count, void *stream);

/* Seed layout converter (reading R2).  Eq. (1) names the n+l-1
 * seed symbols t_0 .. t_{n+l-2} of the n x l matrix T of r = u T: T_{i,j} =
 * t_{i-j} on and below the diagonal, t_{j-i+n-1} above it.  This library's T[i][j] =
 * s[i-j+n-1] (y = T x) is the same hash when s[u] = t_{n-1-u} for u < n and s[u] = t_u
 * for n <= u < n+m-1: the first n symbols reversed.  t_bits -> s_bits, both device,
 * ceil((n+m-1)/32) words, LSB-first; bits past n+m-1 of s_bits are written 0.  The
 * buffers must not overlap (PA_ERR_INVALID_ARG).  Stream-ordered. */
pa_status pa_seed_from_paper_eq1(uint32_t *s_bits, const uint32_t *t_bits, uint64_t n, uint64_t m,
                                 void *stream);

/* y = T x.  key_bits: device, ceil(n/32) uint32 words; bits >= n are ignored.
 * out_bits: device, ceil(m/32) uint32 words; every bit >= m is written 0.  key_bits and
 * out_bits must not overlap (PA_ERR_INVALID_ARG): the output is zeroed while the key is read.
 * Deterministic, bit-exact, stream-ordered, asynchronous. */
pa_status pa_hash(pa_handle h, const uint32_t *key_bits, uint32_t *out_bits, void *stream);

/* count keys against the same seed.  Key k at keys + k*key_stride_words,
 * output k at outs + k*out_stride_words (strides in uint32 words, at least
 * ceil(n/32) and ceil(m/32)).  Output order = input order. */
pa_status pa_hash_batch(pa_handle h, const uint32_t *keys, uint64_t key_stride_words,
                        uint32_t *outs, uint64_t out_stride_words, uint32_t count,
                        void *stream);

/* End-to-end variant with HOST buffers (pinned memory recommended): copies the
 * key host->device, hashes, copies the output device->host, and synchronises
 * the stream before returning. key_host: ceil(n/32) words; out_host: ceil(m/32).
 * Pinned buffers (cudaHostAlloc / cudaHostRegister, e.g. torch pin_memory()) are moved by two
 * copy kernels over the mapped pages inside one cached CUDA graph; pageable buffers by plain
 * stream-ordered copies.  Host pointers need only 4-byte alignment. */
pa_status pa_hash_host(pa_handle h, const uint32_t *key_host, uint32_t *out_host, void *stream);

/* pa_hash_host without the final synchronisation: the copies and kernels are
 * enqueued on `stream` (as one CUDA graph, re-captured when the handle's work buffers have
 * moved or a host buffer's mapping changed) and *out_host is valid once the stream
 * reaches this point.  Lets a caller stream keys through a handle: successive calls
 * on the same stream serialise on the GPU but not on the host.  key_host must stay
 * unchanged and out_host unread until then. */
pa_status pa_hash_host_async(pa_handle h, const uint32_t *key_host, uint32_t *out_host, void *stream);

/* Batched end to end with HOST buffers (pinned memory recommended): count keys at key_host +
 * k*key_stride_words are hashed with the handle's seed and the outputs written to out_host +
 * k*out_stride_words.  Keys move in chunks through two device staging slots: chunk i+1's
 * host->device copy and chunk i-1's device->host copy (copy engines, on a stream of the handle)
 * overlap chunk i's hash on `stream`.  Synchronises `stream` before returning.  Strides in uint32 words (>= ceil(n/32) and
 * ceil(m/32)).  Staging grows on demand; a workspace handle (pa_create_ws) allocates nothing
 * more and hashes the keys one at a time through its own pa_hash_host staging instead.  On an
 * error the copies already enqueued are drained before returning. */
pa_status pa_hash_host_batch(pa_handle h, const uint32_t *keys_host, uint64_t key_stride_words,
                             uint32_t *outs_host, uint64_t out_stride_words, uint32_t count, void *stream);

/* uint64-packed aliases (same bits on little-endian).  pa_hash_u64 writes all
 * ceil(m/64) output words, zero-filling the half-word past ceil(m/32). */
pa_status pa_create_u64(pa_handle *h, uint64_t n, uint64_t m, const uint64_t *seed_bits,
                        void *stream);
pa_status pa_hash_u64(pa_handle h, const uint64_t *key_bits, uint64_t *out_bits, void *stream);

/* Route (a): synchronises `stream`, returns the largest |v - rint(v)| seen over
 * output-window values since the previous call (0 for route b), and resets it.
 * Returns PA_ERR_PRECISION if it exceeded PA_RESIDUAL_LIMIT. */
pa_status pa_residual(pa_handle h, double *max_residual, void *stream);

pa_status pa_get_info(pa_handle h, pa_info *info);

/* Host-only planning query (no device work, no handle): fills the route, the
 * transform length and the N1 x N2 split pa_create would choose for (n, m) with
 * default options.  workspace_bytes is the device memory the handle would own. */
pa_status pa_plan(uint64_t n, uint64_t m, pa_info *info);

/* Per-kernel device timing (for bench.py's roofline): while enabled, every
 * kernel libpa launches for this handle is bracketed by a CUDA event pair on
 * the launching stream.  pa_profile_read synchronises those events, returns
 * up to `max` entries {kernel name, launches, total milliseconds} accumulated
 * since the previous read, and resets the counters. */
typedef struct pa_kernel_time {
    char name[32];
    uint64_t launches;
    double total_ms;
} pa_kernel_time;

pa_status pa_profile_enable(pa_handle h, int enable);
pa_status pa_profile_read(pa_handle h, pa_kernel_time *out, uint32_t max, uint32_t *count);

/* Length-compatible hashing for keys whose single transform would be too long
 * (Sec. 3, Fig. 1, Eq. (4)-(7)): T is cut into row blocks of mb rows and
 * key (column) blocks of nb bits, nb + mb - 1 <= max_block_bits (0 = library choice: the block
 * length, up to the largest one handle plans, whose blocks the planner's cost model prices
 * cheapest in total), nb and mb multiples of 32 with the least total transform work for the
 * limit; block (r0, c0) is a Toeplitz hash on the seed window
 * at bit r0 + n - c0 - nb (zero-padded before s[0]; the last key block's bits past n and the
 * last row block's rows past m are padding), and each row block's output is the XOR of its
 * column blocks (Eq. (7)).  One handle of the block shape serves every block (pa_set_seed per
 * block).  seed_bits: n+m-1 bits, key_bits: n bits, out_bits: ceil(m/32) words, all device;
 * out bits >= m are written 0.  Synchronises `stream` before returning. */
pa_status pa_hash_blocked(uint64_t n, uint64_t m, const uint32_t *seed_bits, const uint32_t *key_bits,
                          uint32_t *out_bits, uint64_t max_block_bits, void *stream);

/* pa_hash_blocked with the seed, key and output in HOST memory (pinned recommended): keys of
 * 10^9-10^10 bits need not fit the device.  Each block's key and seed words move
 * host->device on a copy stream into one of two staging slots while the previous block is
 * hashed, and every finished row block's output moves device->host the same way.
 * device_budget_bytes > 0 caps the device memory the call uses (block handle + staging): the
 * block length is the largest within it (PA_ERR_NOMEM if even a 64-bit block does not fit);
 * 0 = no cap (max_block_bits or the planner's limit).  Synchronises `stream` before returning. */
pa_status pa_hash_blocked_host(uint64_t n, uint64_t m, const uint32_t *seed_host, const uint32_t *key_host,
                               uint32_t *out_host, uint64_t max_block_bits, uint64_t device_budget_bytes,
                               void *stream);

/* The block shape pa_hash_blocked / pa_hash_blocked_host would use for (n, m, max_block_bits,
 * device_budget_bytes) -- same arguments, same rules (Eq. (4)-(7)): nb key
 * bits and mb rows per block (multiples of 32, nb + mb - 1 <= the limit) and the number of
 * blocks ceil(m/mb) * ceil(n/nb).  Host-only planning (no device work); PA_ERR_NOMEM when the
 * budget cannot hold the smallest block, PA_ERR_INVALID_ARG for m > n, m = 0 or NULL outputs. */
pa_status pa_blocked_plan(uint64_t n, uint64_t m, uint64_t max_block_bits, uint64_t device_budget_bytes,
                          uint64_t *nb, uint64_t *mb, uint64_t *blocks);

/* pa_hash_blocked / pa_hash_blocked_host keep their block handle and staging buffers (one set per
 * process, reused by calls of the same block shape on the same device; calls are serialised)
 * because creating and freeing a multi-GB handle costs more than hashing a block.  This frees
 * them. */
void pa_hash_blocked_release(void);

/* Modulo-2 addition of partial hashes (Eq. (7)): dst[w] = XOR over
 * g < count of src[g * src_stride_words + w], w < words.  Device pointers,
 * 16-byte aligned, src_stride_words a multiple of 4; dst may alias src's first
 * vector.  Used by the multi-GPU input-column split after NCCL gathers partials. */
pa_status pa_xor_fold(uint32_t *dst, const uint32_t *src, uint64_t words, uint32_t count,
                      uint64_t src_stride_words, void *stream);

/* The Eq. (7) merge over peer memory (multi-GPU input-column split): dst[w] =
 * XOR over g < count of srcs[g][first_word + w], w < words.  srcs is a DEVICE array of count
 * device pointers -- this rank's partial and the peers' partials mapped through pa_peer_open
 * (NVLink / NVSwitch loads); dst 16-byte aligned, first_word a multiple of 4.  The caller orders
 * it after every rank's hash (e.g. a one-element NCCL all-reduce as a stream barrier). */
pa_status pa_xor_fold_peers(uint32_t *dst, const uint32_t *const *srcs, uint32_t count, uint64_t first_word,
                            uint64_t words, void *stream);

/* Peer-mappable device memory for pa_xor_fold_peers: pa_peer_alloc returns a whole cudaMalloc
 * allocation on the current device (free with pa_peer_free); pa_peer_export fills a 64-byte
 * handle (CUDA IPC) another process passes to pa_peer_open, which maps the allocation into its
 * address space (lazy peer access; unmap with pa_peer_close).  A process cannot open its own
 * handle -- use the pointer directly. */
typedef struct pa_peer_handle {
    unsigned char bytes[64];
} pa_peer_handle;
pa_status pa_peer_alloc(uint64_t bytes, void **dev_ptr);
pa_status pa_peer_free(void *dev_ptr);
pa_status pa_peer_export(const void *dev_ptr, pa_peer_handle *handle);
pa_status pa_peer_open(const pa_peer_handle *handle, void **dev_ptr);
pa_status pa_peer_close(void *dev_ptr);

/* Stream-ordered release of everything the handle owns.  Safe on NULL. */
void pa_destroy(pa_handle h);

const char *pa_last_error(void);
const char *pa_status_string(pa_status s);
uint32_t pa_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PA_H */
