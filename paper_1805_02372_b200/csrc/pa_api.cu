// pa_api.cu -- the C ABI declared in include/pa.h: argument validation, route
// selection and dispatch.  No exceptions cross this boundary.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <cmath>
#include <new>
#include <tuple>
#include <string>
#include <vector>

#include "pa_internal.h"

namespace pa {

static thread_local std::string g_err;

void set_error(const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
}

pa_status cuda_fail(cudaError_t e, const char *what)
{
    set_error("%s: CUDA error %d (%s)", what, (int)e, cudaGetErrorString(e));
    return PA_ERR_CUDA;
}

// Route (b) costs ~n*m/1024 SHF+LOP3 pairs per SM-cycle; route (a) a few
// microseconds of fixed latency plus ~40 bytes of HBM traffic per output
// point.  Below ~2^26 bit-products (e.g. n = 4096, m = 1024: 2^22) the direct
// product wins (SURVEY.md Sec. 8(d) crossover).
static int choose_route(uint64_t n, uint64_t m)
{
    double prod = (double)n * (double)m;
    return prod <= 67108864.0 ? PA_ROUTE_BITPACKED : PA_ROUTE_TRANSFORM;
}

static pa_status check_dev_ptr(const void *p, const char *name, int device)
{
    if (!p) {
        set_error("%s is NULL", name);
        return PA_ERR_INVALID_ARG;
    }
    if ((uintptr_t)p & 15) {
        set_error("%s = %p is not 16-byte aligned", name, p);
        return PA_ERR_INVALID_ARG;
    }
    cudaPointerAttributes at;
    cudaError_t e = cudaPointerGetAttributes(&at, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("%s = %p: cudaPointerGetAttributes failed (%s)", name, p, cudaGetErrorString(e));
        return PA_ERR_INVALID_ARG;
    }
    if (at.type != cudaMemoryTypeDevice && at.type != cudaMemoryTypeManaged) {
        set_error("%s = %p is not device memory (cudaMemoryType %d); use pa_hash_host for host "
                  "buffers", name, p, (int)at.type);
        return PA_ERR_INVALID_ARG;
    }
    if (at.type == cudaMemoryTypeDevice && at.device != device) {
        set_error("%s = %p lives on device %d, the handle on device %d", name, p, at.device, device);
        return PA_ERR_INVALID_ARG;
    }
    return PA_OK;
}

pa_status dev_alloc(pa_ctx *h, void **p, size_t bytes, const char *what)
{
    *p = nullptr;
    bytes = al256(bytes);
    if (h->arena) {
        Arena &A = *h->arena;
        if (A.used + bytes > A.size) {
            set_error("%s: workspace too small (%llu bytes used + %llu needed > %llu; see "
                      "pa_workspace_size)", what, (unsigned long long)A.used, (unsigned long long)bytes,
                      (unsigned long long)A.size);
            return PA_ERR_NOMEM;
        }
        *p = A.base + A.used;
        A.used += bytes;
    } else {
        cudaError_t e = cudaMalloc(p, bytes);
        if (e != cudaSuccess) {
            *p = nullptr;
            cudaGetLastError();
            set_error("%s: cudaMalloc of %llu bytes failed: %s", what, (unsigned long long)bytes,
                      cudaGetErrorString(e));
            return PA_ERR_NOMEM;
        }
    }
    h->ws_bytes += bytes;
    return PA_OK;
}

void dev_free(pa_ctx *h, void *p)
{
    if (p && !h->arena) cudaFree(p);
}

void reap(pa_ctx *h, bool wait)
{
    int k = 0;
    for (int i = 0; i < h->ngrave; ++i) {
        if (wait) cudaEventSynchronize(h->grave_ev[i]);
        if (wait || cudaEventQuery(h->grave_ev[i]) == cudaSuccess) {
            cudaFree(h->grave[i]);
            cudaEventDestroy(h->grave_ev[i]);
        } else {
            h->grave[k] = h->grave[i];
            h->grave_ev[k++] = h->grave_ev[i];
        }
    }
    cudaGetLastError();  // a not-ready query is not an error
    h->ngrave = k;
}

void defer_free(pa_ctx *h, void *p, cudaStream_t s)
{
    if (!p || h->arena) return;
    reap(h, false);
    if (h->ngrave == pa_ctx::kGrave) {  // full: wait for the oldest
        cudaEventSynchronize(h->grave_ev[0]);
        reap(h, false);
    }
    cudaEvent_t ev = nullptr;
    if (h->ngrave == pa_ctx::kGrave || cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(ev, s) != cudaSuccess) {
        if (ev) cudaEventDestroy(ev);
        cudaGetLastError();
        cudaStreamSynchronize(s);
        cudaFree(p);
        return;
    }
    h->grave[h->ngrave] = p;
    h->grave_ev[h->ngrave++] = ev;
}

static cudaEvent_t prof_event(Profiler &P)
{
    if (P.npool > 0) return P.pool[--P.npool];
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

// column-block sub-handles report into their parent's profiler
void prof_begin(pa_ctx *h, int k, cudaStream_t s)
{
    Profiler &P = (h->parent ? h->parent : h)->prof;
    if (!P.on) return;
    if (P.npend == P.cap) {
        int nc = P.cap ? 2 * P.cap : 64;
        Profiler::Pending *np = (Profiler::Pending *)realloc(P.pend, nc * sizeof *np);
        if (!np) return;
        P.pend = np;
        P.cap = nc;
    }
    Profiler::Pending &q = P.pend[P.npend++];
    q.k = k;
    q.e0 = prof_event(P);
    q.e1 = nullptr;
    cudaEventRecord(q.e0, s);
}

void prof_end(pa_ctx *h, cudaStream_t s)
{
    Profiler &P = (h->parent ? h->parent : h)->prof;
    if (!P.on || P.npend == 0 || P.pend[P.npend - 1].e1) return;
    Profiler::Pending &q = P.pend[P.npend - 1];
    q.e1 = prof_event(P);
    cudaEventRecord(q.e1, s);
}

static void prof_release(Profiler &P, cudaEvent_t e)
{
    if (!e) return;
    if (P.npool == P.poolcap) {
        int nc = P.poolcap ? 2 * P.poolcap : 128;
        cudaEvent_t *np = (cudaEvent_t *)realloc(P.pool, nc * sizeof *np);
        if (!np) {
            cudaEventDestroy(e);
            return;
        }
        P.pool = np;
        P.poolcap = nc;
    }
    P.pool[P.npool++] = e;
}

static void prof_free(Profiler &P)
{
    for (int i = 0; i < P.npend; ++i) {
        if (P.pend[i].e0) cudaEventDestroy(P.pend[i].e0);
        if (P.pend[i].e1) cudaEventDestroy(P.pend[i].e1);
    }
    for (int i = 0; i < P.npool; ++i) cudaEventDestroy(P.pool[i]);
    free(P.pend);
    free(P.pool);
    P = Profiler{};
}

}  // namespace pa

using namespace pa;

namespace {
// Every call on a handle runs on the handle's device (pa_options.device): switch for the call
// and back (a no-op when it is already current).
struct DeviceGuard {
    int prev = -1;
    bool sw = false;
    explicit DeviceGuard(int dev)
    {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) sw = cudaSetDevice(dev) == cudaSuccess;
    }
    ~DeviceGuard()
    {
        if (sw) cudaSetDevice(prev);
    }
};
}  // namespace

extern "C" {

static void drop_host_graph(pa_ctx *h);

uint32_t pa_version(void) { return PA_VERSION; }

const char *pa_last_error(void) { return g_err.c_str(); }

const char *pa_status_string(pa_status s)
{
    switch (s) {
    case PA_OK: return "PA_OK";
    case PA_ERR_INVALID_ARG: return "PA_ERR_INVALID_ARG";
    case PA_ERR_UNSUPPORTED: return "PA_ERR_UNSUPPORTED";
    case PA_ERR_NOMEM: return "PA_ERR_NOMEM";
    case PA_ERR_CUDA: return "PA_ERR_CUDA";
    case PA_ERR_PRECISION: return "PA_ERR_PRECISION";
    }
    return "PA_ERR_UNKNOWN";
}

pa_status pa_options_init(pa_options *opt)
{
    if (!opt) {
        set_error("opt is NULL");
        return PA_ERR_INVALID_ARG;
    }
    memset(opt, 0, sizeof *opt);
    opt->struct_size = sizeof *opt;
    opt->route = PA_ROUTE_AUTO;
    opt->arith = PA_ARITH_AUTO;
    opt->device = -1;
    return PA_OK;
}

static void destroy_ctx(pa_ctx *h)
{
    for (uint32_t g = 0; h->sub && g < h->nsub; ++g)
        if (h->sub[g]) destroy_ctx(h->sub[g]);
    delete[] h->sub;
    delete[] h->sub_c0;
    prof_free(h->prof);
    drop_host_graph(h);
    reap(h, true);
    ra_destroy(h);
    rb_destroy(h);
    dev_free(h, h->stage_blk);
    if (h->bstage) cudaFree(h->bstage);
    for (cudaEvent_t &ev : h->pev)
        if (ev) cudaEventDestroy(ev);
    if (h->cstream) cudaStreamDestroy(h->cstream);
    if (h->own_arena) delete h->arena;
    delete h;
}

void pa_destroy(pa_handle h)
{
    if (!h) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(h->device);
    destroy_ctx(h);
    cudaSetDevice(prev);
}

// Validate and complete the caller's options.
static pa_status parse_options(const pa_options *opt, uint64_t n, uint64_t m, pa_options *o)
{
    pa_options_init(o);
    if (opt) {
        if (opt->struct_size != sizeof(pa_options)) {
            set_error("opt->struct_size = %u, expected %u (call pa_options_init)", opt->struct_size,
                      (unsigned)sizeof(pa_options));
            return PA_ERR_INVALID_ARG;
        }
        *o = *opt;
    }
    if (n == 0 || m == 0 || (m > n && !o->allow_wide)) {
        set_error("need 1 <= m <= n (or opt->allow_wide), got n = %llu, m = %llu", (unsigned long long)n,
                  (unsigned long long)m);
        return PA_ERR_INVALID_ARG;
    }
    if (n > (1ull << 40) || m > (1ull << 40)) {
        set_error("n = %llu, m = %llu: lengths beyond 2^40 bits are unsupported", (unsigned long long)n,
                  (unsigned long long)m);
        return PA_ERR_UNSUPPORTED;
    }
    if (o->route < PA_ROUTE_AUTO || o->route > PA_ROUTE_BITPACKED) {
        set_error("opt->route = %d is not a pa_route", o->route);
        return PA_ERR_INVALID_ARG;
    }
    if (o->allow_wide > 1) {
        set_error("opt->allow_wide = %u must be 0 or 1", o->allow_wide);
        return PA_ERR_INVALID_ARG;
    }
    if (o->batch_keys > 4096) {
        set_error("opt->batch_keys = %u exceeds 4096", o->batch_keys);
        return PA_ERR_INVALID_ARG;
    }
    if (o->arith == PA_ARITH_NTT32 || o->arith == PA_ARITH_NTT64) {
        set_error("opt->arith = %d: the number-theoretic transforms are not built (FP64 is the route-(a) "
                  "arithmetic; use PA_ARITH_AUTO or PA_ARITH_FP64)", o->arith);
        return PA_ERR_UNSUPPORTED;
    }
    if (o->arith != PA_ARITH_AUTO && o->arith != PA_ARITH_FP64) {
        set_error("opt->arith = %d is not a pa_arith", o->arith);
        return PA_ERR_INVALID_ARG;
    }
    if (o->plan_mode > PA_PLAN_MEASURE) {
        set_error("opt->plan_mode = %u is not a pa_plan_mode", o->plan_mode);
        return PA_ERR_INVALID_ARG;
    }
    if (o->device < -1) {
        set_error("opt->device = %d: use -1 (current device) or a CUDA device ordinal", o->device);
        return PA_ERR_INVALID_ARG;
    }

    if (o->route == PA_ROUTE_AUTO) o->route = choose_route(n, m);
    return PA_OK;
}

// (an upper bound on) the longest real transform one route-(a) plan reaches: a K2 row (N1
// points) and a K1/K3 column (N2 points) must each fit one CTA's 227 KB of shared memory at
// 17 bytes per padded complex point, so N1, N2 <~ 13.3 k; two reals per complex point
static const uint64_t kMaxPlanLen = 2ull * 13312 * 13312;

static bool plan_fits(uint64_t n, uint64_t m, uint64_t maxlen)  // route (a) can plan within the cap
{
    Geometry g;
    char err[256];
    return ra_plan(n, m, &g, err, sizeof err, maxlen) == PA_OK;
}

// The automatic split's block length: the longest blocks one plan holds are not the fastest
// (their plans are one-column, general-kernel ones).  Among caps from kMaxPlanLen down to a
// third of it -- each also stretched to the longest block its plan holds, 2 N1 N2 -- take the
// one the cost model prices cheapest as key blocks x model time per hash (x 1.2 for plans
// without the shape-specialised kernels; measured n = 3e8, m = 3e7: see DESIGN.md Sec. 6d).
// Memoised per (n, m): ~80 plans per search.
static uint64_t auto_cap(uint64_t n, uint64_t m)
{
    static std::mutex mu;
    static std::map<std::pair<uint64_t, uint64_t>, uint64_t> memo;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = memo.find({n, m});
        if (it != memo.end()) return it->second;
    }
    uint64_t pick = kMaxPlanLen;
    double best = 1e300;
    auto price = [&](uint64_t L, Geometry *g) -> bool {
        if (L > kMaxPlanLen || L + 1 < m + 128) return false;
        uint64_t nb = (L + 1 - m) / 128 * 128;
        if (nb >= n) nb = (n + 127) / 128 * 128;
        char err[256];
        if (ra_plan(nb, m, g, err, sizeof err, kMaxPlanLen) != PA_OK) return false;
        const double t = (double)((n + nb - 1) / nb) * ra_last_plan_cost() * (ra_plan_specialised(*g) ? 1.0 : 1.2);
        if (t < best) {
            best = t;
            pick = L;
        }
        return true;
    };
    for (int i = 0; i < 48; ++i) {
        const uint64_t L = (uint64_t)((double)kMaxPlanLen * std::pow(0.977, i));
        Geometry g, g2;
        if (!price(L, &g)) continue;
        price(std::min<uint64_t>(2ull * g.N1 * g.N2, kMaxPlanLen), &g2);
    }
    std::lock_guard<std::mutex> lock(mu);
    memo[{n, m}] = pick;
    return pick;
}

// Eq. (4) column blocks for a transform-length cap: equal blocks of nb key
// bits (a multiple of 128, so every block's key pointer stays 16-byte aligned) and a
// shorter last one.  c0 receives the block starts; one entry = no split.
static pa_status split_plan(uint64_t n, uint64_t m, uint64_t maxlen, std::vector<uint64_t> *c0)
{
    c0->assign(1, 0);
    if (!maxlen) {
        // no cap requested: split only when no single transform can be planned (n + m beyond
        // ~3.5e8 bits -- the paper's length-compatible regime), with the block length
        // the cost model prices cheapest (auto_cap)
        if (plan_fits(n, m, 0)) return PA_OK;
        maxlen = auto_cap(n, m);
    }
    if (plan_fits(n, m, maxlen)) return PA_OK;
    if (maxlen + 1 < m + 128) {
        set_error("max_transform_len = %llu cannot hold even a 128-bit key block with m = %llu "
                  "(needs >= %llu)", (unsigned long long)maxlen, (unsigned long long)m,
                  (unsigned long long)(m + 127));
        return PA_ERR_UNSUPPORTED;
    }
    uint64_t nb = (maxlen + 1 - m) / 128 * 128;  // nb + m - 1 <= maxlen
    if (nb >= n) nb = (n - 1) / 128 * 128;       // the whole key did not fit: split it anyway
    while (nb >= 128) {
        const uint64_t last = n - (n - 1) / nb * nb;
        if (plan_fits(nb, m, maxlen) && plan_fits(last, m, maxlen)) break;
        uint64_t step = (nb / 64 + 127) / 128 * 128;
        nb = nb > step ? nb - step : 0;
    }
    if (nb < 128) {
        set_error("max_transform_len = %llu: no 128-bit-aligned key block plan fits (m = %llu)",
                  (unsigned long long)maxlen, (unsigned long long)m);
        return PA_ERR_UNSUPPORTED;
    }
    const uint64_t G = (n + nb - 1) / nb;
    if (G > 65536) {
        set_error("max_transform_len = %llu would cut the key into %llu blocks (> 65536)",
                  (unsigned long long)maxlen, (unsigned long long)G);
        return PA_ERR_UNSUPPORTED;
    }
    c0->clear();
    for (uint64_t g = 0; g < G; ++g) c0->push_back(g * nb);
    return PA_OK;
}

static size_t stage_bytes(uint64_t n, uint64_t m) { return al256((n + 31) / 32 * 4) + al256((m + 31) / 32 * 4); }

// Exact device bytes a handle takes for (n, m, o) -- the sum of its dev_alloc calls.
static pa_status handle_bytes(uint64_t n, uint64_t m, const pa_options &o, bool arena, size_t *bytes)
{
    *bytes = arena ? stage_bytes(n, m) : 0;  // without a workspace staging is allocated lazily
    if (o.route == PA_ROUTE_BITPACKED) {
        *bytes += rb_bytes(n, m);
        return PA_OK;
    }
    std::vector<uint64_t> c0;
    pa_status st = split_plan(n, m, o.max_transform_len, &c0);
    if (st != PA_OK) return st;
    const uint32_t cap = (arena || c0.size() > 1) && o.batch_keys ? o.batch_keys : 1;
    const uint64_t cap_len = c0.size() > 1 && !o.max_transform_len ? kMaxPlanLen : o.max_transform_len;
    size_t w0 = 0;
    for (size_t g = 0; g < c0.size(); ++g) {
        const uint64_t ng = (g + 1 < c0.size() ? c0[g + 1] : n) - c0[g];
        Geometry geo;
        char err[256];
        if ((st = ra_plan(ng, m, &geo, err, sizeof err, cap_len)) != PA_OK) {
            set_error("%s", err);
            return st;
        }
        const size_t w = ra_work_bytes(geo, cap);
        *bytes += ra_persist_bytes(geo);
        if (g == 0) w0 = w;
        if (g == 0 || w > w0) *bytes += w;  // later blocks borrow block 0's work buffers (create_impl)
    }
    return PA_OK;
}

static pa_status measure_plan(uint64_t n, uint64_t m, const uint32_t *seed_bits, const pa_options &o,
                              cudaStream_t s, PlanChoice *best);

static pa_status create_impl(pa_handle *out, uint64_t n, uint64_t m, const uint32_t *seed_bits,
                             const pa_options *opt, void *workspace, uint64_t workspace_bytes, void *stream,
                             const PlanChoice *force = nullptr)
{
    if (!out) {
        set_error("h (output handle pointer) is NULL");
        return PA_ERR_INVALID_ARG;
    }
    *out = nullptr;
    pa_options o;
    pa_status st = parse_options(opt, n, m, &o);
    if (st != PA_OK) return st;
    int dev = 0, ndev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (o.device >= 0) {
        if ((e = cudaGetDeviceCount(&ndev)) != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
        if (o.device >= ndev) {
            set_error("opt->device = %d, but %d CUDA device(s) are visible", o.device, ndev);
            return PA_ERR_INVALID_ARG;
        }
        dev = o.device;
    }
    DeviceGuard dg(dev);
    if ((st = check_dev_ptr(seed_bits, "seed_bits", dev)) != PA_OK) return st;
    if (workspace) {
        if ((st = check_dev_ptr(workspace, "workspace", dev)) != PA_OK) return st;
        if ((uintptr_t)workspace & 255) {
            set_error("workspace = %p is not 256-byte aligned", workspace);
            return PA_ERR_INVALID_ARG;
        }
    }
    std::vector<uint64_t> c0;
    if (o.route == PA_ROUTE_TRANSFORM && (st = split_plan(n, m, o.max_transform_len, &c0)) != PA_OK) return st;
    // measured planning (PA_PLAN_MEASURE): an unsplit route-(a) handle without a caller workspace
    // (whose size pa_workspace_size fixed from the model's plan) times the model's best candidates
    PlanChoice measured;
    if (!force && o.plan_mode == PA_PLAN_MEASURE && o.route == PA_ROUTE_TRANSFORM && c0.size() == 1 && !workspace) {
        if ((st = measure_plan(n, m, seed_bits, o, (cudaStream_t)stream, &measured)) != PA_OK) return st;
        if (measured.N1) force = &measured;
    }

    pa_ctx *h = new (std::nothrow) pa_ctx();
    if (!h) {
        set_error("host allocation of the handle failed");
        return PA_ERR_NOMEM;
    }
    h->device = dev;
    h->n = n;
    h->m = m;
    h->L = n + m - 1;
    h->off = o.seed_bit_offset;
    h->route = o.route;
    h->batch_opt = o.batch_keys;
    h->max_len = o.route == PA_ROUTE_TRANSFORM ? o.max_transform_len : 0;
    if (force && c0.size() == 1) {
        h->force = *force;
        h->has_force = true;
    }
    if (o.route == PA_ROUTE_TRANSFORM && c0.size() > 1 && !h->max_len) h->max_len = kMaxPlanLen;  // auto split
    if (workspace) {
        h->arena = new (std::nothrow) Arena();
        if (!h->arena) {
            delete h;
            set_error("host allocation of the handle failed");
            return PA_ERR_NOMEM;
        }
        h->own_arena = true;
        h->arena->base = (char *)workspace;
        h->arena->size = workspace_bytes;
        // staging for pa_hash_host comes out of the workspace up front
        if ((st = dev_alloc(h, (void **)&h->stage_blk, stage_bytes(n, m), "pa_hash_host staging")) == PA_OK) {
            h->stage_key = (uint32_t *)h->stage_blk;
            h->stage_out = (uint32_t *)(h->stage_blk + al256((n + 31) / 32 * 4));
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (st == PA_OK && c0.size() > 1) {
        // Eq. (4) split: block g = key bits [c0, c0 + ng), seed window offset n - ng - c0
        const uint32_t nb = (uint32_t)c0.size();
        h->sub = new (std::nothrow) pa_ctx *[nb]();
        h->sub_c0 = new (std::nothrow) uint64_t[nb];
        if (!h->sub || !h->sub_c0) {
            set_error("host allocation of %u block handles failed", nb);
            st = PA_ERR_NOMEM;
        } else {
            h->nsub = nb;  // only now: destroy_ctx walks sub[0 .. nsub)
        }
        for (uint32_t g = 0; st == PA_OK && g < h->nsub; ++g) {
            const uint64_t ng = (g + 1 < h->nsub ? c0[g + 1] : n) - c0[g];
            pa_ctx *b = new (std::nothrow) pa_ctx();
            if (!b) {
                set_error("host allocation of block handle %u failed", g);
                st = PA_ERR_NOMEM;
                break;
            }
            h->sub[g] = b;
            h->sub_c0[g] = c0[g];
            b->parent = h;
            b->arena = h->arena;
            b->device = dev;
            b->n = ng;
            b->m = m;
            b->L = ng + m - 1;
            b->off = h->off + (n - ng - c0[g]);
            b->route = PA_ROUTE_TRANSFORM;
            b->batch_opt = h->batch_opt;
            b->max_len = h->max_len;
            if (g > 0) {
                b->share_w = h->sub[0]->a.wblk;
                b->share_w_bytes = ra_work_bytes(h->sub[0]->a.g, h->sub[0]->a.cap);
            }
            st = ra_create(b, seed_bits, s);
            h->kernels_per_hash += b->kernels_per_hash;
        }
    } else if (st == PA_OK) {
        st = h->route == PA_ROUTE_TRANSFORM ? ra_create(h, seed_bits, s) : rb_create(h, seed_bits, s);
    }
    if (st != PA_OK) {
        std::string keep = g_err;
        pa_destroy(h);
        g_err = keep;
        return st;
    }
    *out = h;
    return PA_OK;
}

// Measured planning: the model's best few candidate plans, each built as a real handle on the
// caller's seed and timed on an all-zero key (route (a)'s time is independent of the data) after
// an L2 flush, median of five (a challenger must beat the model's pick by 2%); the fastest is
// remembered per (n, m, max_transform_len, device)
// for the life of the process (FFTW-style "wisdom"), so later handles of the shape skip it.
static std::mutex g_wisdom_mutex;
static std::map<std::tuple<uint64_t, uint64_t, uint64_t, int>, PlanChoice> g_wisdom;

static pa_status measure_plan(uint64_t n, uint64_t m, const uint32_t *seed_bits, const pa_options &o,
                              cudaStream_t s, PlanChoice *best)
{
    int dev = 0;
    cudaGetDevice(&dev);
    const auto key = std::make_tuple(n, m, (uint64_t)o.max_transform_len, dev);
    {
        std::lock_guard<std::mutex> lock(g_wisdom_mutex);
        auto it = g_wisdom.find(key);
        if (it != g_wisdom.end()) {
            *best = it->second;
            return PA_OK;
        }
    }
    constexpr int kCand = 6;
    PlanChoice cand[kCand];
    const int k = ra_plan_candidates(n, m, o.max_transform_len, cand, kCand);
    *best = PlanChoice{};
    if (k <= 1) {
        if (k == 1) *best = cand[0];
        return PA_OK;
    }
    uint32_t *key_bits = nullptr, *out_bits = nullptr;
    void *flush = nullptr;
    const size_t kb = ((n + 31) / 32 + 4) * 4, ob = ((m + 31) / 32 + 4) * 4, fb = 256u << 20;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&key_bits, kb)) != cudaSuccess || (e = cudaMalloc(&out_bits, ob)) != cudaSuccess ||
        (e = cudaMemsetAsync(key_bits, 0, kb, s)) != cudaSuccess || (e = cudaEventCreate(&e0)) != cudaSuccess ||
        (e = cudaEventCreate(&e1)) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(key_bits);
        cudaFree(out_bits);
        if (e0) cudaEventDestroy(e0);
        return cuda_fail(e, "measured planning scratch");
    }
    if (cudaMalloc(&flush, fb) != cudaSuccess) {  // no room for an L2 flush: time warm
        cudaGetLastError();
        flush = nullptr;
    } else {
        cudaMemsetAsync(flush, 0, fb, s);  // first touch outside the timings
    }
    pa_options oo = o;
    oo.plan_mode = PA_PLAN_MODEL;
    float best_ms = 3.4e38f;
    for (int i = 0; i < k; ++i) {
        pa_handle t = nullptr;
        if (create_impl(&t, n, m, seed_bits, &oo, nullptr, 0, s, &cand[i]) != PA_OK) {
            cudaGetLastError();
            continue;  // e.g. out of memory for a larger candidate: skip it
        }
        float ms[5];
        pa_status st = pa_hash(t, key_bits, out_bits, s);  // warm-up (code, tables)
        if (st == PA_OK) st = pa_hash(t, key_bits, out_bits, s);
        for (int r = 0; r < 5 && st == PA_OK; ++r) {
            if (flush) cudaMemsetAsync(flush, 0, fb, s);
            cudaEventRecord(e0, s);
            st = pa_hash(t, key_bits, out_bits, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms[r], e0, e1);
        }
        pa_destroy(t);
        if (st != PA_OK) continue;
        std::sort(ms, ms + 5);
#ifdef PA_DEV
        if (dev_env("PA_PLAN_DEBUG"))
            fprintf(stderr, "measure_plan n=%llu m=%llu cand %d: %ux%u C=%u median %.2f us (min %.2f max %.2f)\n",
                    (unsigned long long)n, (unsigned long long)m, i, cand[i].N1, cand[i].N2, cand[i].C, ms[2] * 1e3,
                    ms[0] * 1e3, ms[4] * 1e3);
#endif
        // a challenger must beat the incumbent by 2% (measurement noise must not trade the
        // model's choice for an equal plan)
        if (ms[2] < best_ms * (best->N1 ? 0.98f : 1.0f)) {
            best_ms = ms[2];
            *best = cand[i];
        }
    }
    cudaStreamSynchronize(s);
    cudaFree(key_bits);
    cudaFree(out_bits);
    if (flush) cudaFree(flush);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (best->N1) {
        std::lock_guard<std::mutex> lock(g_wisdom_mutex);
        g_wisdom[key] = *best;
    }
    return PA_OK;
}

pa_status pa_create_ex(pa_handle *out, uint64_t n, uint64_t m, const uint32_t *seed_bits,
                       const pa_options *opt, void *stream)
{
    return create_impl(out, n, m, seed_bits, opt, nullptr, 0, stream);
}

pa_status pa_workspace_size(uint64_t n, uint64_t m, const pa_options *opt, uint64_t *bytes)
{
    if (!bytes) {
        set_error("pa_workspace_size: bytes is NULL");
        return PA_ERR_INVALID_ARG;
    }
    *bytes = 0;
    pa_options o;
    pa_status st = parse_options(opt, n, m, &o);
    if (st != PA_OK) return st;
    size_t b = 0;
    if ((st = handle_bytes(n, m, o, true, &b)) != PA_OK) return st;
    *bytes = b;
    return PA_OK;
}

pa_status pa_create_ws(pa_handle *h, uint64_t n, uint64_t m, const uint32_t *seed_bits, const pa_options *opt,
                       void *workspace, uint64_t workspace_bytes, void *stream)
{
    if (!workspace) {
        if (h) *h = nullptr;
        set_error("pa_create_ws: workspace is NULL (use pa_create_ex for library-owned memory)");
        return PA_ERR_INVALID_ARG;
    }
    return create_impl(h, n, m, seed_bits, opt, workspace, workspace_bytes, stream);
}

pa_status pa_create(pa_handle *h, uint64_t n, uint64_t m, const uint32_t *seed_bits, void *stream)
{
    return pa_create_ex(h, n, m, seed_bits, nullptr, stream);
}

pa_status pa_create_u64(pa_handle *h, uint64_t n, uint64_t m, const uint64_t *seed_bits,
                        void *stream)
{
    return pa_create_ex(h, n, m, (const uint32_t *)seed_bits, nullptr, stream);
}

static pa_status seed_impl(pa_ctx *h, const uint32_t *seed_bits, cudaStream_t s)
{
    if (h->nsub) {
        for (uint32_t g = 0; g < h->nsub; ++g) {
            pa_status st = ra_seed(h->sub[g], seed_bits, s);
            if (st != PA_OK) return st;
        }
        return PA_OK;
    }
    return h->route == PA_ROUTE_TRANSFORM ? ra_seed(h, seed_bits, s) : rb_seed(h, seed_bits, s);
}

pa_status pa_set_seed(pa_handle h, const uint32_t *seed_bits, void *stream)
{
    if (!h) {
        set_error("handle is NULL");
        return PA_ERR_INVALID_ARG;
    }
    DeviceGuard dg(h->device);
    pa_status st = check_dev_ptr(seed_bits, "seed_bits", h->device);
    if (st != PA_OK) return st;
    return seed_impl(h, seed_bits, (cudaStream_t)stream);
}

// Keys [0, count) of a batch; the column blocks of a split handle XOR into the
// outputs the first block zeroed (Eq. (7)).
static pa_status batch_impl(pa_ctx *h, const uint32_t *keys, uint64_t key_stride, uint32_t *outs,
                            uint64_t out_stride, uint32_t count, uint64_t zero_words, cudaStream_t s)
{
    if (h->nsub) {
        for (uint32_t g = 0; g < h->nsub; ++g) {
            pa_status st = batch_impl(h->sub[g], keys + h->sub_c0[g] / 32, key_stride, outs, out_stride, count,
                                      g ? 0 : zero_words, s);
            if (st != PA_OK) return st;
        }
        return PA_OK;
    }
    if (h->route != PA_ROUTE_TRANSFORM) return rb_hash_batch(h, keys, key_stride, outs, out_stride, count, zero_words, s);
    // keys in chunks: all kernels take the key index from the grid
    const uint32_t chunk = ra_batch_keys(h);
    for (uint32_t k0 = 0; k0 < count; k0 += chunk) {
        const uint32_t c = count - k0 < chunk ? count - k0 : chunk;
        pa_status st = ra_hash_batch(h, keys + k0 * key_stride, key_stride, outs + k0 * out_stride, out_stride, c,
                                     zero_words, s);
        if (st != PA_OK) return st;
    }
    return PA_OK;
}

// would a batch of `count` keys grow (reallocate) some work buffer?
static bool batch_grows(const pa_ctx *h, uint32_t count)
{
    if (h->nsub) {
        for (uint32_t g = 0; g < h->nsub; ++g)
            if (batch_grows(h->sub[g], count)) return true;
        return false;
    }
    if (h->route != PA_ROUTE_TRANSFORM || h->arena || h->parent) return false;
    const uint32_t chunk = ra_batch_keys(h);
    return h->a.cap < (count < chunk ? count : chunk);
}

// [a, a + na) and [b, b + nb) bytes overlap?
static bool overlaps(const void *a, uint64_t na, const void *b, uint64_t nb)
{
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + nb && y < x + na;
}

static pa_status hash_impl(pa_handle h, const uint32_t *key, uint32_t *out, uint64_t zero_words,
                           cudaStream_t s, bool validate)
{
    if (!h) {
        set_error("handle is NULL");
        return PA_ERR_INVALID_ARG;
    }
    DeviceGuard dg(h->device);
    if (validate) {
        pa_status st;
        // the output is zeroed before (or while) the key is read: they must not share memory
        if (overlaps(key, (h->n + 31) / 32 * 4, out, zero_words * 4)) {
            set_error("key_bits (%p, %llu words) and out_bits (%p, %llu words) overlap", (const void *)key,
                      (unsigned long long)((h->n + 31) / 32), (void *)out, (unsigned long long)zero_words);
            return PA_ERR_INVALID_ARG;
        }
        if (key != h->ok_key) {
            if ((st = check_dev_ptr(key, "key_bits", h->device)) != PA_OK) return st;
            h->ok_key = key;
        }
        if (out != h->ok_out) {
            if ((st = check_dev_ptr(out, "out_bits", h->device)) != PA_OK) return st;
            h->ok_out = out;
        }
    }
    if (h->nsub) return batch_impl(h, key, 0, out, 0, 1, zero_words, s);
    return h->route == PA_ROUTE_TRANSFORM ? ra_hash(h, key, out, zero_words, s)
                                          : rb_hash(h, key, out, zero_words, s);
}

pa_status pa_hash(pa_handle h, const uint32_t *key_bits, uint32_t *out_bits, void *stream)
{
    if (!h) {
        set_error("handle is NULL");
        return PA_ERR_INVALID_ARG;
    }
    return hash_impl(h, key_bits, out_bits, (h->m + 31) / 32, (cudaStream_t)stream, true);
}

pa_status pa_hash_u64(pa_handle h, const uint64_t *key_bits, uint64_t *out_bits, void *stream)
{
    if (!h) {
        set_error("handle is NULL");
        return PA_ERR_INVALID_ARG;
    }
    return hash_impl(h, (const uint32_t *)key_bits, (uint32_t *)out_bits, 2 * ((h->m + 63) / 64),
                     (cudaStream_t)stream, true);
}

static pa_status check_strides(pa_handle h, uint64_t key_stride_words, uint64_t out_stride_words)
{
    if (key_stride_words < (h->n + 31) / 32 || out_stride_words < (h->m + 31) / 32) {
        set_error("key_stride_words = %llu (need >= %llu), out_stride_words = %llu (need >= %llu)",
                  (unsigned long long)key_stride_words, (unsigned long long)((h->n + 31) / 32),
                  (unsigned long long)out_stride_words, (unsigned long long)((h->m + 31) / 32));
        return PA_ERR_INVALID_ARG;
    }
    if ((key_stride_words & 3) || (out_stride_words & 3)) {
        set_error("strides must keep every key/output 16-byte aligned (multiples of 4 words)");
        return PA_ERR_INVALID_ARG;
    }
    return PA_OK;
}

pa_status pa_hash_batch(pa_handle h, const uint32_t *keys, uint64_t key_stride_words,
                        uint32_t *outs, uint64_t out_stride_words, uint32_t count, void *stream)
{
    if (!h) {
        set_error("handle is NULL");
        return PA_ERR_INVALID_ARG;
    }
    DeviceGuard dg(h->device);
    pa_status st;
    if ((st = check_strides(h, key_stride_words, out_stride_words)) != PA_OK) return st;
    if (count == 0) return PA_OK;
    if ((st = check_dev_ptr(keys, "keys", h->device)) != PA_OK) return st;
    if ((st = check_dev_ptr(outs, "outs", h->device)) != PA_OK) return st;
    if (overlaps(keys, ((uint64_t)(count - 1) * key_stride_words + (h->n + 31) / 32) * 4, outs,
                 ((uint64_t)(count - 1) * out_stride_words + (h->m + 31) / 32) * 4)) {
        set_error("keys and outs overlap");
        return PA_ERR_INVALID_ARG;
    }
    // growing the work buffers reallocates them: a captured pa_hash_host graph must go
    if (count > 1 && batch_grows(h, count)) drop_host_graph(h);
    return batch_impl(h, keys, key_stride_words, outs, out_stride_words, count, (h->m + 31) / 32,
                      (cudaStream_t)stream);
}

pa_status pa_hash_fresh_batch(pa_handle h, const uint32_t *seeds, uint64_t seed_stride_words,
                              const uint32_t *keys, uint64_t key_stride_words, uint32_t *outs,
                              uint64_t out_stride_words, uint32_t count, void *stream)
{
    if (!h) {
        set_error("handle is NULL");
        return PA_ERR_INVALID_ARG;
    }
    DeviceGuard dg(h->device);
    pa_status st;
    if ((st = check_strides(h, key_stride_words, out_stride_words)) != PA_OK) return st;
    if (seed_stride_words < (h->off + h->L + 31) / 32 || (seed_stride_words & 3)) {
        set_error("seed_stride_words = %llu: need >= %llu and a multiple of 4", (unsigned long long)seed_stride_words,
                  (unsigned long long)((h->off + h->L + 31) / 32));
        return PA_ERR_INVALID_ARG;
    }
    if (count == 0) return PA_OK;
    if ((st = check_dev_ptr(seeds, "seeds", h->device)) != PA_OK) return st;
    if ((st = check_dev_ptr(keys, "keys", h->device)) != PA_OK) return st;
    if ((st = check_dev_ptr(outs, "outs", h->device)) != PA_OK) return st;
    // K1 zeroes the outputs while keys and seeds are being read: no sharing with them
    const uint64_t out_bytes = ((uint64_t)(count - 1) * out_stride_words + (h->m + 31) / 32) * 4;
    if (overlaps(keys, ((uint64_t)(count - 1) * key_stride_words + (h->n + 31) / 32) * 4, outs, out_bytes) ||
        overlaps(seeds, ((uint64_t)(count - 1) * seed_stride_words + (h->off + h->L + 31) / 32) * 4, outs,
                 out_bytes)) {
        set_error("pa_hash_fresh_batch: outs overlaps keys or seeds");
        return PA_ERR_INVALID_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    if (h->route == PA_ROUTE_TRANSFORM && !h->nsub) {  // batched seed transforms + batched hashes
        st = ra_fresh_batch(h, seeds, seed_stride_words, keys, key_stride_words, outs, out_stride_words, count,
                            (h->m + 31) / 32, s);
        if (st != PA_ERR_UNSUPPORTED && st != PA_ERR_NOMEM) return st;
    }
    for (uint32_t k = 0; k < count; ++k) {  // one key at a time: set_seed + hash (less memory)
        if ((st = seed_impl(h, seeds + k * seed_stride_words, s)) != PA_OK) return st;
        if ((st = hash_impl(h, keys + k * key_stride_words, outs + k * out_stride_words, (h->m + 31) / 32, s,
                            false)) != PA_OK)
            return st;
    }
    return PA_OK;
}

// pa_hash_host's transfers.  When both host buffers are pinned (mapped into the device's
// address space), two copy kernels move the key in and the output out, PDL-chained to the hash
// kernels, instead of copy-engine nodes: the engines' latency around the hash cost more than the
// bytes (tools/dev/h2d_kernel.cu: 15.5 vs 10.2 us for 125 KB in + 31 KB out).  Measured e2e,
// Gbit/s, engines -> kernels: C2 17.9 -> 21.1, C3 41.2 -> 45.2, C4 32.1 -> 33.5, C5c 33.4 -> 42.8,
// so there is no size threshold by default.  Pageable buffers use plain copies (no graph).
__global__ void k_host_copy(const uint32_t *__restrict__ src, uint32_t *__restrict__ dst, uint64_t nw)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");  // whatever wrote src precedes us
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, nth = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i0 = 0;
    if ((((uintptr_t)src | (uintptr_t)dst) & 15) == 0) {
        const uint64_t n4 = nw / 4;
        for (uint64_t i = tid; i < n4; i += nth) ((uint4 *)dst)[i] = ((const uint4 *)src)[i];
        i0 = 4 * n4;
    }
    for (uint64_t i = i0 + tid; i < nw; i += nth) dst[i] = src[i];
}

static uint64_t host_copy_max_bytes()
{
    static const uint64_t v = [] {
        const char *e = dev_env("PA_HOST_COPY_MAX");  // developer override: 0 = always the copy engines
        return e ? (uint64_t)strtoull(e, nullptr, 0) : ~(uint64_t)0;
    }();
    return v;
}

// device-side address of a pinned host buffer, or NULL when it is pageable / not mapped
static void *mapped_ptr(const void *p)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return at.type == cudaMemoryTypeHost ? at.devicePointer : nullptr;
}

// 0: pageable buffer(s) -- plain stream-ordered copies, no graph (a captured copy needs pinned
// memory); 1: pinned, large -- graph with copy-engine nodes; 2: pinned, small -- graph with
// copy kernels
static int pick_host_copy(const pa_ctx *h, const void *key_host, const void *out_host)
{
    if (!mapped_ptr(key_host) || !mapped_ptr(out_host)) return 0;
    return (h->n + 31) / 32 * 4 > host_copy_max_bytes() ? 1 : 2;
}

static cudaError_t launch_host_copy(const uint32_t *src, uint32_t *dst, uint64_t nw, cudaStream_t s)
{
    const uint64_t blocks = (nw / 4 + 255) / 256;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(blocks < 1 ? 1 : blocks > 296 ? 296 : blocks));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_host_copy, src, dst, nw);
}

static cudaError_t set_copy_node(cudaGraphExec_t ex, cudaGraphNode_t node, const uint32_t *src, uint32_t *dst,
                                 uint64_t nw)
{
    cudaKernelNodeParams p;
    cudaError_t e = cudaGraphKernelNodeGetParams(node, &p);
    if (e != cudaSuccess) return e;
    void *args[] = {(void *)&src, (void *)&dst, (void *)&nw};
    p.kernelParams = args;
    p.extra = nullptr;
    return cudaGraphExecKernelNodeSetParams(ex, node, &p);
}

// generation of every work buffer a pa_hash_host graph may have captured (bumped by each
// reallocation, route_a.cu carve_work): a graph captured under another generation is stale
static uint64_t work_gen(const pa_ctx *h)
{
    uint64_t g = h->a.wgen;
    for (uint32_t i = 0; h->sub && i < h->nsub; ++i) g += work_gen(h->sub[i]);
    return g;
}

static void drop_host_graph(pa_ctx *h)
{
    if (h->host_exec) cudaGraphExecDestroy(h->host_exec);
    if (h->host_graph) cudaGraphDestroy(h->host_graph);
    h->host_exec = nullptr;
    h->host_graph = nullptr;
    h->h2d_node = h->d2h_node = nullptr;
    h->host_copy = 0;
    h->g_key_host = nullptr;
    h->g_out_host = nullptr;
    h->g_key_dev = nullptr;
    h->g_out_dev = nullptr;
}

// Capture H2D + the hash kernels + D2H once; later calls patch the two memcpy
// nodes' host pointers and relaunch: one graph launch instead of six API calls.
static pa_status build_host_graph(pa_ctx *h, const uint32_t *key_host, uint32_t *out_host, size_t kb, size_t ob,
                                  int mode)
{
    cudaStream_t cs;
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e, "pa_hash_host capture stream");
    pa_status st = PA_OK;
    if ((e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) {
        cudaStreamDestroy(cs);
        return cuda_fail(e, "pa_hash_host begin capture");
    }
    if (mode == 2) launch_host_copy((const uint32_t *)mapped_ptr(key_host), h->stage_key, kb / 4, cs);
    else cudaMemcpyAsync(h->stage_key, key_host, kb, cudaMemcpyHostToDevice, cs);
    st = hash_impl(h, h->stage_key, h->stage_out, (h->m + 31) / 32, cs, false);
    if (mode == 2) launch_host_copy(h->stage_out, (uint32_t *)mapped_ptr(out_host), ob / 4, cs);
    else cudaMemcpyAsync(out_host, h->stage_out, ob, cudaMemcpyDeviceToHost, cs);
    cudaGraph_t g = nullptr;
    e = cudaStreamEndCapture(cs, &g);
    cudaStreamDestroy(cs);
    if (st != PA_OK || e != cudaSuccess || !g) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        return st != PA_OK ? st : cuda_fail(e, "pa_hash_host end capture");
    }
    size_t nn = 0;
    cudaGraphGetNodes(g, nullptr, &nn);
    cudaGraphNode_t nodes[64];
    if (nn > 64) nn = 64;
    cudaGraphGetNodes(g, nodes, &nn);
    cudaGraphNode_t h2d = nullptr, d2h = nullptr;
    for (size_t i = 0; i < nn; ++i) {
        cudaGraphNodeType ty;
        cudaGraphNodeGetType(nodes[i], &ty);
        if (mode == 2 && ty == cudaGraphNodeTypeKernel) {
            cudaKernelNodeParams kp;
            cudaGraphKernelNodeGetParams(nodes[i], &kp);
            if (kp.func != (void *)k_host_copy) continue;
            const uint32_t *dst = *(uint32_t *const *)kp.kernelParams[1];
            if (dst == h->stage_key) h2d = nodes[i];
            else d2h = nodes[i];
            continue;
        }
        if (mode != 1 || ty != cudaGraphNodeTypeMemcpy) continue;
        cudaMemcpy3DParms pr;
        cudaGraphMemcpyNodeGetParams(nodes[i], &pr);
        if (pr.kind == cudaMemcpyHostToDevice || pr.dstPtr.ptr == h->stage_key) h2d = nodes[i];
        else d2h = nodes[i];
    }
    cudaGraphExec_t ex = nullptr;
    if (!h2d || !d2h || (e = cudaGraphInstantiate(&ex, g, 0)) != cudaSuccess) {
        cudaGraphDestroy(g);
        cudaGetLastError();
        return cuda_fail(e == cudaSuccess ? cudaErrorUnknown : e, "pa_hash_host graph instantiate");
    }
    h->host_graph = g;
    h->host_exec = ex;
    h->h2d_node = h2d;
    h->d2h_node = d2h;
    h->host_copy = mode;
    h->g_key_host = key_host;
    h->g_out_host = out_host;
    h->g_key_dev = mode == 2 ? mapped_ptr(key_host) : nullptr;
    h->g_out_dev = mode == 2 ? mapped_ptr(out_host) : nullptr;
    h->g_wgen = work_gen(h);
    return PA_OK;
}

static pa_status hash_host_impl(pa_handle h, const uint32_t *key_host, uint32_t *out_host, void *stream,
                                bool sync)
{
    if (!h || !key_host || !out_host) {
        set_error("pa_hash_host: NULL argument (h=%p key_host=%p out_host=%p)", (void *)h,
                  (const void *)key_host, (void *)out_host);
        return PA_ERR_INVALID_ARG;
    }
    DeviceGuard dg(h->device);
    cudaStream_t s = (cudaStream_t)stream;
    size_t kb = ((h->n + 31) / 32) * 4, ob = ((h->m + 31) / 32) * 4;
    cudaError_t e;
    if (!h->stage_blk) {  // library-owned memory: staging on first use
        pa_status st = dev_alloc(h, (void **)&h->stage_blk, stage_bytes(h->n, h->m), "pa_hash_host staging");
        if (st != PA_OK) return st;
        h->stage_key = (uint32_t *)h->stage_blk;
        h->stage_out = (uint32_t *)(h->stage_blk + al256(kb));
    }
    // a graph captured before the work buffers moved (a larger batch / fresh-seed batch since)
    // holds stale kernel arguments: capture again
    if (h->host_exec && work_gen(h) != h->g_wgen) drop_host_graph(h);
    // copy kernels address the host buffers through their mapped device pointers: re-derive them
    // every call (a freed pinned buffer's address may come back pageable or mapped elsewhere)
    const void *kdev = mapped_ptr(key_host);
    void *odev = mapped_ptr(out_host);
    if (h->host_exec && h->host_copy == 2 && (!kdev || !odev)) drop_host_graph(h);
    const bool moved = key_host != h->g_key_host || out_host != h->g_out_host || kdev != h->g_key_dev ||
                       odev != h->g_out_dev;
    const int mode = h->host_exec && !moved ? h->host_copy : !kdev || !odev ? 0 : pick_host_copy(h, key_host, out_host);
    if (h->prof.on || mode == 0) {  // per-launch profiling events need the plain launches
        if ((e = cudaMemcpyAsync(h->stage_key, key_host, kb, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return cuda_fail(e, "pa_hash_host H2D");
        pa_status st = hash_impl(h, h->stage_key, h->stage_out, (h->m + 31) / 32, s, false);
        if (st != PA_OK) return st;
        if ((e = cudaMemcpyAsync(out_host, h->stage_out, ob, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
            return cuda_fail(e, "pa_hash_host D2H");
    } else {
        if (h->host_exec && mode != h->host_copy) drop_host_graph(h);  // pinned <-> pageable: other nodes
        if (!h->host_exec) {
            pa_status st = build_host_graph(h, key_host, out_host, kb, ob, mode);
            if (st != PA_OK) return st;
        }
        if (key_host != h->g_key_host || (mode == 2 && kdev != h->g_key_dev)) {
            e = mode == 2 ? set_copy_node(h->host_exec, h->h2d_node, (const uint32_t *)kdev, h->stage_key, kb / 4)
                          : cudaGraphExecMemcpyNodeSetParams1D(h->host_exec, h->h2d_node, h->stage_key, key_host,
                                                               kb, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return cuda_fail(e, "pa_hash_host graph update (key)");
            h->g_key_host = key_host;
            h->g_key_dev = mode == 2 ? kdev : nullptr;
        }
        if (out_host != h->g_out_host || (mode == 2 && odev != h->g_out_dev)) {
            e = mode == 2 ? set_copy_node(h->host_exec, h->d2h_node, h->stage_out, (uint32_t *)odev, ob / 4)
                          : cudaGraphExecMemcpyNodeSetParams1D(h->host_exec, h->d2h_node, out_host, h->stage_out,
                                                               ob, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) return cuda_fail(e, "pa_hash_host graph update (out)");
            h->g_out_host = out_host;
            h->g_out_dev = mode == 2 ? odev : nullptr;
        }
        if ((e = cudaGraphLaunch(h->host_exec, s)) != cudaSuccess) return cuda_fail(e, "pa_hash_host graph launch");
    }
    if (sync && (e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "pa_hash_host sync");
    return PA_OK;
}

pa_status pa_hash_host_batch(pa_handle h, const uint32_t *keys_host, uint64_t key_stride_words,
                             uint32_t *outs_host, uint64_t out_stride_words, uint32_t count, void *stream)
{
    if (!h || !keys_host || !outs_host) {
        set_error("pa_hash_host_batch: NULL argument");
        return PA_ERR_INVALID_ARG;
    }
    DeviceGuard dg(h->device);
    const uint64_t kw = (h->n + 31) / 32, ow = (h->m + 31) / 32;
    if (key_stride_words < kw || out_stride_words < ow) {
        set_error("pa_hash_host_batch: key_stride_words = %llu (need >= %llu), out_stride_words = %llu (need >= "
                  "%llu)", (unsigned long long)key_stride_words, (unsigned long long)kw,
                  (unsigned long long)out_stride_words, (unsigned long long)ow);
        return PA_ERR_INVALID_ARG;
    }
    if (count == 0) return PA_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (h->arena) {  // a workspace handle allocates nothing more: one key at a time
        for (uint32_t k = 0; k < count; ++k) {
            pa_status st = hash_host_impl(h, keys_host + k * key_stride_words, outs_host + k * out_stride_words,
                                          stream, k + 1 == count);
            if (st != PA_OK) return st;
        }
        return PA_OK;
    }
    // Chunks of keys in a software pipeline over two staging slots: the copy stream moves chunk
    // i+1's keys in and chunk i-1's outputs out (copy engines, PCIe) while `stream` hashes chunk
    // i, so the transfers hide behind the kernels except the first chunk's H2D and the last D2H.
    const uint64_t kw4 = (kw + 3) / 4 * 4, ow4 = (ow + 3) / 4 * 4;
    const pa_ctx *leaf = h->nsub ? h->sub[0] : h;
    uint32_t chunk = leaf->route == PA_ROUTE_TRANSFORM ? ra_batch_keys(leaf) : 4096;
    // at least four chunks when the keys allow, so that the copies of neighbouring chunks have
    // a hash to hide behind (one chunk of all keys serialises H2D, hash and D2H: C3 x 16 keys
    // 221 us per key against ~153 us of kernels)
    const uint32_t quarter = (count + 3) / 4;
    if (chunk > quarter) chunk = quarter;
    if (chunk > count) chunk = count;
    if (chunk == 0) chunk = 1;
    const uint32_t nslot = count > chunk ? 2 : 1;
    const size_t slot_words = (size_t)chunk * (kw4 + ow4), need = nslot * slot_words * 4;
    cudaError_t e;
    if (need > h->bstage_bytes) {
        if (h->bstage) {
            cudaStreamSynchronize(s);
            cudaFree(h->bstage);
            h->bstage = nullptr;
            h->bstage_bytes = 0;
        }
        if ((e = cudaMalloc(&h->bstage, need)) != cudaSuccess) {
            h->bstage = nullptr;
            cudaGetLastError();
            set_error("pa_hash_host_batch: staging of %llu bytes: %s", (unsigned long long)need,
                      cudaGetErrorString(e));
            return PA_ERR_NOMEM;
        }
        h->bstage_bytes = need;
    }
    if (!h->cstream) {
        if ((e = cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking)) != cudaSuccess)
            return cuda_fail(e, "pa_hash_host_batch copy stream");
        for (cudaEvent_t &ev : h->pev)
            if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(e, "pa_hash_host_batch events");
    }
    if (chunk > 1 && batch_grows(h, chunk)) drop_host_graph(h);  // work buffers are about to move
    cudaStream_t cs = h->cstream;
    cudaEvent_t *h2d = h->pev, *comp = h->pev + 2, start = h->pev[4];
    // an error mid-pipeline: copies into the caller's host buffers may be in flight on the copy
    // stream -- let them finish before returning, so the caller may free / reuse the buffers
    auto fail = [&](pa_status st) {
        cudaStreamSynchronize(cs);
        cudaStreamSynchronize(s);
        return st;
    };
    auto kslot = [&](uint32_t i) { return (uint32_t *)h->bstage + (i % nslot) * slot_words; };
    auto oslot = [&](uint32_t i) { return kslot(i) + (size_t)chunk * kw4; };
    auto keys_of = [&](uint32_t i) { return count - i * chunk < chunk ? count - i * chunk : chunk; };
    auto h2d_chunk = [&](uint32_t i) {
        return cudaMemcpy2DAsync(kslot(i), kw4 * 4, keys_host + (size_t)i * chunk * key_stride_words,
                                 key_stride_words * 4, kw * 4, keys_of(i), cudaMemcpyHostToDevice, cs);
    };
    const uint32_t nch = (count + chunk - 1) / chunk;
    cudaEventRecord(start, s);  // earlier work on `stream` may still use the staging / work buffers
    cudaStreamWaitEvent(cs, start, 0);
    if ((e = h2d_chunk(0)) != cudaSuccess) return fail(cuda_fail(e, "pa_hash_host_batch H2D"));
    cudaEventRecord(h2d[0], cs);
    for (uint32_t i = 0; i < nch; ++i) {
        const uint32_t sl = i % nslot;
        if (i + 1 < nch) {  // next chunk's keys, once chunk i-1 (same slot) has consumed its own
            if (i >= 1) cudaStreamWaitEvent(cs, comp[(i + 1) % nslot], 0);
            if ((e = h2d_chunk(i + 1)) != cudaSuccess) return fail(cuda_fail(e, "pa_hash_host_batch H2D"));
            cudaEventRecord(h2d[(i + 1) % nslot], cs);
        }
        // chunk i-2's outputs left this slot before chunk i's keys arrived (copy stream order)
        cudaStreamWaitEvent(s, h2d[sl], 0);
        pa_status st = batch_impl(h, kslot(i), kw4, oslot(i), ow4, keys_of(i), ow, s);
        if (st != PA_OK) return fail(st);
        cudaEventRecord(comp[sl], s);
        cudaStreamWaitEvent(cs, comp[sl], 0);
        if ((e = cudaMemcpy2DAsync(outs_host + (size_t)i * chunk * out_stride_words, out_stride_words * 4, oslot(i),
                                   ow4 * 4, ow * 4, keys_of(i), cudaMemcpyDeviceToHost, cs)) != cudaSuccess)
            return fail(cuda_fail(e, "pa_hash_host_batch D2H"));
    }
    cudaEventRecord(start, cs);
    cudaStreamWaitEvent(s, start, 0);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "pa_hash_host_batch sync");
    return PA_OK;
}

pa_status pa_hash_host(pa_handle h, const uint32_t *key_host, uint32_t *out_host, void *stream)
{
    return hash_host_impl(h, key_host, out_host, stream, true);
}

pa_status pa_hash_host_async(pa_handle h, const uint32_t *key_host, uint32_t *out_host, void *stream)
{
    return hash_host_impl(h, key_host, out_host, stream, false);
}

pa_status pa_residual(pa_handle h, double *max_residual, void *stream)
{
    if (!h || !max_residual) {
        set_error("pa_residual: NULL argument");
        return PA_ERR_INVALID_ARG;
    }
    DeviceGuard dg(h->device);
    *max_residual = 0.0;
    if (h->route != PA_ROUTE_TRANSFORM) return PA_OK;
    cudaStream_t s = (cudaStream_t)stream;
    double r = 0.0;
    const uint32_t nb = h->nsub ? h->nsub : 1;
    for (uint32_t g = 0; g < nb; ++g) {  // max over the column blocks of a split handle
        pa_ctx *b = h->nsub ? h->sub[g] : h;
        unsigned long long bits = 0;
        cudaError_t e;
        if ((e = cudaMemcpyAsync(&bits, b->a.resid, sizeof bits, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
            (e = cudaStreamSynchronize(s)) != cudaSuccess ||
            (e = cudaMemsetAsync(b->a.resid, 0, sizeof bits, s)) != cudaSuccess)
            return cuda_fail(e, "pa_residual");
        double rb;
        memcpy(&rb, &bits, sizeof rb);
        if (rb > r) r = rb;
    }
    *max_residual = r;
    if (r > PA_RESIDUAL_LIMIT) {
        set_error("FP64 residual %.3e exceeds PA_RESIDUAL_LIMIT %.2f", r, PA_RESIDUAL_LIMIT);
        return PA_ERR_PRECISION;
    }
    return PA_OK;
}

pa_status pa_profile_enable(pa_handle h, int enable)
{
    if (!h) {
        set_error("pa_profile_enable: handle is NULL");
        return PA_ERR_INVALID_ARG;
    }
    h->prof.on = enable != 0;
    return PA_OK;
}

pa_status pa_profile_read(pa_handle h, pa_kernel_time *out, uint32_t max, uint32_t *count)
{
    if (!h || (!out && max) || !count) {
        set_error("pa_profile_read: NULL argument");
        return PA_ERR_INVALID_ARG;
    }
    Profiler &P = h->prof;
    for (int i = 0; i < P.npend; ++i) {
        Profiler::Pending &q = P.pend[i];
        if (q.e0 && q.e1) {
            cudaError_t e = cudaEventSynchronize(q.e1);
            if (e != cudaSuccess) return cuda_fail(e, "pa_profile_read");
            float ms = 0.f;
            cudaEventElapsedTime(&ms, q.e0, q.e1);
            P.launches[q.k] += 1;
            P.total_ms[q.k] += ms;
        }
        prof_release(P, q.e0);
        prof_release(P, q.e1);
    }
    P.npend = 0;
    uint32_t n = 0;
    for (int k = 0; k < Profiler::kKernels; ++k) {
        if (!P.launches[k]) continue;
        if (n < max) {
            memset(out[n].name, 0, sizeof out[n].name);
            strncpy(out[n].name, P.names[k], sizeof out[n].name - 1);
            out[n].launches = P.launches[k];
            out[n].total_ms = P.total_ms[k];
        }
        ++n;
        P.launches[k] = 0;
        P.total_ms[k] = 0;
    }
    *count = n < max ? n : max;
    return PA_OK;
}

pa_status pa_plan(uint64_t n, uint64_t m, pa_info *info)
{
    if (!info || n == 0 || m == 0) {
        set_error("pa_plan: need info != NULL and n, m >= 1 (n = %llu, m = %llu)", (unsigned long long)n,
                  (unsigned long long)m);
        return PA_ERR_INVALID_ARG;
    }
    memset(info, 0, sizeof *info);
    info->n = n;
    info->m = m;
    info->route = choose_route(n, m);
    info->device = -1;
    if (info->route == PA_ROUTE_BITPACKED) {
        info->workspace_bytes = rb_bytes(n, m);
        info->kernels_per_hash = 1;
        info->column_blocks = 1;
        return PA_OK;
    }
    // the column split pa_create falls back to when no single transform can be planned
    std::vector<uint64_t> c0;
    pa_status st = split_plan(n, m, 0, &c0);
    if (st != PA_OK) return st;
    Geometry g;
    char err[256];
    const uint64_t n0 = c0.size() > 1 ? c0[1] : n;
    if ((st = ra_plan(n0, m, &g, err, sizeof err, c0.size() > 1 ? kMaxPlanLen : 0)) != PA_OK) {
        set_error("%s", err);
        return st;
    }
    info->transform_len = 2 * g.M;
    info->n1 = g.N1;
    info->n2 = g.N2;
    info->cols_per_cta = g.C;
    info->k3_cols_per_cta = g.C3;
    pa_options o;
    pa_options_init(&o);
    o.route = PA_ROUTE_TRANSFORM;
    size_t b = 0;
    if ((st = handle_bytes(n, m, o, false, &b)) != PA_OK) return st;
    info->workspace_bytes = b;
    info->kernels_per_hash = (uint64_t)c0.size() * (g.C >= 16 ? 3 : 4);
    info->column_blocks = c0.size();
    return PA_OK;
}

pa_status pa_get_info(pa_handle h, pa_info *info)
{
    if (!h || !info) {
        set_error("pa_get_info: NULL argument");
        return PA_ERR_INVALID_ARG;
    }
    memset(info, 0, sizeof *info);
    info->n = h->n;
    info->m = h->m;
    info->route = h->route;
    info->device = h->device;
    info->column_blocks = h->nsub ? h->nsub : 1;
    info->workspace_bytes = h->ws_bytes;
    for (uint32_t g = 0; g < h->nsub; ++g) info->workspace_bytes += h->sub[g]->ws_bytes;
    // geometry: the handle's own, or its first (largest) column block's
    const pa_ctx *b = h->nsub ? h->sub[0] : h;
    if (h->route == PA_ROUTE_TRANSFORM) {
        info->transform_len = 2 * b->a.g.M;
        info->n1 = b->a.g.N1;
        info->n2 = b->a.g.N2;
        info->cols_per_cta = b->a.g.C;
        info->k3_cols_per_cta = b->a.g.C3;
    }
    info->kernels_per_hash = h->kernels_per_hash;
    return PA_OK;
}

}  // extern "C"
