// pa_api.cu -- the C ABI declared in include/pa.h: argument validation, route
// selection and dispatch.  No exceptions cross this boundary.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <new>
#include <string>

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

static cudaEvent_t prof_event(Profiler &P)
{
    if (P.npool > 0) return P.pool[--P.npool];
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}

void prof_begin(pa_ctx *h, int k, cudaStream_t s)
{
    Profiler &P = h->prof;
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
    Profiler &P = h->prof;
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
    return PA_OK;
}

void pa_destroy(pa_handle h)
{
    if (!h) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(h->device);
    prof_free(h->prof);
    drop_host_graph(h);
    ra_destroy(h);
    rb_destroy(h);
    if (h->stage_key) cudaFree(h->stage_key);
    if (h->stage_out) cudaFree(h->stage_out);
    cudaSetDevice(prev);
    delete h;
}

pa_status pa_create_ex(pa_handle *out, uint64_t n, uint64_t m, const uint32_t *seed_bits,
                       const pa_options *opt, void *stream)
{
    if (!out) {
        set_error("h (output handle pointer) is NULL");
        return PA_ERR_INVALID_ARG;
    }
    *out = nullptr;
    pa_options o;
    pa_options_init(&o);
    if (opt) {
        if (opt->struct_size != sizeof(pa_options)) {
            set_error("opt->struct_size = %u, expected %u (call pa_options_init)",
                      opt->struct_size, (unsigned)sizeof(pa_options));
            return PA_ERR_INVALID_ARG;
        }
        o = *opt;
    }
    if (n == 0 || m == 0 || (m > n && !o.allow_wide)) {
        set_error("need 1 <= m <= n (or opt->allow_wide), got n = %llu, m = %llu",
                  (unsigned long long)n, (unsigned long long)m);
        return PA_ERR_INVALID_ARG;
    }
    if (n > (1ull << 40) || m > (1ull << 40)) {
        set_error("n = %llu, m = %llu: lengths beyond 2^40 bits are unsupported",
                  (unsigned long long)n, (unsigned long long)m);
        return PA_ERR_UNSUPPORTED;
    }
    if (o.route < PA_ROUTE_AUTO || o.route > PA_ROUTE_BITPACKED) {
        set_error("opt->route = %d is not a pa_route", o.route);
        return PA_ERR_INVALID_ARG;
    }
    if (o.allow_wide > 1) {
        set_error("opt->allow_wide = %u must be 0 or 1", o.allow_wide);
        return PA_ERR_INVALID_ARG;
    }
    for (int i = 0; i < 7; ++i)
        if (o.reserved[i]) {
            set_error("opt->reserved[%d] = %u must be 0", i, o.reserved[i]);
            return PA_ERR_INVALID_ARG;
        }
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    pa_status st = check_dev_ptr(seed_bits, "seed_bits", dev);
    if (st != PA_OK) return st;

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
    h->route = o.route == PA_ROUTE_AUTO ? choose_route(n, m) : o.route;
    cudaStream_t s = (cudaStream_t)stream;
    st = h->route == PA_ROUTE_TRANSFORM ? ra_create(h, seed_bits, s) : rb_create(h, seed_bits, s);
    if (st != PA_OK) {
        std::string keep = g_err;
        pa_destroy(h);
        g_err = keep;
        return st;
    }
    *out = h;
    return PA_OK;
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

pa_status pa_set_seed(pa_handle h, const uint32_t *seed_bits, void *stream)
{
    if (!h) {
        set_error("handle is NULL");
        return PA_ERR_INVALID_ARG;
    }
    pa_status st = check_dev_ptr(seed_bits, "seed_bits", h->device);
    if (st != PA_OK) return st;
    return h->route == PA_ROUTE_TRANSFORM ? ra_seed(h, seed_bits, (cudaStream_t)stream)
                                          : rb_seed(h, seed_bits, (cudaStream_t)stream);
}

static pa_status hash_impl(pa_handle h, const uint32_t *key, uint32_t *out, uint64_t zero_words,
                           cudaStream_t s, bool validate)
{
    if (!h) {
        set_error("handle is NULL");
        return PA_ERR_INVALID_ARG;
    }
    if (validate) {
        pa_status st;
        if (key != h->ok_key) {
            if ((st = check_dev_ptr(key, "key_bits", h->device)) != PA_OK) return st;
            h->ok_key = key;
        }
        if (out != h->ok_out) {
            if ((st = check_dev_ptr(out, "out_bits", h->device)) != PA_OK) return st;
            h->ok_out = out;
        }
    }
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

pa_status pa_hash_batch(pa_handle h, const uint32_t *keys, uint64_t key_stride_words,
                        uint32_t *outs, uint64_t out_stride_words, uint32_t count, void *stream)
{
    if (!h) {
        set_error("handle is NULL");
        return PA_ERR_INVALID_ARG;
    }
    if (key_stride_words < (h->n + 31) / 32 || out_stride_words < (h->m + 31) / 32) {
        set_error("key_stride_words = %llu (need >= %llu), out_stride_words = %llu (need >= %llu)",
                  (unsigned long long)key_stride_words, (unsigned long long)((h->n + 31) / 32),
                  (unsigned long long)out_stride_words, (unsigned long long)((h->m + 31) / 32));
        return PA_ERR_INVALID_ARG;
    }
    if (count == 0) return PA_OK;
    if ((key_stride_words & 3) || (out_stride_words & 3)) {
        set_error("strides must keep every key/output 16-byte aligned (multiples of 4 words)");
        return PA_ERR_INVALID_ARG;
    }
    pa_status st;
    if ((st = check_dev_ptr(keys, "keys", h->device)) != PA_OK) return st;
    if ((st = check_dev_ptr(outs, "outs", h->device)) != PA_OK) return st;
    if (h->route == PA_ROUTE_TRANSFORM) {
        // keys in chunks: all kernels take the key index from the grid.  Growing the
        // work buffers reallocates them: a captured pa_hash_host graph must go.
        if (count > 1 && h->a.cap < (count < ra_batch_keys(h) ? count : ra_batch_keys(h))) drop_host_graph(h);
        const uint32_t chunk = ra_batch_keys(h);
        for (uint32_t k0 = 0; k0 < count; k0 += chunk) {
            const uint32_t c = count - k0 < chunk ? count - k0 : chunk;
            st = ra_hash_batch(h, keys + k0 * key_stride_words, key_stride_words, outs + k0 * out_stride_words,
                               out_stride_words, c, (h->m + 31) / 32, (cudaStream_t)stream);
            if (st != PA_OK) return st;
        }
        return PA_OK;
    }
    for (uint32_t k = 0; k < count; ++k) {
        st = hash_impl(h, keys + k * key_stride_words, outs + k * out_stride_words,
                       (h->m + 31) / 32, (cudaStream_t)stream, false);
        if (st != PA_OK) return st;
    }
    return PA_OK;
}

static void drop_host_graph(pa_ctx *h)
{
    if (h->host_exec) cudaGraphExecDestroy(h->host_exec);
    if (h->host_graph) cudaGraphDestroy(h->host_graph);
    h->host_exec = nullptr;
    h->host_graph = nullptr;
    h->h2d_node = h->d2h_node = nullptr;
    h->g_key_host = nullptr;
    h->g_out_host = nullptr;
}

// Capture H2D + the hash kernels + D2H once; later calls patch the two memcpy
// nodes' host pointers and relaunch: one graph launch instead of six API calls.
static pa_status build_host_graph(pa_ctx *h, const uint32_t *key_host, uint32_t *out_host, size_t kb, size_t ob)
{
    cudaStream_t cs;
    cudaError_t e = cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e, "pa_hash_host capture stream");
    pa_status st = PA_OK;
    if ((e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) {
        cudaStreamDestroy(cs);
        return cuda_fail(e, "pa_hash_host begin capture");
    }
    cudaMemcpyAsync(h->stage_key, key_host, kb, cudaMemcpyHostToDevice, cs);
    st = hash_impl(h, h->stage_key, h->stage_out, (h->m + 31) / 32, cs, false);
    cudaMemcpyAsync(out_host, h->stage_out, ob, cudaMemcpyDeviceToHost, cs);
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
        if (ty != cudaGraphNodeTypeMemcpy) continue;
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
    h->g_key_host = key_host;
    h->g_out_host = out_host;
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
    cudaStream_t s = (cudaStream_t)stream;
    size_t kb = ((h->n + 31) / 32) * 4, ob = ((h->m + 31) / 32) * 4;
    cudaError_t e;
    if (!h->stage_key) {
        if ((e = cudaMalloc(&h->stage_key, kb)) != cudaSuccess) {
            h->stage_key = nullptr;
            return cuda_fail(e, "pa_hash_host staging alloc");
        }
        if ((e = cudaMalloc(&h->stage_out, ob)) != cudaSuccess) {
            h->stage_out = nullptr;
            return cuda_fail(e, "pa_hash_host staging alloc");
        }
        h->ws_bytes += kb + ob;
    }
    if (h->prof.on) {  // per-launch profiling events need the plain launches
        if ((e = cudaMemcpyAsync(h->stage_key, key_host, kb, cudaMemcpyHostToDevice, s)) != cudaSuccess)
            return cuda_fail(e, "pa_hash_host H2D");
        pa_status st = hash_impl(h, h->stage_key, h->stage_out, (h->m + 31) / 32, s, false);
        if (st != PA_OK) return st;
        if ((e = cudaMemcpyAsync(out_host, h->stage_out, ob, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
            return cuda_fail(e, "pa_hash_host D2H");
    } else {
        if (!h->host_exec) {
            pa_status st = build_host_graph(h, key_host, out_host, kb, ob);
            if (st != PA_OK) return st;
        }
        if (key_host != h->g_key_host) {
            if ((e = cudaGraphExecMemcpyNodeSetParams1D(h->host_exec, h->h2d_node, h->stage_key, key_host, kb,
                                                        cudaMemcpyHostToDevice)) != cudaSuccess)
                return cuda_fail(e, "pa_hash_host graph update (key)");
            h->g_key_host = key_host;
        }
        if (out_host != h->g_out_host) {
            if ((e = cudaGraphExecMemcpyNodeSetParams1D(h->host_exec, h->d2h_node, out_host, h->stage_out, ob,
                                                        cudaMemcpyDeviceToHost)) != cudaSuccess)
                return cuda_fail(e, "pa_hash_host graph update (out)");
            h->g_out_host = out_host;
        }
        if ((e = cudaGraphLaunch(h->host_exec, s)) != cudaSuccess) return cuda_fail(e, "pa_hash_host graph launch");
    }
    if (sync && (e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "pa_hash_host sync");
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
    *max_residual = 0.0;
    if (h->route != PA_ROUTE_TRANSFORM) return PA_OK;
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long bits = 0;
    cudaError_t e;
    if ((e = cudaMemcpyAsync(&bits, h->a.resid, sizeof bits, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess ||
        (e = cudaMemsetAsync(h->a.resid, 0, sizeof bits, s)) != cudaSuccess)
        return cuda_fail(e, "pa_residual");
    double r;
    memcpy(&r, &bits, sizeof r);
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
        info->workspace_bytes = 4 * ((m + 31) / 32 + (n + 31) / 32 + 4);
        info->kernels_per_hash = 1;
        return PA_OK;
    }
    Geometry g;
    char err[256];
    pa_status st = ra_plan(n, m, &g, err, sizeof err);
    if (st != PA_OK) {
        set_error("%s", err);
        return st;
    }
    info->transform_len = 2 * g.M;
    info->n1 = g.N1;
    info->n2 = g.N2;
    info->cols_per_cta = g.C;
    info->workspace_bytes = 32 * g.M + (uint64_t)(g.N1 / g.C) * g.kbw * 4;
    info->kernels_per_hash = 4;
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
    if (h->route == PA_ROUTE_TRANSFORM) {
        info->transform_len = 2 * h->a.g.M;
        info->n1 = h->a.g.N1;
        info->n2 = h->a.g.N2;
        info->cols_per_cta = h->a.g.C;
    }
    info->workspace_bytes = h->ws_bytes;
    info->kernels_per_hash = h->kernels_per_hash;
    return PA_OK;
}

}  // extern "C"
