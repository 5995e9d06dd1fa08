// route_a.cu -- route (a): exact integer convolution by an FP64 transform.
//
// The paper recasts r = uT as a polynomial product (Sec. 3 Steps 1-3,
// P:128-136): zero-pad, FFT both, multiply, IFFT, take the window
// [n-1, n+m-1) (one-based "nth to (n+k-1)th") and reduce mod 2.  Here:
//
//  * Length (reading R4): a wrap-free window needs only N >= n+m-1
//    real points (not the paper's 2n+l-2), and the NEGACYCLIC product mod
//    X^N + 1 serves as well as the cyclic one (wrapped terms land below n-1).
//    A real negacyclic product of length N = 2M is a complex cyclic product of
//    length M of the "right-angle" packed, twisted sequence
//        z[u] = (x[u] + i x[u+M]) * zeta^u,   zeta = exp(i pi / N),  u < M,
//    so every transform is a plain complex DFT of length M (no real-to-complex
//    post-pass), 16 bytes per 2 real points.
//  * Four-step split M = N1 * N2, u = a + N1 b (a < N1 contiguous), frequency
//    k = N2 k_a + k_b; all kernels launched with programmatic dependent launch:
//      K0  bit transpose of the key into one bit stream per K1 column group
//          (skipped when C = 16: K1 then gathers its 2-byte runs itself).
//      K1  strided pass, C columns per CTA: z = (x_re + i x_im) theta_b
//          (theta_b = zeta^{N1 b}), DIF over b (N2 points) in shared memory,
//          stored to the [N2][N1] work array (row = DIF output position p,
//          k_b = rev2[p]); zeroes the output words.
//      K2  row pass, one row per CTA: the first DIF stage reads the row from
//          HBM and multiplies by tau(a, k_b) = rho^a (four-step twiddle and
//          column twist as one per-row power, tables built at create), DIF over
//          a, [last DIF stage * spectrum * first DIT stage] fused in registers
//          (spectrum in the same digit-reversed order, scaled by 1/M), DIT, the
//          last stage multiplying by conj rho^a and storing to global memory.
//      K3  strided pass: the C-column tile (cp.async, or read by the first DIT
//          stage when C >= 4), DIT over k_b -> natural b, then the epilogue:
//          untwist by conj theta_b, keep t in [n-1, n+m-1) (Re part = c[u], Im
//          part = c[u+M]), rint, &1, ballot-pack runs of C bits, atomicXor into
//          the output words; records max |v - rint(v)| (PA_ERR_PRECISION).
//  * The seed goes through K0, K1 and K2's forward half once at create.
//  * Opt-in variants (measured): a TMEM-staged persistent K3
//    (k3t_inv_columns, PA_K3T=1) and a row-block layout of K2's output
//    (PA_LR=1).
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <atomic>
#include <vector>

#include "bits.cuh"
#include "fft_core.cuh"
#include "pa_internal.h"

namespace pa {
namespace {

constexpr uint32_t kSmemLimit = 232448;  // 227 KB opt-in dynamic shared memory per CTA
#ifndef PA_TMAX
#define PA_TMAX 512
#endif
#ifndef PA_MINB
#define PA_MINB 1
#endif

#ifdef PA_TIMING
__device__ unsigned long long g_k2_clk[3][64][16];
#ifndef PA_STAMP_BASE
#define PA_STAMP_BASE 0  // first CTA recorded (e.g. 2048: a steady-state wave of a many-wave grid)
#endif
#define TSTAMPK(k, i) do { __syncthreads(); const unsigned _lb = blockIdx.x + gridDim.x * blockIdx.y - PA_STAMP_BASE; \
    if (threadIdx.x == 0 && _lb < 64) g_k2_clk[k][_lb][i] = clock64(); } while (0)
#define TSTAMP(i) TSTAMPK(1, i)
__device__ unsigned long long g_trace[4][8192][3];  // per kernel (K0..K3), per CTA: smid, start, end ns
__device__ __forceinline__ unsigned long long gtimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid()
{
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}
#define TRACE_BEGIN(k) unsigned long long _t0 = gtimer()
#define TRACE_END(k) do { __syncthreads(); if (threadIdx.x == 0 && blockIdx.x + gridDim.x * blockIdx.y < 8192) { \
    unsigned _b = blockIdx.x + gridDim.x * blockIdx.y; g_trace[k][_b][0] = smid(); g_trace[k][_b][1] = _t0; \
    g_trace[k][_b][2] = gtimer(); } } while (0)
#else
#define TSTAMP(i) do { } while (0)
#define TSTAMPK(k, i) do { } while (0)
#define TRACE_BEGIN(k) do { } while (0)
#define TRACE_END(k) do { } while (0)
#endif

// Programmatic dependent launch: the prologue (tables, per-row constants) of a
// kernel overlaps the tail of the previous one; grid_dep_wait() blocks until the
// previous grid has completed and its memory is visible.
// Layout of the array K2 writes and K3 reads (buf2).  Element (row b, column a): rows are
// grouped in blocks of R = 2^lr and columns in groups of C, and an R x C block of a column
// group is contiguous -- K3's loads of a C-column group move runs of 16 C R bytes (128 B for
// C = 2, R = 4) instead of 16 C, while K2 writes its row as C-element pieces at a 16 C R-byte
// stride (stores do not stall; K2's reads stay row-major in buf: as pieces they measured 15%
// slower).  lr = 0: plain row-major and buf2 == buf (K2 in place).
__device__ __forceinline__ uint64_t wrow(const Geometry &g, uint32_t b)
{
    return (((uint64_t)(b >> g.lr) * g.N1) << g.lr) + ((uint64_t)(b & ((1u << g.lr) - 1)) << g.logC);
}
__device__ __forceinline__ uint32_t wcol(const Geometry &g, uint32_t a)
{
    return ((a >> g.logC) << (g.logC + g.lr)) + (a & (g.C - 1));
}

__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void grid_dep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem)
{
    unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// The four-step twiddle and the twist's column factor, tau(a, k_b) =
// zeta^a omega_M^{a k_b} = rho^a with rho = exp(2 pi i (1 - 4 k_b) / 4M), are a
// power of one per-row constant: K2 builds rho^e (e < 64) and rho^{64 h} in
// shared memory with sincospi of the exact integer exponent.
__device__ __forceinline__ void rho_tables(double2 *rlo, double2 *rhi, uint32_t nhi, uint64_t M, uint32_t kb)
{
    const int64_t M4 = 4 * (int64_t)M;
    const int64_t step = 1 - 4 * (int64_t)kb;  // exponent of rho in units of 2 pi i / 4M
    for (uint32_t i = threadIdx.x; i < 64 + nhi; i += blockDim.x) {
        int64_t e = (i < 64) ? (int64_t)i : 64 * (int64_t)(i - 64);
        int64_t E = (e % M4) * (step % M4) % M4;
        if (E < 0) E += M4;
        double s, c;
        sincospi((double)E / (double)(2 * M), &s, &c);
        if (i < 64) rlo[i] = make_double2(c, s);
        else rhi[i - 64] = make_double2(c, s);
    }
}

__device__ __forceinline__ void load_tables(double2 *wlo, double2 *whi, const double2 *glo,
                                            const double2 *ghi, uint32_t nhi)
{
    for (uint32_t i = threadIdx.x; i < 64 + nhi; i += blockDim.x) {
        if (i < 64) wlo[i] = glo[i];
        else whi[i - 64] = ghi[i - 64];
    }
}

// the same with cp.async: the table loads overlap whatever the CTA issues next (the key bits,
// its row or tile); cp_async_wait_all() + __syncthreads() before the first use
__device__ __forceinline__ void load_tables_async(double2 *wlo, double2 *whi, const double2 *glo,
                                                  const double2 *ghi, uint32_t nhi)
{
    for (uint32_t i = threadIdx.x; i < 64 + nhi; i += blockDim.x) {
        if (i < 64) cp_async16(wlo + i, glo + i);
        else cp_async16(whi + i - 64, ghi + i - 64);
    }
}

// bulk L2 prefetch of one N1-element row (warp 0 issues 32 pieces)
__device__ __forceinline__ void l2_prefetch_row(const double2 *row, uint32_t N1)
{
    const uint32_t q = threadIdx.x;
    if (q >= 32) return;
    const char *src = reinterpret_cast<const char *>(row);
    const uint32_t bytes = N1 * 16u, chunk = ((bytes + 31) / 32 + 15) & ~15u;
    if (q * chunk < bytes) {
        const uint32_t sz = bytes - q * chunk < chunk ? bytes - q * chunk : chunk;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + (size_t)q * chunk), "r"(sz) : "memory");
    }
}

// ------------------------------------------------------------------ tables
// K1's first DIF stage reads x, not z: with b = j + r Ls (Ls = N2 / R), theta_b = theta_j c_r,
// c_r = e^{i pi r / 2R}, so DFT_R(z)_k = theta_j (T[p_re][k] + i T[p_im][k]) where p_re / p_im
// hold the R real / imaginary key bits of the butterfly and T[p][k] = sum_{r in p} c_r w_R^{rk}
// = sum_{r in p} e^{i pi r (1 - 4k) / 2R} (each term an exactly-argued sincospi)
__global__ void k_bits_table(uint32_t R, double2 *tb)
{
    for (uint32_t e = threadIdx.x; e < (1u << R) * R; e += blockDim.x) {
        const uint32_t p = e / R, k = e % R;
        double re = 0.0, im = 0.0;
        for (uint32_t r = 0; r < R; ++r) {
            if (!((p >> r) & 1u)) continue;
            // angle r (1 - 4k) / 2R in half turns, reduced mod 2 exactly in integers
            const int64_t num = ((int64_t)r * (1 - 4 * (int64_t)k)) % (int64_t)(4 * R);
            double s, c;
            sincospi((double)num / (double)(2 * R), &s, &c);
            re += c;
            im += s;
        }
        tb[e] = make_double2(re, im);
    }
}

__global__ void k_tables(Geometry g, RouteTables T)
{
    uint64_t tot = std::max<uint64_t>(std::max<uint64_t>(g.N1, g.N2), 64);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < tot;
         e += (uint64_t)gridDim.x * blockDim.x) {
        double s, c;
        if (e < 64) {
            sincospi(2.0 * (double)e / (double)g.N1, &s, &c);
            T.W1lo[e] = make_double2(c, -s);
            sincospi(2.0 * (double)e / (double)g.N2, &s, &c);
            T.W2lo[e] = make_double2(c, -s);
        }
        if (e < g.f1.nhi) {
            sincospi(2.0 * (double)(e * 64) / (double)g.N1, &s, &c);
            T.W1hi[e] = make_double2(c, -s);
        }
        if (e < g.f2.nhi) {
            sincospi(2.0 * (double)(e * 64) / (double)g.N2, &s, &c);
            T.W2hi[e] = make_double2(c, -s);
        }
        if (e < 64) {  // theta_b = exp(i pi b / (2 N2)) = thhi[b >> 6] * thlo[b & 63]
            sincospi((double)e / (double)(2 * (uint64_t)g.N2), &s, &c);
            T.thlo[e] = make_double2(c, s);
        }
        if (e < g.f2.nhi) {
            sincospi((double)(64 * e) / (double)(2 * (uint64_t)g.N2), &s, &c);
            T.thhi[e] = make_double2(c, s);
        }
        if (e < g.N2) {
            // DIF output position e -> frequency index
            uint32_t rem = (uint32_t)e, L = g.N2, mult = 1, k = 0;
            for (int i = 0; i < g.f2.S; ++i) {
                uint32_t R = g.f2.st[i].R, Ls = L / R;
                k += (rem / Ls) * mult;
                rem %= Ls;
                mult *= R;
                L = Ls;
            }
            T.rev2[e] = k;
        }
    }
}

// Per-stage twiddle tables (create time; see stage_twiddle in fft_core.cuh): stage s of plan
// P holds omega_Lt^{jG} for j < min(64, Ls) at hi + toff and, when Ls > 64, omega_Lt^{64 j' G}
// for j' < Ls/64 at hi + toff + 64.  `hi` is the plan's global hi[] table.
__global__ void k_stage_tables(FftPlan P, double2 *hi)
{
    for (int s = 0; s < P.S; ++s) {
        const StageDesc &d = P.st[s];
        if (d.G == 1 || d.Ls <= 1) continue;
        const uint32_t nlo = d.Ls > 64 ? 64 : d.Ls, nh = d.Ls > 64 ? (d.Ls + 63) / 64 : 0;
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nlo + nh; i += gridDim.x * blockDim.x) {
            const uint64_t e = i < nlo ? (uint64_t)i * d.G : 64ull * (i - nlo) * d.G;
            double sn, cs;
            sincospi(2.0 * (double)e / (double)P.Lt, &sn, &cs);
            hi[d.toff + (i < nlo ? i : 64 + (i - nlo))] = make_double2(cs, -sn);
        }
    }
}

// Per-row twist tables for K2 (create time): row p holds rho^e, rho = e^{2 pi i (1-4k)/4M},
// k = rev2[p], as rlo[e & 63] * rhi[e >> 6] -- computing them in K2's prologue costs a
// chain of 64-bit remainders, an FP64 division and sincospi per thread on every hash.
__global__ void k_rho_tables(Geometry g, RouteTables T)
{
    const uint32_t w = 64 + g.f1.nhi;
    double2 *r = T.rho + (size_t)blockIdx.x * w;
    rho_tables(r, r + 64, g.f1.nhi, g.M, T.rev2[blockIdx.x]);
}

// ------------------------------------------------------------------ K0
// Bit transpose of the zero-padded input into one bit stream per K1 column
// group: group g (columns [gC, gC+C)) holds, for each row b < N2, the 2C bits
// x[N1 b + gC + c] (c < C) then x[M + N1 b + gC + c] -- entry b of the stream,
// EPW = 32 / 2C entries per uint32 word, g.kbw words per group.  A CTA transposes
// a tile of 64 rows x 1024 columns through shared memory, so both the key reads
// (128-byte row segments) and the stream writes are coalesced; K1 then loads its
// group's bits with a few contiguous words instead of N2 scattered gathers.
constexpr uint32_t kK0Rows = 64, kK0Cols = 1024;  // largest tile (shared arrays sized for it)

// tile rows x cols: 64 x 1024 for large transforms, 16 x 256 for small ones (more CTAs)
__host__ __device__ inline uint32_t k0_rows(const Geometry &g) { return g.k0rb; }
__host__ __device__ inline uint32_t k0_cols(const Geometry &g) { return g.k0cb; }

__global__ void __launch_bounds__(256)
k0_bits_transpose(const uint32_t *__restrict__ w, uint64_t off, uint64_t nbits, uint32_t *__restrict__ kb,
                  Geometry g, uint64_t key_stride)
{
    w += blockIdx.z * key_stride;                             // batch: key blockIdx.z
    kb += (uint64_t)blockIdx.z * (g.N1 / g.C) * g.kbw;
    TRACE_BEGIN(0);
    __shared__ uint32_t tre[kK0Rows][kK0Cols / 32 + 1], tim[kK0Rows][kK0Cols / 32 + 1];
    grid_dep_wait();    // launched with PDL itself: whatever wrote the key precedes us
    grid_dep_launch();  // K1 may start its prologue (K0 is a single short wave)
    const uint32_t C = g.C, twoC = 2 * C, epw = 32 / twoC;
    const uint32_t RB = k0_rows(g), CB = k0_cols(g), CW = CB / 32;
    const uint32_t c0 = blockIdx.x * CB, b0 = blockIdx.y * RB;
    const int64_t lo = (int64_t)off, hi = (int64_t)(off + nbits);
    for (uint32_t i = threadIdx.x; i < RB * CW; i += blockDim.x) {
        const uint32_t r = i / CW, k = i % CW;
        const uint32_t b = b0 + r, col = c0 + 32 * k;
        uint32_t re = 0, im = 0;
        if (b < g.N2 && col < g.N1) {
            const int64_t P = (int64_t)g.N1 * b + col;
            re = bits32(w, P + lo, lo, hi);
            im = bits32(w, P + (int64_t)g.M + lo, lo, hi);
            const uint32_t valid = g.N1 - col;  // columns past N1 belong to the next row
            if (valid < 32) {
                re &= (1u << valid) - 1u;
                im &= (1u << valid) - 1u;
            }
        }
        tre[r][k] = re;
        tim[r][k] = im;
    }
    __syncthreads();
    const uint32_t groups = CB / C;                 // groups in this column tile
    const uint32_t wpg = RB / epw;                  // stream words per group in this row tile
    const uint32_t cmask = (C == 32) ? 0xFFFFFFFFu : ((1u << C) - 1u);
    for (uint32_t i = threadIdx.x; i < groups * wpg; i += blockDim.x) {
        const uint32_t gl = i / wpg, k = i % wpg;
        const uint32_t gg = c0 / C + gl;
        const uint32_t wb = b0 / epw + k;           // word index in the group's stream
        if (gg >= g.N1 / C || wb * epw >= g.N2) continue;
        const uint32_t cb = gl * C;                 // bit column within the tile
        uint32_t word = 0;
        for (uint32_t e = 0; e < epw; ++e) {
            const uint32_t r = k * epw + e;
            const uint32_t re = (tre[r][cb >> 5] >> (cb & 31)) & cmask;
            const uint32_t im = (tim[r][cb >> 5] >> (cb & 31)) & cmask;
            word |= (re | (im << C)) << (e * twoC);
        }
        kb[(uint64_t)gg * g.kbw + wb] = word;
    }
    TRACE_END(0);
}

// ------------------------------------------------------------------ K1
// Column DIF of C adjacent columns; input = this group's bit stream from K0.
// Column-pass stage dispatch for plans [A, B, (C), 16, ...] known at compile time (A = 0: the
// general radix switch).  Instantiating only the radices a plan uses keeps K1/K3's code small,
// which measurably matters (k2_rows_t).
// K1/K3 keep their stages as calls: inlining them (K13_STAGE=stage_inl) helped the
// throughput configs a little (C5d 1026 -> 1014 us) but cost the cold small ones more
// (C2 37.9 -> 40 us, C3 188 -> 194 us: more code to fetch cold); K2 inlines (below)
#ifndef K13_STAGE
#define K13_STAGE stage_smem
#endif
template <bool INV, int MODE, int A, int B, int C>
__device__ __forceinline__ void stage_t(double2 *sm, const FftPlan &P, int i, uint32_t logC, const double2 *wlo,
                                        const double2 *whi, const StageCtx &x = StageCtx{})
{
    if (A == 0) stage_any<INV, MODE>(sm, P.st[i], logC, wlo, whi, x);
    else if (i == 0) K13_STAGE<A ? A : 16, INV, MODE>(sm, P.st[0], logC, wlo, whi, x);
    else if (i == 1) K13_STAGE<B ? B : 16, INV, MODE>(sm, P.st[1], logC, wlo, whi, x);
    else if (i == 2 && C) K13_STAGE<C ? C : 16, INV, MODE>(sm, P.st[2], logC, wlo, whi, x);
    else K13_STAGE<16, INV, MODE>(sm, P.st[i], logC, wlo, whi, x);
}
template <int A, int B, int C>
__device__ __forceinline__ void dif_t(double2 *sm, const FftPlan &P, int i0, int i1, uint32_t logC,
                                      const double2 *wlo, const double2 *whi)
{
    for (int i = i0; i < i1; ++i) {
        stage_t<false, MODE_PLAIN, A, B, C>(sm, P, i, logC, wlo, whi);
        __syncthreads();
    }
}
template <int A, int B, int C>
__device__ __forceinline__ void dit_t(double2 *sm, const FftPlan &P, int i0, int i1, uint32_t logC,
                                      const double2 *wlo, const double2 *whi)
{
    for (int i = i1 - 1; i >= i0; --i) {
        stage_t<true, MODE_PLAIN, A, B, C>(sm, P, i, logC, wlo, whi);
        __syncthreads();
    }
}

// K1's stage 0 (radix R, span N2, G = 1) straight from the key bits (k_bits_table): per
// butterfly (column c, j < Ls) the R real and R imaginary bits of rows j + r Ls index the table,
// v_k = theta_j (T[p_re][k] + i T[p_im][k]) * w_N2^{jk}, written where stage 0 writes.  Replaces
// the z generation pass and stage 0's DFT.
struct NoHook {
    __device__ __forceinline__ void operator()() const {}
};
// Hook: called once per butterfly iteration (K1P drains a piece of the previous tile there)
template <int R, typename Hook = NoHook>
__device__ __forceinline__ void k1_first_stage_bits(double2 *sm, const StageDesc &sd, uint32_t logC,
                                                    const uint32_t *rowbits, const double2 *tb,
                                                    const double2 *thlo, const double2 *thhi,
                                                    const double2 *wlo, const double2 *whi, Hook hook = Hook{})
{
    const uint32_t C = 1u << logC, twoC = 2 * C, epw = 32 / twoC;
    const uint32_t nb = sd.nb << logC, cm = C - 1, stride = sd.Ls << logC;
    for (uint32_t q = threadIdx.x; q < nb; q += blockDim.x) {
        const uint32_t c = q & cm, j = q >> logC;
        uint32_t pr = 0, pi = 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const uint32_t b = j + r * sd.Ls;
            const uint32_t rb = rowbits[b / epw] >> ((b % epw) * twoC);
            pr |= ((rb >> c) & 1u) << r;
            pi |= ((rb >> (C + c)) & 1u) << r;
        }
        const double2 th = twiddle(thlo, thhi, j);
        double2 v[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            const double2 a = tb[pr * R + k], bi = tb[pi * R + k];
            v[k] = cmul(make_double2(a.x - bi.y, a.y + bi.x), th);
        }
        if (j) apply_twiddles<R, false>(v, stage_twiddle(sd, j, wlo, whi));
        const uint32_t base = (j << logC) + c;
#pragma unroll
        for (int r = 0; r < R; ++r) sm[pidx(base + r * stride)] = v[r];
        hook();
    }
}

template <int RA, int RB, int RC>
__global__ void __launch_bounds__(PA_TMAX, PA_MINB)
k1_fwd_columns(const uint32_t *__restrict__ kb, double2 *__restrict__ buf, Geometry g, RouteTables T,
               uint32_t *__restrict__ zero_out, uint64_t zero_words, uint64_t out_stride,
               const uint32_t *__restrict__ xkey, uint64_t xstride, uint64_t xbits)
{
    kb += (uint64_t)blockIdx.y * (g.N1 / g.C) * g.kbw;        // batch: key blockIdx.y
    buf += (uint64_t)blockIdx.y * g.M;
    if (zero_out) zero_out += blockIdx.y * out_stride;
    extern __shared__ double2 sm[];
    const uint32_t logC = g.logC, C = 1u << logC;
    double2 *wlo = sm + g.tile1, *whi = wlo + 64, *thlo = whi + g.f2.nhi + g.f2.ntw, *thhi = thlo + 64;
    uint32_t *rowbits = reinterpret_cast<uint32_t *>(thhi + g.f2.nhi);
    double2 *tb = reinterpret_cast<double2 *>(rowbits + g.kbw);  // g.ntb entries (first stage from bits)
    // first stage from the key bits for R0 <= 4 only: same-box, R0 = 3 gains (C4 K1 781 -> 738 us,
    // C5a 37.8 -> 35.8 us) but R0 = 5 / 7 lose (C2 37.9 -> 39.9 us, C3 188 -> 199 us: 2.5 / 14 KB
    // tables, bank-conflicted lookups, more code)
    constexpr bool kBits = RA >= 2 && RA <= 4;
    const uint32_t a0 = blockIdx.x * C;
    const uint32_t tot = g.N2 << logC;
    TRACE_BEGIN(1);
    TSTAMPK(0, 0);
    load_tables_async(wlo, whi, T.W2lo, T.W2hi, g.f2.nhi + g.f2.ntw);
    load_tables_async(thlo, thhi, T.thlo, T.thhi, g.f2.nhi);
    if (kBits)
        for (uint32_t i = threadIdx.x; i < g.ntb; i += blockDim.x) cp_async16(tb + i, T.tb + i);
    grid_dep_wait();  // K0's bit streams
    if (zero_out) {  // K3 XORs this hash's output bits in (zero_words = 0: accumulate)
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < zero_words;
             i += (uint64_t)gridDim.x * blockDim.x)
            zero_out[i] = 0u;
    }
    if (xkey) {
        // wide column groups (C >= 8: runs of >= 1 byte per row) gather their bit stream
        // from the key directly instead of through K0 -- the same entries K0 would write:
        // row b holds x[a0 + N1 b + c] (c < C) then x[M + a0 + N1 b + c], zero past n
        const uint32_t *kx = xkey + blockIdx.y * xstride;
        const uint32_t twoC = 2 * C, epw = 32 / twoC, mask = (1u << C) - 1u;
        for (uint32_t i = threadIdx.x; i < g.kbw; i += blockDim.x) rowbits[i] = 0u;
        __syncthreads();
        for (uint32_t b = threadIdx.x; b < g.N2; b += blockDim.x) {
            const int64_t u = (int64_t)a0 + (int64_t)g.N1 * b;
            const uint32_t re = bits32(kx, u, 0, (int64_t)xbits) & mask;
            const uint32_t im = bits32(kx, u + (int64_t)g.M, 0, (int64_t)xbits) & mask;
            const uint32_t ent = re | (im << C);
            if (epw == 1) rowbits[b] = ent;
            else if (ent) atomicOr(rowbits + b / epw, ent << ((b % epw) * twoC));
        }
    } else {
        const uint32_t *src = kb + (uint64_t)blockIdx.x * g.kbw;
        for (uint32_t i = threadIdx.x; i < g.kbw; i += blockDim.x) rowbits[i] = __ldg(src + i);
    }
    cp_async_wait_all();  // the tables
    TSTAMPK(0, 1);
    __syncthreads();
    TSTAMPK(0, 2);
    // z(b, c) = (x[a + N1 b] + i x[a + N1 b + M]) * theta_b; entry b of the stream holds
    // the C real-part bits then the C imaginary-part bits of row b
    int s0 = 0;  // first stage still to run
    if (kBits && g.ntb) {
        k1_first_stage_bits<kBits ? RA : 2>(sm, g.f2.st[0], logC, rowbits, tb, thlo, thhi, wlo, whi);
        s0 = 1;
    } else {
        const uint32_t twoC = 2 * C, epw = 32 / twoC;
        for (uint32_t e = threadIdx.x; e < tot; e += blockDim.x) {
            const uint32_t b = e >> logC, c = e & (C - 1);
            const uint32_t rb = rowbits[b / epw] >> ((b % epw) * twoC);
            const double xr = (double)((rb >> c) & 1u), xi = (double)((rb >> (C + c)) & 1u);
            const double2 th = twiddle(thlo, thhi, b);
            sm[pidx(e)] = make_double2(xr * th.x - xi * th.y, xr * th.y + xi * th.x);
        }
    }
    __syncthreads();
    TSTAMPK(0, 3);
    // row p of the work array = DIF output position p (k_b = rev2[p]).  The last forward
    // stage writes it straight to global when C >= g.k1gout (2: 32-byte row pieces)
    const bool direct = g.f2.S > 1 && C >= g.k1gout;
    if (direct) {
        dif_t<RA, RB, RC>(sm, g.f2, s0, g.f2.S - 1, logC, wlo, whi);
        grid_dep_launch();  // K2 may start its prologue
        StageCtx gx;
        gx.gout = buf + a0;
        gx.ld = g.N1;
        stage_t<false, MODE_GCOL_OUT, RA, RB, RC>(sm, g.f2, g.f2.S - 1, logC, wlo, whi, gx);
        TSTAMPK(0, 4);
    } else {
        dif_t<RA, RB, RC>(sm, g.f2, s0, g.f2.S, logC, wlo, whi);
        grid_dep_launch();  // K2 may start its prologue
        TSTAMPK(0, 4);
        for (uint32_t e = threadIdx.x; e < tot; e += blockDim.x)
            buf[(uint64_t)(e >> logC) * g.N1 + a0 + (e & (C - 1))] = sm[pidx(e)];
    }
    TSTAMPK(0, 5);
    TRACE_END(1);
}

// ------------------------------------------------------------------ TMEM helpers
__device__ __forceinline__ void tm_st32(uint32_t taddr, const uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
        "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
        "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
        "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]));
}
__device__ __forceinline__ void tm_ld32(uint32_t taddr, uint32_t (&r)[32])
{
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}
__device__ __forceinline__ void cta_sync_tmem()  // barrier ordering tcgen05 traffic across warps
{
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ------------------------------------------------------------------ K1P (TMEM write-behind K1)
// K1 for one-CTA-per-SM tiles of a multi-wave grid (C4, C5c/d): every non-persistent K1 CTA
// ends with a burst of N2 x C scattered 32-byte row-piece stores (the last DIF stage writing
// HBM; ~14 k of ~43 k cycles per tile at C4) that nothing overlaps, because shared memory
// holds one tile.  Tensor memory (256 KB per SM, idle in this pass) holds the finished tile
// instead: K1P is persistent (one CTA per SM, tables loaded once, the next tile's key bits
// prefetched with cp.async), its last DIF stage writes each butterfly's 16 outputs to the
// thread's own TMEM lane (tcgen05.st), and during the NEXT tile's stages every thread drains
// its own columns back out (tcgen05.ld -> 16-byte stores), so the stores stream under the
// FP64 stages.  A thread reads only what it wrote (its lane, its columns): no cross-thread
// TMEM hazard, only tcgen05.wait::st/ld ordering within the thread.
// TMEM layout: warp w owns lane quarter w & 3; thread (w, l) -> lane 32 (w & 3) + l, butterfly
// k of the thread (q = tid + k * 512) -> columns [64 ((w >> 2) kmax + k), + 64): complex r at
// words 4r..4r+3 (re lo, re hi, im lo, im hi).
__device__ __forceinline__ uint32_t k1p_col(uint32_t k, uint32_t kmax)
{
    return (((threadIdx.x >> 5) >> 2) * kmax + k) * 64u;
}

// last DIF stage (radix 16, Ls = 1: no twiddles) of the tile in shared memory -> TMEM
__device__ __forceinline__ void k1p_last_stage(const double2 *sm, const StageDesc &sd, uint32_t logC, uint32_t tm,
                                               uint32_t kmax)
{
    const uint32_t nb = sd.nb << logC, cm = (1u << logC) - 1;
    const uint32_t lane_base = tm + ((32u * ((threadIdx.x >> 5) & 3)) << 16);
    uint32_t k = 0;
    for (uint32_t qb = threadIdx.x & ~31u; qb < nb; qb += blockDim.x, ++k) {  // warp-uniform trip count
        const uint32_t q = qb + (threadIdx.x & 31);
        double2 v[16];
        if (q < nb) {
            const uint32_t c = q & cm, g = q >> logC;
            const uint32_t base = ((g * 16u) << logC) + c;
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = sm[pidx(base + (r << logC))];
            Dft<16, false>::run(v);
        } else {
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            uint32_t w[32];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double2 d = v[8 * h + i];
                w[4 * i] = __double2loint(d.x);
                w[4 * i + 1] = __double2hiint(d.x);
                w[4 * i + 2] = __double2loint(d.y);
                w[4 * i + 3] = __double2hiint(d.y);
            }
            tm_st32(lane_base + k1p_col(k, kmax) + 32u * h, w);
        }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// drain pieces [p0, p1) of the previous tile: piece = 2 outputs of one butterfly (k = pc / 8,
// outputs 2 (pc % 8) and 2 (pc % 8) + 1) -- small pieces spread over the next tile's first
// stage keep the store queue from filling (lg_throttle) as whole 8-output chunks did
__device__ __forceinline__ void tm_ld16(uint32_t taddr, uint32_t (&r)[16])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
                 "%14, %15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(taddr));
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, uint32_t (&r)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}
template <int PW>  // outputs per piece: 2, 4 or 8
__device__ __forceinline__ void k1p_drain_pieces_t(double2 *__restrict__ dst, uint32_t N1, uint32_t nb, uint32_t logC,
                                                   uint32_t tm, uint32_t kmax, uint32_t p0, uint32_t p1)
{
    constexpr uint32_t PPB = 16 / PW;  // pieces per butterfly
    const uint32_t cm = (1u << logC) - 1;
    const uint32_t lane_base = tm + ((32u * ((threadIdx.x >> 5) & 3)) << 16);
    for (uint32_t pc = p0; pc < p1; ++pc) {
        const uint32_t k = pc / PPB, pr = pc % PPB;
        const uint32_t qb = (threadIdx.x & ~31u) + k * blockDim.x;
        if (k >= kmax || qb >= nb) break;  // warp-uniform
        uint32_t w[4 * PW];
        const uint32_t ta = lane_base + k1p_col(k, kmax) + 4u * PW * pr;
        if constexpr (PW == 2) {
            uint32_t (&v)[8] = reinterpret_cast<uint32_t (&)[8]>(w);
            tm_ld8(ta, v);
        } else if constexpr (PW == 4) {
            uint32_t (&v)[16] = reinterpret_cast<uint32_t (&)[16]>(w);
            tm_ld16(ta, v);
        } else {
            uint32_t (&v)[32] = reinterpret_cast<uint32_t (&)[32]>(w);
            tm_ld32(ta, v);
        }
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const uint32_t q = qb + (threadIdx.x & 31);
        if (q < nb) {
            const uint32_t c = q & cm, g = q >> logC;
            double2 *p = dst + (uint64_t)(16u * g + PW * pr) * N1 + c;
#pragma unroll
            for (int i = 0; i < PW; ++i)
                p[(uint64_t)i * N1] = make_double2(__hiloint2double(w[4 * i + 1], w[4 * i]),
                                                   __hiloint2double(w[4 * i + 3], w[4 * i + 2]));
        }
    }
}
__device__ __forceinline__ void k1p_drain_pieces(double2 *__restrict__ dst, uint32_t N1, uint32_t nb, uint32_t logC,
                                                 uint32_t tm, uint32_t kmax, uint32_t p0, uint32_t p1, uint32_t pw)
{
    if (pw == 2) k1p_drain_pieces_t<2>(dst, N1, nb, logC, tm, kmax, p0, p1);
    else if (pw == 4) k1p_drain_pieces_t<4>(dst, N1, nb, logC, tm, kmax, p0, p1);
    else k1p_drain_pieces_t<8>(dst, N1, nb, logC, tm, kmax, p0, p1);
}

template <int RA, int RB, int RC>
__global__ void __launch_bounds__(PA_TMAX, 1)
k1p_fwd_columns(const uint32_t *__restrict__ kb, double2 *__restrict__ buf, Geometry g, RouteTables T,
                uint32_t *__restrict__ zero_out, uint64_t zero_words, uint64_t out_stride, uint32_t count)
{
    const uint32_t tcols = g.k1p_tcols;  // 512 (one CTA per SM) or 256 (two)
    extern __shared__ double2 sm[];
    __shared__ uint32_t tm_base;
    const uint32_t logC = g.logC, C = 1u << logC;
    double2 *wlo = sm + g.tile1, *whi = wlo + 64, *thlo = whi + g.f2.nhi + g.f2.ntw, *thhi = thlo + 64;
    uint32_t *rowbits0 = reinterpret_cast<uint32_t *>(thhi + g.f2.nhi);
    double2 *tb = reinterpret_cast<double2 *>(rowbits0 + g.kbw);
    uint32_t *rowbits1 = reinterpret_cast<uint32_t *>(tb + g.ntb);
    constexpr bool kBits = RA >= 2 && RA <= 4;
    const uint32_t ngroups = g.N1 / C, ntiles = ngroups * count;
    const int S = g.f2.S;
    const StageDesc &last = g.f2.st[S - 1];
    const uint32_t nb_last = last.nb << logC, kmax = g.k1p_kmax;
    load_tables_async(wlo, whi, T.W2lo, T.W2hi, g.f2.nhi + g.f2.ntw);
    load_tables_async(thlo, thhi, T.thlo, T.thhi, g.f2.nhi);
    if (kBits)
        for (uint32_t i = threadIdx.x; i < g.ntb; i += blockDim.x) cp_async16(tb + i, T.tb + i);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tm_base)), "r"(tcols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    grid_dep_wait();  // K0's bit streams
    if (zero_out) {   // K3 XORs this hash's output bits in
        for (uint32_t key = 0; key < count; ++key)
            for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < zero_words;
                 i += (uint64_t)gridDim.x * blockDim.x)
                zero_out[key * out_stride + i] = 0u;
    }
    auto fetch_bits = [&](uint32_t t, uint32_t *dst) {
        const uint32_t *src = kb + (uint64_t)t * g.kbw;  // tile t = key * ngroups + group
        for (uint32_t i = 4 * threadIdx.x; i < g.kbw; i += 4 * blockDim.x) cp_async16(dst + i, src + i);
    };
    if (blockIdx.x < ntiles) fetch_bits(blockIdx.x, rowbits0);
    cta_sync_tmem();
    const uint32_t tm = tm_base;
    double2 *prev = nullptr;  // previous tile's column group (key's work array + a0), drained below
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const uint32_t key = t / ngroups, a0 = (t % ngroups) * C;
        uint32_t *rowbits = (it & 1) ? rowbits1 : rowbits0;
        cp_async_wait_all();
        __syncthreads();  // this tile's bits (and the tables) landed; the last tile's smem reads done
        if (t + gridDim.x < ntiles) fetch_bits(t + gridDim.x, (it & 1) ? rowbits0 : rowbits1);
        // spread the previous tile's drain (npieces pieces of 2 outputs per thread) over this tile:
        // one piece per first-stage butterfly iteration, the rest before the later stage passes
        uint32_t pc = 0;
        const uint32_t pw = g.k1p_piece, npieces = (16 / pw) * kmax;
        auto drain_upto = [&](uint32_t upto) {
            if (!prev || upto <= pc) return;
            k1p_drain_pieces(prev, g.N1, nb_last, logC, tm, kmax, pc, upto, pw);
            pc = upto;
        };
        auto drain_step = [&](int i) {  // before stage i (1 <= i <= S - 1): an even share of what is left
            const uint32_t left = npieces - pc, passes = (uint32_t)(S - i);
            drain_upto(pc + (left + passes - 1) / passes);
        };
        int s0 = 0;
        const uint32_t nb0 = g.f2.st[0].nb << logC;
        if (kBits && g.ntb) {
            if (prev && nb0 % 32 == 0) {  // warp-uniform trip counts: the warp-collective TMEM loads may sit in the loop
                auto hook = [&]() { drain_upto(pc + 1 < npieces ? pc + 1 : npieces); };
                k1_first_stage_bits<kBits ? RA : 2>(sm, g.f2.st[0], logC, rowbits, tb, thlo, thhi, wlo, whi, hook);
            } else {
                k1_first_stage_bits<kBits ? RA : 2>(sm, g.f2.st[0], logC, rowbits, tb, thlo, thhi, wlo, whi);
            }
            s0 = 1;
        } else {
            const uint32_t twoC = 2 * C, epw = 32 / twoC, tot = g.N2 << logC;
            for (uint32_t e = threadIdx.x; e < tot; e += blockDim.x) {
                const uint32_t b = e >> logC, c = e & (C - 1);
                const uint32_t rb = rowbits[b / epw] >> ((b % epw) * twoC);
                const double xr = (double)((rb >> c) & 1u), xi = (double)((rb >> (C + c)) & 1u);
                const double2 th = twiddle(thlo, thhi, b);
                sm[pidx(e)] = make_double2(xr * th.x - xi * th.y, xr * th.y + xi * th.x);
            }
        }
        __syncthreads();
        for (int i = s0; i < S - 1; ++i) {
            if (i > 0) drain_step(i);
            stage_t<false, MODE_PLAIN, RA, RB, RC>(sm, g.f2, i, logC, wlo, whi);
            __syncthreads();
        }
        drain_upto(npieces);  // everything of the previous tile is out of TMEM now
        k1p_last_stage(sm, last, logC, tm, kmax);
        prev = buf + (uint64_t)key * g.M + a0;
    }
    grid_dep_launch();  // K2 may start its prologue
    if (prev) k1p_drain_pieces(prev, g.N1, nb_last, logC, tm, kmax, 0, (16 / g.k1p_piece) * kmax, g.k1p_piece);
    cta_sync_tmem();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(tcols) : "memory");
}

// ------------------------------------------------------------------ K2
// Fused last DIF stage (Ls = 1, no twiddles) * spectrum * first DIT stage.  The
// spectrum row is stored [r][g] (element g*R + r at sp[r * nb + g]) so that the
// lanes of a warp (consecutive g) read it coalesced.
template <int R>
__device__ __noinline__ void fused_mid(StageDesc sd, double2 *sm, const double2 *__restrict__ sp)
{
    for (uint32_t gq = threadIdx.x; gq < sd.nb; gq += blockDim.x) {
        const uint32_t base = gq * R;
        double2 s[R], v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) s[r] = __ldg(sp + r * sd.nb + gq);
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = sm[pidx(base + r)];
        Dft<R, false>::run(v);
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = cmul(v[r], s[r]);
        Dft<R, true>::run(v);
#pragma unroll
        for (int r = 0; r < R; ++r) sm[pidx(base + r)] = v[r];
    }
}

__device__ __forceinline__ void fused_mid_any(const StageDesc &sd, double2 *sm, const double2 *sp)
{
    switch (sd.R) {
    case 2: fused_mid<2>(sd, sm, sp); break;
    case 3: fused_mid<3>(sd, sm, sp); break;
    case 4: fused_mid<4>(sd, sm, sp); break;
    case 5: fused_mid<5>(sd, sm, sp); break;
    case 7: fused_mid<7>(sd, sm, sp); break;
    case 8: fused_mid<8>(sd, sm, sp); break;
    default: fused_mid<16>(sd, sm, sp); break;
    }
}

// mode 0 (hash): in place, buf row -> tau -> DIF, * spec, DIT -> conj tau -> buf row.
// mode 1 (create): buf row -> tau -> DIF -> * scale -> spec row.
__global__ void __launch_bounds__(PA_TMAX, PA_MINB)
k2_rows(double2 *buf, double2 *out2, double2 *__restrict__ spec, Geometry g, RouteTables T, int mode,
        double scale, uint64_t spec_stride)
{
    // buf and out2 may be the same array (K2 in place when lr = 0): no __restrict__ on them
    extern __shared__ double2 sm[];
    const uint32_t N1 = g.N1;
    double2 *wlo = sm + g.tile2, *whi = wlo + 64, *rlo = whi + g.f1.nhi + g.f1.ntw, *rhi = rlo + 64;
    // grid (keys, rows): the CTAs of one spectrum row run back to back, so the row is
    // read from HBM once per batch and served from L2 to the other keys
    const uint32_t row = blockIdx.y;
    buf += (uint64_t)blockIdx.x * g.M;
    out2 += (uint64_t)blockIdx.x * g.M;
    TRACE_BEGIN(2);
    TSTAMP(0);
    double2 *rp = buf + (uint64_t)row * N1;  // input row (row-major)
    double2 *rq = out2 + wrow(g, row);        // output row: element a at rq[wcol(g, a)]
    double2 *sp = spec + blockIdx.x * spec_stride + (uint64_t)row * N1;  // per-key spectra: fresh seeds
    load_tables_async(wlo, whi, T.W1lo, T.W1hi, g.f1.nhi + g.f1.ntw);
    {
        const double2 *rt0 = T.rho + (size_t)row * (64 + g.f1.nhi);
        load_tables_async(rlo, rhi, rt0, rt0 + 64, g.f1.nhi);
    }
    if (g.pfs && mode == 0 && (blockIdx.x == 0 || spec_stride)) l2_prefetch_row(sp, N1);  // see k2_rows_t
    grid_dep_wait();  // K1's work array
    const FftPlan &P0 = g.f1;
    if (P0.S <= 1) {  // tiny rows: stage through shared memory
        for (uint32_t e = threadIdx.x; e < N1; e += blockDim.x) cp_async16(sm + pidx(e), rp + e);
    }
    cp_async_wait_all();  // tables (and the staged row)
    __syncthreads();
    TSTAMP(1);
    const FftPlan &P = g.f1;
    StageCtx rt;
    rt.rlo = rlo;
    rt.rhi = rhi;
    rt.gout = rq;
    if (P.S <= 1) {  // N1 <= 16: tau elementwise, then the single stage below runs plain
        for (uint32_t e = threadIdx.x; e < N1; e += blockDim.x) sm[pidx(e)] = cmul(sm[pidx(e)], twiddle(rlo, rhi, e));
        __syncthreads();
    } else {
        rt.gin = rp;  // the first stage reads the row straight from global memory
        stage_any<false, MODE_TAU_IN>(sm, P.st[0], 0, wlo, whi, rt);
        rt.gin = nullptr;
        __syncthreads();
    }
    const int dif_from = P.S <= 1 ? 0 : 1;
    if (mode == 1) {
        dif_stages(sm, P, dif_from, P.S, 0, wlo, whi);
        // spectrum row in the [r][g] order fused_mid reads (R = last stage's radix): consecutive
        // threads write consecutive spectrum entries (element g R + r at sp[r nbl + g])
        grid_dep_launch();
        const uint32_t R = P.S ? P.st[P.S - 1].R : 1, nbl = N1 / R;
        for (uint32_t f = threadIdx.x; f < N1; f += blockDim.x) {
            const uint32_t r = f / nbl, gq = f - r * nbl;
            sp[f] = cscale(sm[pidx(gq * R + r)], scale);
        }
        return;
    }
    if (P.S == 0) {
        if (threadIdx.x == 0) rq[0] = cmul(sm[0], sp[0]);
        return;
    }
    TSTAMP(2);
    if (g.pf2 && mode == 0 && blockIdx.x == 0 && row + g.pf2 < g.N2 && threadIdx.x < 32) {
        // a CTA pf2 rows later will load row + pf2: start pulling it into L2 now, under this
        // row's compute (multi-wave grids only, see ra_plan; C4 K2 1219 -> 1129 us.  Prefetching
        // the next spectrum row as well, or K3's next column group, measured slower)
        const uint32_t q = threadIdx.x;
        const char *src = reinterpret_cast<const char *>(rp + (size_t)g.pf2 * N1);
        const uint32_t bytes = N1 * 16u, chunk = ((bytes + 31) / 32 + 15) & ~15u;
        if (q * chunk < bytes) {
            const uint32_t sz = bytes - q * chunk < chunk ? bytes - q * chunk : chunk;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + (size_t)q * chunk), "r"(sz) : "memory");
        }
    }
    dif_stages(sm, P, dif_from, P.S - 1, 0, wlo, whi);
    TSTAMP(3);
    fused_mid_any(P.st[P.S - 1], sm, sp);
    TSTAMP(4);
    __syncthreads();
    if (P.S == 1) {
        for (uint32_t e = threadIdx.x; e < N1; e += blockDim.x)
            rq[wcol(g, e)] = cmulc(sm[pidx(e)], twiddle(rlo, rhi, e));
        return;
    }
    dit_stages(sm, P, 1, P.S - 1, 0, wlo, whi);
    grid_dep_launch();  // K3 may start its prologue
    TSTAMP(5);
    rt.lr = g.lr;  // the output row in buf2's layout
    rt.lc = g.logC;
    stage_any<true, MODE_TAU_OUT>(sm, P.st[0], 0, wlo, whi, rt);
    TSTAMP(6);
    TRACE_END(2);
}

// ------------------------------------------------------------------ K2 for fixed radix shapes
// TMEM columns of a fresh-seed K2 CTA (k2_rows_t<..., kFresh>): 256 when two CTAs share the SM
// (<= 256 threads and two tiles of shared memory), else 512
__host__ __device__ inline uint32_t k2f_tcols(const Geometry &g, uint32_t nth)
{
    return nth <= PA_TMAX / 2 && 2 * (g.smem2 + 16) <= kSmemLimit ? 256u : 512u;
}
// a fresh-seed K2 fits when every thread's last-stage butterflies (64 columns each) fit its
// lane quarter's share of the columns
inline bool k2f_fits(const Geometry &g, uint32_t nth)
{
    if (!g.k2shape || g.smem2 + 16 > kSmemLimit) return false;
    const uint32_t nb = g.f1.st[g.f1.S - 1].nb, kmax = (nb + nth - 1) / nth;
    return (nth / 128) * kmax * 64 <= k2f_tcols(g, nth);
}
// The hash path of k2_rows for row plans [R0, R1, 16, ..., 16] (S >= 3): 4096 = [16, 16, 16]
// (C2, C3, C5), 10240 = [5, 8, 16, 16] (C4, C5d), 6144 = [3, 8, 16, 16], 7168 = [7, 4, 16, 16],
// calling those stage routines directly: the general kernel's radix switch instantiates every
// radix and mode, and K2's speed is sensitive to its code.
// K2's shape-specialised kernel inlines its stages (same-box A/B: C4 K2 1114 -> 1019 us,
// C3 192.5 -> 188.5 us, C2 unchanged)
#ifndef K2T_STAGE
#define K2T_STAGE stage_inl
#endif
#ifndef PA_K2MAX
#define PA_K2MAX PA_TMAX  // developer experiments: K2's launch bound (PA_FORCE_T2 up to it)
#endif
// KM = kSeed: the create-time / fresh-seed forward half instead (k2_rows mode 1): the last DIF
// stage (radix 16, span 16, no twiddles) runs from shared memory straight into the spectrum row,
// scaled by 1/M, in the [r][g] order fused_mid reads -- coalesced across lanes, no write-back.
// KM = kFresh: a fresh seed per key fused into the hash (pa_hash_fresh_batch): `spec` is the
// seeds' K1 output, not spectra.  The CTA first runs the seed row's forward half and keeps the
// scaled spectrum row in tensor memory (each thread its own last-stage butterflies, in its TMEM
// lane: the layout K1P uses), then the key row's forward half, whose fused middle stage
// multiplies by the spectrum read back from TMEM -- the spectrum never goes through HBM.
enum { kHash = 0, kSeed = 1, kFresh = 2 };
template <int R0, int R1, int NS, int KM = kHash>
__global__ void __launch_bounds__(PA_K2MAX, PA_MINB)
k2_rows_t(double2 *buf, double2 *out2, double2 *__restrict__ spec, Geometry g, RouteTables T,
          uint64_t spec_stride)
{
    extern __shared__ double2 sm[];
    const uint32_t N1 = g.N1;
    double2 *wlo = sm + g.tile2, *whi = wlo + 64, *rlo = whi + g.f1.nhi + g.f1.ntw, *rhi = rlo + 64;
    const uint32_t row = blockIdx.y;
    buf += (uint64_t)blockIdx.x * g.M;
    out2 += (uint64_t)blockIdx.x * g.M;
    TRACE_BEGIN(2);
    TSTAMP(0);
    double2 *rp = buf + (uint64_t)row * N1;
    double2 *rq = out2 + wrow(g, row);
    double2 *sp = spec + blockIdx.x * spec_stride + (uint64_t)row * N1;
    load_tables_async(wlo, whi, T.W1lo, T.W1hi, g.f1.nhi + g.f1.ntw);
    {
        const double2 *rt0 = T.rho + (size_t)row * (64 + g.f1.nhi);
        load_tables_async(rlo, rhi, rt0, rt0 + 64, g.f1.nhi);
    }
    // this row's spectrum, pulled into L2 under the forward stages -- by the first key's CTA only
    // (unless each key has its own spectrum): a batch's CTAs of one row run back to back and share
    // it (C5d x 16: 881.8 -> 867.8 us per key with no prefetch at all, whereas a single C4 key
    // needs it: 2179 -> 2219 us without)
    if (KM == kHash && g.pfs && (blockIdx.x == 0 || spec_stride)) l2_prefetch_row(sp, N1);
    // kFresh: TMEM for the spectrum row (256 columns when two CTAs share the SM, else 512)
    uint32_t *tmb = reinterpret_cast<uint32_t *>(rhi + g.f1.nhi);
    const uint32_t tcols = k2f_tcols(g, blockDim.x);
    if (KM == kFresh && threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(tmb)), "r"(tcols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    grid_dep_wait();  // K1's work array
    cp_async_wait_all();  // the tables
    if (KM == kFresh) cta_sync_tmem();
    else __syncthreads();
    TSTAMP(1);
    const FftPlan &P = g.f1;
    StageCtx rt;
    rt.rlo = rlo;
    rt.rhi = rhi;
    // stages 0 .. NS-2 of the forward half on the row at `src` (global), into shared memory
    auto forward = [&](const double2 *src, bool prefetch) {
        rt.gin = src;
        K2T_STAGE<R0, false, MODE_TAU_IN>(sm, P.st[0], 0, wlo, whi, rt);
        __syncthreads();
        if (prefetch && g.pf2 && blockIdx.x == 0 && row + g.pf2 < g.N2 && threadIdx.x < 32) {
            const uint32_t q = threadIdx.x;
            const char *pre = reinterpret_cast<const char *>(src + (size_t)g.pf2 * N1);
            const uint32_t bytes = N1 * 16u, chunk = ((bytes + 31) / 32 + 15) & ~15u;
            if (q * chunk < bytes) {
                const uint32_t sz = bytes - q * chunk < chunk ? bytes - q * chunk : chunk;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pre + (size_t)q * chunk), "r"(sz)
                             : "memory");
            }
        }
        K2T_STAGE<R1, false, MODE_PLAIN>(sm, P.st[1], 0, wlo, whi, StageCtx{});
        __syncthreads();
#pragma unroll
        for (int i = 2; i < NS - 1; ++i) {
            K2T_STAGE<16, false, MODE_PLAIN>(sm, P.st[i], 0, wlo, whi, StageCtx{});
            __syncthreads();
        }
    };
    const StageDesc &sd = P.st[NS - 1];  // radix 16, span 16: no twiddles
    const double sc = 1.0 / (double)g.M;
    const uint32_t kmax = (sd.nb + blockDim.x - 1) / blockDim.x;
    const uint32_t lane_base = (KM == kFresh ? *tmb : 0u) + ((32u * ((threadIdx.x >> 5) & 3)) << 16);
    if constexpr (KM == kFresh) {
        // the seed row's forward half, its last DIF stage scaled into this thread's TMEM columns
        forward(spec + blockIdx.x * spec_stride + (uint64_t)row * N1, false);
        uint32_t k = 0;
        for (uint32_t qb = threadIdx.x & ~31u; qb < sd.nb; qb += blockDim.x, ++k) {  // warp-uniform
            const uint32_t gq = qb + (threadIdx.x & 31);
            double2 v[16];
            if (gq < sd.nb) {
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = sm[pidx(gq * 16 + r)];
                Dft<16, false>::run(v);
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = cscale(v[r], sc);
                if (g.fout && blockIdx.x == g.fkey) {  // the handle keeps this key's seed: its spectrum row
                    double2 *so = g.fout + (uint64_t)row * N1;
#pragma unroll
                    for (int r = 0; r < 16; ++r) so[r * sd.nb + gq] = v[r];
                }
            } else {
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t w[32];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const double2 d = v[8 * h + i];
                    w[4 * i] = __double2loint(d.x);
                    w[4 * i + 1] = __double2hiint(d.x);
                    w[4 * i + 2] = __double2loint(d.y);
                    w[4 * i + 3] = __double2hiint(d.y);
                }
                tm_st32(lane_base + k1p_col(k, kmax) + 32u * h, w);
            }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        __syncthreads();  // the shared tile is the key row's next
    }
    forward(rp, true);
    TSTAMP(3);
    if constexpr (KM == kSeed) {
        grid_dep_launch();
        for (uint32_t gq = threadIdx.x; gq < sd.nb; gq += blockDim.x) {
            double2 v[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) v[r] = sm[pidx(gq * 16 + r)];
            Dft<16, false>::run(v);
#pragma unroll
            for (int r = 0; r < 16; ++r) sp[r * sd.nb + gq] = cscale(v[r], sc);
        }
        return;
    }
    if constexpr (KM == kFresh) {
        // fused_mid with the spectrum from this thread's TMEM columns
        uint32_t k = 0;
        for (uint32_t qb = threadIdx.x & ~31u; qb < sd.nb; qb += blockDim.x, ++k) {  // warp-uniform
            const uint32_t gq = qb + (threadIdx.x & 31);
            double2 s16[16];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t w[32];
                tm_ld32(lane_base + k1p_col(k, kmax) + 32u * h, w);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    s16[8 * h + i] = make_double2(__hiloint2double(w[4 * i + 1], w[4 * i]),
                                                  __hiloint2double(w[4 * i + 3], w[4 * i + 2]));
            }
            if (gq < sd.nb) {
                double2 v[16];
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = sm[pidx(gq * 16 + r)];
                Dft<16, false>::run(v);
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = cmul(v[r], s16[r]);
                Dft<16, true>::run(v);
#pragma unroll
                for (int r = 0; r < 16; ++r) sm[pidx(gq * 16 + r)] = v[r];
            }
        }
    } else {
        fused_mid<16>(sd, sm, sp);
    }
    __syncthreads();
    TSTAMP(4);
#pragma unroll
    for (int i = NS - 2; i >= 2; --i) {
        K2T_STAGE<16, true, MODE_PLAIN>(sm, P.st[i], 0, wlo, whi, StageCtx{});
        __syncthreads();
    }
    K2T_STAGE<R1, true, MODE_PLAIN>(sm, P.st[1], 0, wlo, whi, StageCtx{});
    __syncthreads();
    grid_dep_launch();  // K3 may start its prologue
    TSTAMP(5);
    rt.gin = nullptr;
    rt.gout = rq;
    rt.lr = g.lr;
    rt.lc = g.logC;
    K2T_STAGE<R0, true, MODE_TAU_OUT>(sm, P.st[0], 0, wlo, whi, rt);
    if constexpr (KM == kFresh) {
        cta_sync_tmem();
        if (threadIdx.x < 32)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(*tmb), "r"(tcols) : "memory");
    }
    TSTAMP(6);
    TRACE_END(2);
}

// the shapes k2_rows_t is instantiated for (g.k2shape: 0 = general k2_rows)
// shape-specialised K2 instantiations: rows [R0, R1, 16, ...] with NS stages (kK2[0] = general)
using K2Fn = void (*)(double2 *, double2 *, double2 *, Geometry, RouteTables, uint64_t);
struct K2Shape {
    int a, b, s;
    K2Fn fn, seed, fresh;  // hash path, seed forward half, fresh seed fused into the hash
};
#define PA_K2(A, B, S) {A, B, S, k2_rows_t<A, B, S>, k2_rows_t<A, B, S, kSeed>, k2_rows_t<A, B, S, kFresh>}
static const K2Shape kK2[] = {
    {0, 0, 0, nullptr, nullptr, nullptr},
    PA_K2(16, 16, 3),  // 4096 (C2, C3, C5a-c)
    PA_K2(5, 8, 4),    // 10240 (C4, C5d)
    PA_K2(3, 8, 4),    // 6144
    PA_K2(7, 4, 4),    // 7168
    PA_K2(2, 16, 4),   // 8192 (round 2: the calibration sweep's worst misses)
    PA_K2(3, 16, 4),   // 12288
    PA_K2(7, 5, 4),    // 8960
    PA_K2(5, 4, 4),    // 5120
    PA_K2(8, 16, 3),   // 2048
    PA_K2(3, 4, 4),    // 3072
    PA_K2(5, 5, 4),    // 6400 (round 2)
    PA_K2(7, 7, 4),    // 12544 (round 2: next to the longest plans, where the blocked / split
                       // block-length search meets it)
};
#undef PA_K2

static int k2_shape(const FftPlan &p)
{
    if (p.S < 3) return 0;
    for (int i = 2; i < p.S; ++i)
        if (p.st[i].R != 16) return 0;
    const int a = (int)p.st[0].R, b = (int)p.st[1].R;  // the stage count is a template parameter too
    for (int k = 1; k < (int)(sizeof kK2 / sizeof kK2[0]); ++k)
        if (kK2[k].a == a && kK2[k].b == b && kK2[k].s == p.S) return k;
    return 0;
}


// ------------------------------------------------------------------ K3
// Rows b of column group a0 that hold output-window bits: [b_lo, b_hi).
__device__ __forceinline__ void k3_window_rows(const Geometry &g, uint32_t a0, uint32_t C, uint64_t n, uint64_t m,
                                               int64_t *blo, int64_t *bhi)
{
    const int64_t t0 = (int64_t)n - 1, t1 = t0 + (int64_t)m;  // output window [t0, t1)
    // only rows b holding some t in the window: u = a0 + c + N1 b (Re) or u + M (Im)
    auto row_lo = [&](int64_t tmin) -> int64_t {  // first b with a0 + C - 1 + N1 b >= tmin
        int64_t d = tmin - (int64_t)a0 - (int64_t)(C - 1);
        return d <= 0 ? 0 : (d + g.N1 - 1) / g.N1;
    };
    auto row_hi = [&](int64_t tmax) -> int64_t {  // one past the last b with a0 + N1 b < tmax
        int64_t d = tmax - (int64_t)a0;
        return d <= 0 ? 0 : std::min<int64_t>((int64_t)g.N2, (d + g.N1 - 1) / g.N1);
    };
    const int64_t rb0 = row_lo(t0), rb1 = row_hi(t1);
    const int64_t ib0 = row_lo(t0 - (int64_t)g.M), ib1 = row_hi(t1 - (int64_t)g.M);
    *blo = std::min(rb1 > rb0 ? rb0 : (int64_t)g.N2, ib1 > ib0 ? ib0 : (int64_t)g.N2);
    *bhi = std::max(rb1 > rb0 ? rb1 : 0, ib1 > ib0 ? ib1 : 0);
}

// Window + parity + packing of one column group (threads tid, tid + nth, ...; nth a multiple
// of 32 and of C).  Element (b, c) is w[u], u = a0 + c + N1 b; Re -> c[u], Im -> c[u + M].
// Returns this thread's largest |v - rint v| over window values.
// FR >= 2: the last inverse stage (radix FR, span N2, Ls = N2 / FR) is not run over the
// whole tile; each window element takes it here from the previous stage's output instead:
// row b = j + k Ls gets sum_r v[j + r Ls] conj(w_N2^{r b}) (the stage's twiddle and inverse
// DFT_R in one), so only window rows pay for it.
template <int FR = 0>
__device__ __forceinline__ double k3_epilogue(const double2 *sm, const Geometry &g, uint32_t a0, uint32_t logC,
                                              uint64_t n, uint64_t m, const double2 *thlo, const double2 *thhi,
                                              uint32_t *out, uint32_t b_lo, uint32_t b_hi, uint32_t tid, uint32_t nth,
                                              const double2 *wlo = nullptr, const double2 *whi = nullptr)
{
    const uint32_t C = 1u << logC;
    const int64_t t0 = (int64_t)n - 1, t1 = t0 + (int64_t)m;
    const uint32_t lane = tid & 31;
    const uint32_t runmask = (C == 32) ? 0xFFFFFFFFu : ((1u << C) - 1u);
    double rmax = 0.0;
    const uint32_t e_lo = b_hi > b_lo ? (b_lo << logC) : 0;
    const uint32_t e_hi = b_hi > b_lo ? (b_hi << logC) : 0;
    for (uint32_t e = e_lo + tid; e < e_hi; e += nth) {
        const uint32_t b = e >> logC, c = e & (C - 1);
        double2 x;
        if constexpr (FR >= 2) {
            const uint32_t Ls = g.f2.st[0].Ls;
            const uint32_t j = b - (uint32_t)(((uint64_t)b * g.f2.st[0].magic) >> 40) * Ls;  // b mod Ls
            const double2 w1 = twiddle(wlo, whi, b);  // w_N2^b
            double2 p = w1;
            x = cadd(sm[pidx((j << logC) + c)], cmulc(sm[pidx(((j + Ls) << logC) + c)], w1));
#pragma unroll
            for (int r = 2; r < FR; ++r) {
                p = cmul(p, w1);  // w_N2^{r b}
                x = cadd(x, cmulc(sm[pidx(((j + r * Ls) << logC) + c)], p));
            }
        } else {
            x = sm[pidx(e)];
        }
        const double2 wv = cmulc(x, twiddle(thlo, thhi, b));
        const int64_t u = (int64_t)a0 + c + (int64_t)g.N1 * b;
#pragma unroll
        for (int part = 0; part < 2; ++part) {
            const int64_t tt = part ? u + (int64_t)g.M : u;
            const double v = part ? wv.y : wv.x;
            const bool in = tt >= t0 && tt < t1;
            const double r = rint(v);
            if (in) rmax = fmax(rmax, fabs(v - r));
            const bool bit = in && (((long long)r) & 1);
            const uint32_t bal = __ballot_sync(__activemask(), bit);
            // lanes c = 0..C-1 of a run hold C consecutive output bits starting at i0
            uint32_t run = (bal >> (lane - c)) & runmask;
            if (c == 0 && run) {
                int64_t i0 = tt - t0;
                if (i0 < 0) {
                    run >>= (int)(-i0);
                    i0 = 0;
                }
                const uint64_t wd = (uint64_t)i0 >> 5;
                const int sh = (int)(i0 & 31);
                // XOR: each output bit is produced once per hash, so on the zeroed output this
                // equals OR; column blocks of the Eq. (4) split accumulate Eq. (7) in place
                atomicXor(out + wd, run << sh);
                if (sh && (run >> (32 - sh))) atomicXor(out + wd + 1, run >> (32 - sh));
            }
        }
    }
    return rmax;
}

__device__ __forceinline__ void k3_residual(double rmax, unsigned long long *resid)
{
#pragma unroll
    for (int d = 16; d; d >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xFFFFFFFFu, rmax, d));
    if ((threadIdx.x & 31) == 0 && rmax > 0.0) atomicMax(resid, (unsigned long long)__double_as_longlong(rmax));
}

template <int RA, int RB, int RC>
__global__ void __launch_bounds__(PA_TMAX, PA_MINB)
k3_inv_columns(const double2 *__restrict__ buf, Geometry g, RouteTables T, uint64_t n, uint64_t m,
               uint32_t *__restrict__ out, unsigned long long *__restrict__ resid, uint64_t out_stride)
{
    buf += (uint64_t)blockIdx.y * g.M;                        // batch: key blockIdx.y
    out += blockIdx.y * out_stride;
    extern __shared__ double2 sm[];
    const uint32_t logC = g.logC, C = 1u << logC;
    double2 *wlo = sm + g.tile1, *whi = wlo + 64, *thlo = whi + g.f2.nhi + g.f2.ntw, *thhi = thlo + 64;
    const uint32_t a0 = blockIdx.x * C;
    const uint32_t tot = g.N2 << logC;
    // the last inverse stage (radix RA <= 7 of a specialised plan, S >= 2) is taken inside the
    // epilogue for the window rows only
    constexpr bool kFuse = RA >= 2 && RA <= 7;
    TRACE_BEGIN(3);
    TSTAMPK(2, 0);
    load_tables_async(wlo, whi, T.W2lo, T.W2hi, g.f2.nhi + g.f2.ntw);
    load_tables_async(thlo, thhi, T.thlo, T.thhi, g.f2.nhi);
    grid_dep_wait();  // K2's rows
    // first inverse stage reads the columns straight from global when the per-row chunk is
    // >= 64 B (C >= 4); with 32 B chunks (C = 2) the staged cp.async copy is faster (round 1:
    // C4 K3 731 vs 986 us; C5c at C = 4 117 -> 111 us, C3 at C = 8 68 -> 64.5 us)
    const bool direct = g.f2.S > 1 && C >= 4;
    // staged tiles load in KP parts (separate cp.async groups), and the first inverse stage
    // (radix 16 over 16 consecutive rows: Ls = 1) runs on each part as soon as it has landed, under
    // the loads of the later parts (developer override PA_K3_PARTS=1 for the single-wait form)
    const uint32_t kp = !direct && g.k3parts > 1 && g.f2.S > 1 && g.f2.st[g.f2.S - 1].Ls == 1 ? g.k3parts : 1;
    if (!direct) {
        for (uint32_t p = 0; p < kp; ++p) {
            const uint32_t e0 = tot / kp * p, e1 = p + 1 == kp ? tot : tot / kp * (p + 1);
            for (uint32_t e = e0 + threadIdx.x; e < e1; e += blockDim.x)
                cp_async16(sm + pidx(e), buf + wrow(g, e >> logC) + ((uint64_t)a0 << g.lr) + (e & (C - 1)));
            asm volatile("cp.async.commit_group;\n" ::: "memory");
        }
    }
    int64_t b_lo, b_hi;
    k3_window_rows(g, a0, C, n, m, &b_lo, &b_hi);
    int s_hi = g.f2.S;  // stages [lo, s_hi) of the DIT still to run
    if (kp > 1) {
        const StageDesc &sd = g.f2.st[g.f2.S - 1];
        const uint32_t nbq = sd.nb << logC;  // butterflies of the stage; part p owns an equal slice
        for (uint32_t p = 0; p < kp; ++p) {
            switch (kp - 1 - p) {  // groups still allowed in flight
            case 0: asm volatile("cp.async.wait_group 0;\n" ::: "memory"); break;
            case 1: asm volatile("cp.async.wait_group 1;\n" ::: "memory"); break;
            case 2: asm volatile("cp.async.wait_group 2;\n" ::: "memory"); break;
            default: asm volatile("cp.async.wait_group 3;\n" ::: "memory"); break;
            }
            __syncthreads();
            StageCtx px;
            px.q0 = nbq / kp * p;
            px.q1 = p + 1 == kp ? nbq : nbq / kp * (p + 1);
            stage_t<true, MODE_PLAIN, RA, RB, RC>(sm, g.f2, g.f2.S - 1, logC, wlo, whi, px);
        }
        __syncthreads();
        s_hi = g.f2.S - 1;
    } else {
        cp_async_wait_all();  // tables (and the staged tile)
        __syncthreads();
    }
    TSTAMPK(2, 1);
    if (direct) {
        StageCtx gx;
        gx.gin = buf + ((uint64_t)a0 << g.lr);
        gx.ld = g.N1 << g.lr;
        gx.lr = g.lr;
        gx.lc = logC;
        stage_t<true, MODE_GCOL, RA, RB, RC>(sm, g.f2, g.f2.S - 1, logC, wlo, whi, gx);
        __syncthreads();
        dit_t<RA, RB, RC>(sm, g.f2, kFuse ? 1 : 0, g.f2.S - 1, logC, wlo, whi);
    } else {
        dit_t<RA, RB, RC>(sm, g.f2, kFuse ? 1 : 0, s_hi, logC, wlo, whi);
    }
    TSTAMPK(2, 2);
    const double rmax = k3_epilogue<kFuse ? RA : 0>(sm, g, a0, logC, n, m, thlo, thhi, out, (uint32_t)b_lo,
                                                    (uint32_t)b_hi, threadIdx.x, blockDim.x, wlo, whi);
    TSTAMPK(2, 3);
    k3_residual(rmax, resid);
    TRACE_END(3);
}

// ------------------------------------------------------------------ K3T (TMEM-staged K3)
// K3 for 32-byte column groups (C = 2) when its grid runs many waves of one CTA per SM (C4,
// C5d).  There the tile load -- N2 scattered 32-byte row pieces -- is a third of K3's time and
// nothing overlaps it: shared memory holds one tile.  Tensor memory (256 KB per SM, otherwise
// idle in this library) holds the next one.  Persistent CTAs (one per SM); warps 0..11 run the
// inverse stages and the window epilogue of tile t from shared memory while warps 12..15, one
// per TMEM lane quarter, load tile t + gridDim.x from HBM into TMEM (ld.global -> tcgen05.st);
// at the switch the compute warps copy TMEM -> shared memory (tcgen05.ld, ~3 k cycles instead
// of a ~13 k-cycle HBM load).  TMEM layout: lane p holds rows b = p + 128 i, columns
// [8 i, 8 i + 8) = the row's two complex values (4 words each).
constexpr uint32_t kK3tCompute = 384;  // compute threads (12 warps); 4 loader warps follow

// loader warps: tile t of the batch into TMEM (8 rows = 16 x 16 B loads in flight per batch)
__device__ __forceinline__ void k3t_load_tile(const double2 *__restrict__ buf, const Geometry &g, uint32_t t,
                                              uint32_t ngroups, uint32_t tm)
{
    const uint32_t key = t / ngroups, grp = t % ngroups;
    const double2 *src = buf + (size_t)key * g.M + ((size_t)grp * 2 << g.lr);
    const uint32_t q = (threadIdx.x >> 5) & 3, p = 32 * q + (threadIdx.x & 31);
    const uint32_t rpl = (g.N2 + 127) / 128;  // rows per lane (planner: <= 64)
    // registers bound the loads in flight (8 rows per thread, ~32 KB per SM): first pull every
    // row piece of this lane into L2 (no registers), so the batches below hit L2
    for (uint32_t i = 0; i < rpl; ++i) {
        const uint32_t b = p + 128 * i;
        if (b < g.N2) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + wrow(g, b)) : "memory");
    }
    for (uint32_t i0 = 0; i0 < rpl; i0 += 8) {
        double2 v[16];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t b = p + 128 * (i0 + k);
            if (i0 + k < rpl && b < g.N2) {
                v[2 * k] = __ldg(src + wrow(g, b));
                v[2 * k + 1] = __ldg(src + wrow(g, b) + 1);
            } else {
                v[2 * k] = v[2 * k + 1] = make_double2(0.0, 0.0);
            }
        }
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            if (i0 + 4 * s < rpl) {  // warp-uniform
                uint32_t r[32];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double2 d = v[8 * s + k];
                    r[4 * k] = __double2loint(d.x);
                    r[4 * k + 1] = __double2hiint(d.x);
                    r[4 * k + 2] = __double2loint(d.y);
                    r[4 * k + 3] = __double2hiint(d.y);
                }
                tm_st32(tm + ((32 * q) << 16) + 8 * (i0 + 4 * s), r);
            }
        }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(PA_TMAX, 1)
k3t_inv_columns(const double2 *__restrict__ buf, Geometry g, RouteTables T, uint64_t n, uint64_t m,
                uint32_t *__restrict__ out, unsigned long long *__restrict__ resid, uint64_t out_stride,
                uint32_t count)
{
    extern __shared__ double2 sm[];
    __shared__ uint32_t tm_base;
    constexpr uint32_t C = 2, logC = 1;
    double2 *wlo = sm + g.tile1, *whi = wlo + 64, *thlo = whi + g.f2.nhi + g.f2.ntw, *thhi = thlo + 64;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t ngroups = g.N1 / C, ntiles = ngroups * count;
    const bool loader = threadIdx.x >= kK3tCompute;
    load_tables(wlo, whi, T.W2lo, T.W2hi, g.f2.nhi + g.f2.ntw);
    load_tables(thlo, thhi, T.thlo, T.thhi, g.f2.nhi);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&tm_base)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    cta_sync_tmem();
    const uint32_t tm = tm_base;
    grid_dep_wait();  // K2's rows
    uint32_t t = blockIdx.x;
    if (loader && t < ntiles) k3t_load_tile(buf, g, t, ngroups, tm);
    double rmax = 0.0;
    const uint32_t rpl = (g.N2 + 127) / 128, nchunk = (rpl + 3) / 4;
    for (; t < ntiles; t += gridDim.x) {
        cta_sync_tmem();  // TMEM holds tile t; the shared tile is free
        if (!loader) {
            // TMEM -> shared memory: warp w reads lane quarter w & 3, column chunks w >> 2, +3, ..
            const uint32_t q = warp & 3, p = 32 * q + lane;
            for (uint32_t ch = warp >> 2; ch < nchunk; ch += 3) {
                uint32_t r[32];
                tm_ld32(tm + ((32 * q) << 16) + 32 * ch, r);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t b = p + 128 * (4 * ch + k);
                    if (b < g.N2) {
                        sm[pidx(2 * b)] = make_double2(__hiloint2double(r[8 * k + 1], r[8 * k]),
                                                       __hiloint2double(r[8 * k + 3], r[8 * k + 2]));
                        sm[pidx(2 * b + 1)] = make_double2(__hiloint2double(r[8 * k + 5], r[8 * k + 4]),
                                                           __hiloint2double(r[8 * k + 7], r[8 * k + 6]));
                    }
                }
            }
        }
        cta_sync_tmem();  // TMEM consumed, tile t in shared memory
        if (loader) {
            if (t + gridDim.x < ntiles) k3t_load_tile(buf, g, t + gridDim.x, ngroups, tm);
            continue;
        }
        const uint32_t key = t / ngroups, a0 = (t % ngroups) * C;
        StageCtx cx;
        cx.nth = kK3tCompute;
        for (int i = g.f2.S - 1; i >= 0; --i) {
            stage_any<true>(sm, g.f2.st[i], logC, wlo, whi, cx);
            asm volatile("bar.sync 1, %0;" ::"r"(kK3tCompute) : "memory");
        }
        int64_t b_lo, b_hi;
        k3_window_rows(g, a0, C, n, m, &b_lo, &b_hi);
        rmax = fmax(rmax, k3_epilogue(sm, g, a0, logC, n, m, thlo, thhi, out + key * out_stride, (uint32_t)b_lo,
                                      (uint32_t)b_hi, threadIdx.x, kK3tCompute));
    }
    if (!loader) k3_residual(rmax, resid);
    cta_sync_tmem();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm) : "memory");
}

// K1 / K3 instantiations for column plans [A, B, (C), 16, ...]: 0 general, then C2 [2, 5, 16],
// C3 [3, 4, 7, 16], C4 [3, 8, 16, 16], C5a/c [3, 3, 16(, 16)], C5b [7, 4, 16], C5d [3, 7, 8, 16]
using K1Fn = void (*)(const uint32_t *, double2 *, Geometry, RouteTables, uint32_t *, uint64_t, uint64_t,
                      const uint32_t *, uint64_t, uint64_t);
using K3Fn = void (*)(const double2 *, Geometry, RouteTables, uint64_t, uint64_t, uint32_t *, unsigned long long *,
                      uint64_t);
using K1pFn = void (*)(const uint32_t *, double2 *, Geometry, RouteTables, uint32_t *, uint64_t, uint64_t, uint32_t);
struct K13 {
    int a, b, c;
    K1Fn k1;
    K3Fn k3;
    K1pFn k1p;
};
#define PA_K13(A, B, C) {A, B, C, k1_fwd_columns<A, B, C>, k3_inv_columns<A, B, C>, k1p_fwd_columns<A, B, C>}
static const K13 kK13[] = {
    PA_K13(0, 0, 0), PA_K13(2, 5, 0), PA_K13(3, 4, 7), PA_K13(3, 8, 0), PA_K13(3, 3, 0), PA_K13(7, 4, 0),
    PA_K13(3, 7, 8),
    // round 2: column lengths the planner reaches for other n (4096, 2048, 1024, 768, 1280, 3072)
    // ([16, 16, 16] columns were tried too: the planner then took 4096-column plans that measured
    // slower -- C5d 7168 x 4096 1040 vs 10240 x 2688 888 us per batched key -- so they stay general)
    PA_K13(8, 16, 0), PA_K13(4, 16, 0), PA_K13(3, 16, 0), PA_K13(5, 16, 0), PA_K13(3, 4, 0),
};
#undef PA_K13

static int k13_shape(const FftPlan &p)
{
    if (p.S < 2) return 0;
    const int a = (int)p.st[0].R, b = (int)p.st[1].R;
    const int c = p.S >= 3 && p.st[2].R != 16 ? (int)p.st[2].R : 0;
    const int from = c ? 3 : 2;
    if (p.S < from + 1) return 0;
    for (int i = from; i < p.S; ++i)
        if (p.st[i].R != 16) return 0;
    for (int k = 1; k < (int)(sizeof kK13 / sizeof kK13[0]); ++k)
        if (kK13[k].a == a && kK13[k].b == b && kK13[k].c == c) return k;
    return 0;
}

// ------------------------------------------------------------------ host plan
std::vector<uint32_t> smooth_numbers(uint32_t limit)
{
    std::vector<uint32_t> v;
    for (uint64_t a = 1; a <= limit; a *= 2)
        for (uint64_t b = a; b <= limit; b *= 3)
            for (uint64_t c = b; c <= limit; c *= 5)
                for (uint64_t d = c; d <= limit; d *= 7) v.push_back((uint32_t)d);
    std::sort(v.begin(), v.end());
    return v;
}

static bool asc_off()  // developer override PA_K13_ASC=0: K1/K3 plans in the default radix order
{
    const char *e = dev_env("PA_K13_ASC");
    return e && atoi(e) == 0;
}

bool make_plan(uint32_t Lt, FftPlan *P, uint32_t rmax = 16, bool ascending = false)
{
    uint32_t L = Lt;
    int e2 = 0, e3 = 0, e5 = 0, e7 = 0;
    while (L % 2 == 0) { L /= 2; ++e2; }
    while (L % 3 == 0) { L /= 3; ++e3; }
    while (L % 5 == 0) { L /= 5; ++e5; }
    while (L % 7 == 0) { L /= 7; ++e7; }
    if (L != 1) return false;
    int R[kMaxStages], S = 0;
    auto push = [&](int r) { if (S < kMaxStages) R[S++] = r; };
    // odd radices first (large spans: lanes take consecutive j), then powers of two
    // ascending so the small-span stages are radix 16 / 8 on the padded layout -- this
    // order keeps every stage's quarter-warp accesses bank-conflict free for the
    // plans the planner emits (modelled in DESIGN.md Sec. 5)
    for (int i = 0; i < e7; ++i) push(7);
    for (int i = 0; i < e5; ++i) push(5);
    for (int i = 0; i < e3; ++i) push(3);
    if (rmax >= 16) {
        if (e2 % 4 == 1) push(2);
        if (e2 % 4 == 2) push(4);
        if (e2 % 4 == 3) push(8);
        for (int i = 0; i < e2 / 4; ++i) push(16);
    } else {  // radix <= 8: more, lighter stages (one butterfly per thread at 512 threads)
        if (e2 % 3 == 1) push(2);
        if (e2 % 3 == 2) push(4);
        for (int i = 0; i < e2 / 3; ++i) push(8);
    }
    // ascending: the smallest radix first (K1/K3, see ra_plan)
    if (ascending) std::stable_sort(R, R + S);
    P->S = S;
    P->Lt = Lt;
    P->nhi = (Lt + 63) / 64;
    uint32_t span = Lt, off = P->nhi;  // per-stage tables follow the plan's hi[] table
    for (int i = 0; i < S; ++i) {
        StageDesc &d = P->st[i];
        d.R = (uint32_t)R[i];
        d.L = span;
        d.Ls = span / d.R;
        d.G = Lt / span;
        d.nb = Lt / d.R;
        d.magic = ((1ull << 40) + d.Ls - 1) / d.Ls;
        d.toff = 0;
        if (d.G > 1 && d.Ls > 1) {  // Ls = 1: j = 0 only, no twiddles
            d.toff = off;
            off += d.Ls > 64 ? 64 + (d.Ls + 63) / 64 : d.Ls;
        }
        span = d.Ls;
    }
    P->ntw = off - P->nhi;
    return S < kMaxStages;
}

uint32_t tile_bytes(uint64_t elems) { return (uint32_t)((elems + (elems >> 4) + 1) * 16); }

}  // namespace

static uint32_t kb_words(uint32_t N2, uint32_t C)  // K0 stream words per group (16-byte multiple)
{
    const uint32_t epw = 16 / C;
    return ((N2 + epw - 1) / epw + 3) / 4 * 4;
}
// tile | twiddle tables (lo, hi, per-stage) | theta (K1/K3) or rho (K2) tables | K1 bit stream
static uint32_t smem_k13(uint32_t N2, uint32_t C, const FftPlan &p2)
{
    return tile_bytes((uint64_t)N2 * C) + (2 * (64 + p2.nhi) + p2.ntw) * 16 + kb_words(N2, C) * 4;
}
static uint32_t smem_k2(uint32_t N1, const FftPlan &p1) { return tile_bytes(N1) + (2 * (64 + p1.nhi) + p1.ntw) * 16; }

// every candidate plan the cost model scored (ra_plan_candidates: measured planning,
// PA_PLAN_MEASURE; pa_dev_plan_features in the developer build)
struct PlanCand {
    double cost;
    uint32_t N1, N2, C;
    double f[9];  // thr13, lat13, thr2, lat2, spec13, spec2, k1p, occ13, occ2 (calibration features)
};
constexpr int kMaxCand = 256;  // the cheapest kMaxCand candidates (a plan search scores thousands)
static thread_local PlanCand g_cand[kMaxCand];
static thread_local int g_ncand = 0;
static thread_local bool g_cand_on = false;
static void keep_cand(const PlanCand &c)
{
    if (g_ncand < kMaxCand) {
        g_cand[g_ncand++] = c;
        return;
    }
    int worst = 0;
    for (int i = 1; i < kMaxCand; ++i)
        if (g_cand[i].cost > g_cand[worst].cost) worst = i;
    if (c.cost < g_cand[worst].cost) g_cand[worst] = c;
}

// the cost model's time (seconds per hash) of the plan the last ra_plan call on this thread chose
static thread_local double g_plan_cost = 0.0;
double ra_last_plan_cost() { return g_plan_cost; }
// whether a planned (N1, N2) runs the shape-specialised K2 and K1 / K3 (the kernels the cost
// model is calibrated on; the general ones measured 16-23% slower per point on 10^8-point plans)
bool ra_plan_specialised(const Geometry &g);

pa_status ra_plan(uint64_t n, uint64_t m, Geometry *g, char *err, size_t errlen, uint64_t max_len,
                  const PlanChoice *force)
{
    const uint64_t L = n + m - 1;
    const uint64_t Mmin = (L + 1) / 2;
    static const std::vector<uint32_t> sm = smooth_numbers(32768);
    double best = 1e300;
    bool found = false;
    // Cost model (per hash), calibrated on B200 with tools/quick_time.py + PA_FORCE_PLAN:
    //  - every FFT stage pass costs ~0.55 cycles per element per SM (shared-memory
    //    round trip + FP64 butterfly; measured 0.5-0.6 across plans),
    //  - HBM bytes at the column-group bandwidth of the access run (K1, K3) or 6.2 TB/s,
    //  - with one CTA per SM memory and compute serialise, with two they overlap,
    //  - a CTA needs >= ~1.6 us per stage pass whatever its size (latency floor).
    const double sm_rate = 148.0 * 1.9e9;
    for (uint32_t N1 : sm) {
        if (tile_bytes(N1) > kSmemLimit) break;
        FftPlan p1;
        if (!make_plan(N1, &p1) || smem_k2(N1, p1) > kSmemLimit) continue;
        uint64_t need = (Mmin + N1 - 1) / N1;
        if (need > 32768) continue;
        // every smooth N2 within +12% of the minimum: a longer but radix-16-friendly
        // length often needs fewer passes than the tightest fit
        auto it0 = std::lower_bound(sm.begin(), sm.end(), (uint32_t)need);
        for (auto it = it0; it != sm.end() && *it <= need * 1.12 + 16; ++it) {
        const uint32_t N2 = *it;
        if (max_len && 2ull * N1 * N2 > max_len) continue;
        FftPlan p2;
        if (!make_plan(N2, &p2)) continue;
        for (uint32_t C = 16; C >= 1; C >>= 1) {
            if (N1 % C) continue;
            uint32_t s13 = smem_k13(N2, C, p2);
            if (s13 > kSmemLimit) continue;
            // measured: every FFT stage pass (and the load / store / twiddle passes around
            // them) costs ~0.62 cycles per element per SM, largely independent of the radix
            const double M = (double)N1 * N2;
            // radix-16 / 8 stages take one or two rounds per thread; the low radices several and
            // measured ~25% dearer per pass (C5a: 2304 = [3, 3, 16, 16] rows lose to 4096 = 16^3)
            auto wsum = [](const FftPlan &p) {
                double w = 0;
                for (int i = 0; i < p.S; ++i) w += p.st[i].R >= 8 ? 1.0 : 1.25;
                return w;
            };
            // radix weights for the column plan as well (round 2: n = 10^6, m = 10^5 took 2048 x 280
            // = [7, 5, 8] columns at 44.0 us over 4096 x 144 = [3, 3, 16] at 33.8 us)
            const double pass13 = wsum(p2) + 2.0, pass2 = 2.0 * wsum(p1) + 1.0;
            const double cfac = C == 1 ? 1.5 : C == 2 ? 1.0 : 0.95;  // short HBM runs (K1/K3)
            const uint32_t occ13 = std::min<uint32_t>(2, kSmemLimit / s13);
            const uint32_t occ2 = std::min<uint32_t>(2, kSmemLimit / smem_k2(N1, p1));
            auto ktime = [&](double passes, double fac, uint32_t occ, double ctas) {
                double thr = M * passes * 0.62 * fac / sm_rate;
                double waves = std::ceil(ctas / (148.0 * occ));
                return std::max(thr, waves * passes * 1.3e-6) + 2e-6;
            };
            // two CTAs per SM overlap one tile's HBM phases with the other's compute (measured:
            // C3 at C = 4, 2 per SM, 192 us vs C = 8, 1 per SM, 206 us -- same waves)
            const double ov13 = occ13 >= 2 ? 0.92 : 1.0, ov2 = occ2 >= 2 ? 0.92 : 1.0;
            // the shape-specialised kernels (k2_rows_t, the kK13 instantiations) run faster than the
            // general ones: prefer plans that have them
            FftPlan p2a;
            const bool spec13 = k13_shape(p2) || (make_plan(N2, &p2a, 16, true) && k13_shape(p2a));
            const double f2 = k2_shape(p1) ? 0.9 : 1.0, f13 = spec13 ? 0.95 : 1.0;
            // K1 runs as the persistent TMEM write-behind K1P on one-CTA-per-SM multi-wave plans
            // (C4: K1 735 -> 670 us; the calibration sweep, tools/dev/plan_calib.py, found the
            // model preferring two-CTA C = 2 plans over faster K1P C = 4 ones without this)
            const bool k1p = spec13 && occ13 == 1 && C >= 2 && C < 16 && N1 / C >= 2 * 148u && p2.S >= 3 &&
                             p2.st[p2.S - 1].R == 16;
            // (a grid refit of the throughput scales on 70 random single-key lengths x 12 plans,
            // tools/dev/plan_refit.py, cut the mean regret 2.9% -> 1.6% there but lost on held-out
            // shapes and batches -- C5b batched 46.0 -> 48.2 us/key, n = 5e7, m = 1e7 1137 -> 1233
            // us -- so the calibrated throughput terms stay as they are)
            const double t13 = f13 * ktime(pass13, cfac * ov13, occ13, (double)(N1 / C));
            double cost = t13 * (k1p ? 0.91 : 1.0) + t13 + f2 * ktime(pass2, ov2, occ2, (double)N2);
            if (g_cand_on) {
                const double th13 = M * pass13 * 0.62 * cfac * ov13 / sm_rate;
                const double la13 = std::ceil((double)(N1 / C) / (148.0 * occ13)) * pass13 * 1.3e-6;
                const double th2 = M * pass2 * 0.62 * ov2 / sm_rate;
                const double la2 = std::ceil((double)N2 / (148.0 * occ2)) * pass2 * 1.3e-6;
                keep_cand({cost, N1, N2, C, {th13, la13, th2, la2, spec13 ? 1.0 : 0.0, k2_shape(p1) ? 1.0 : 0.0,
                                             k1p ? 1.0 : 0.0, (double)occ13, (double)occ2}});
            }
            if (cost < best) {
                best = cost;
                g_plan_cost = cost;
                found = true;
                g->M = (uint64_t)N1 * N2;
                g->N1 = N1;
                g->N2 = N2;
                g->C = C;
            }
        }
        }
    }
    // a plan chosen by measurement (PA_PLAN_MEASURE, pa_api.cu) or the developer override
    // PA_FORCE_PLAN="N1,N2,C" replaces the model's choice when it is valid for (n, m)
    auto apply_force = [&](unsigned f1, unsigned f2, unsigned fc) {
        FftPlan q1, q2;
        if ((uint64_t)f1 * f2 >= Mmin && fc >= 1 && fc <= 16 && (fc & (fc - 1)) == 0 && f1 % fc == 0 &&
            (!max_len || 2ull * f1 * f2 <= max_len) && make_plan(f1, &q1) && make_plan(f2, &q2) &&
            smem_k2(f1, q1) <= kSmemLimit && smem_k13(f2, fc, q2) <= kSmemLimit) {
            g->N1 = f1;
            g->N2 = f2;
            g->C = fc;
            g->M = (uint64_t)f1 * f2;
            found = true;
        }
    };
    if (force) apply_force(force->N1, force->N2, force->C);
    if (const char *fp = dev_env("PA_FORCE_PLAN")) {
        unsigned f1 = 0, f2 = 0, fc = 0;
        if (sscanf(fp, "%u,%u,%u", &f1, &f2, &fc) == 3) apply_force(f1, f2, fc);
    }
    if (!found) {
        snprintf(err, errlen,
                 "route (a): n+m-1 = %llu needs a complex transform of length >= %llu, beyond the "
                 "two-pass plan's limit%s",
                 (unsigned long long)L, (unsigned long long)Mmin,
                 max_len ? " or pa_options.max_transform_len" : "");
        return PA_ERR_UNSUPPORTED;
    }
    uint32_t logC = 0;
    while ((1u << logC) < g->C) ++logC;
    g->logC = logC;
    const char *r1 = dev_env("PA_FORCE_RMAX1");  // developer override: row-plan radix cap
    make_plan(g->N1, &g->f1, r1 ? (uint32_t)atoi(r1) : 16);
    // K1/K3: the radices in ascending order when that puts a radix-2 or -3 stage first (K1 then
    // reads the key bits through an 8- or 24-entry table, k_bits_table).  Same-box: C2 [2, 5, 16]
    // K1 14.2 -> 12.8 us (bench 26.4 -> 27.1 Gbit/s), C3 [3, 4, 7, 16] 186.4 -> 182.3 us, C5d
    // [3, 7, 8, 16] 1005.6 -> 983 us; C5b's [4, 7, 16] (radix 4 first) measured slower and keeps
    // [7, 4, 16]
    make_plan(g->N2, &g->f2);
    if (!asc_off()) {
        FftPlan q;
        if (make_plan(g->N2, &q, 16, true) && q.S >= 2 && q.st[0].R <= 3 && q.st[0].R < g->f2.st[0].R) g->f2 = q;
    }
    g->tile1 = tile_bytes((uint64_t)g->N2 * g->C) / 16;
    g->tile2 = tile_bytes(g->N1) / 16;
    g->smem1 = smem_k13(g->N2, g->C, g->f2);
    g->kbw = kb_words(g->N2, g->C);
    g->smem2 = smem_k2(g->N1, g->f1);
    // 256 threads when two CTAs share an SM (<= 128 registers each), else 512
    g->t1 = 2 * g->smem1 <= kSmemLimit ? PA_TMAX / 2 : PA_TMAX;
    g->t2 = 2 * g->smem2 <= kSmemLimit ? PA_TMAX / 2 : PA_TMAX;
    // K2: L2 prefetch of the row pf2 rows ahead when one CTA per SM runs > 2 waves (C4, C5d); it
    // measured slower at two CTAs per SM
    {
        const char *e = dev_env("PA_PF");
        // distance in rows: 56 (a third of a wave; same-box sweep C4 / C5d: 8 -> 1040 us at C5d,
        // 37-74 -> 2405-2410 / 1010-1012 us, 148 -> 2424 / 1019, 296 -> 2494 / 1070, off -> 2529 /
        // 1067).  Developer override PA_PF=0 (off) or PA_PF=d
        const uint32_t dist = e ? (uint32_t)atoi(e) : 56u;
        g->pf2 = dist && g->t2 == PA_TMAX && g->N2 > 2 * 148u ? dist : 0;
    }
    // K1/K2/K3 specialised for the common plan shapes (developer override PA_K2_T=0 / PA_K13_T=0)
    {
        const char *e = dev_env("PA_K2_T");
        g->k2shape = (!e || atoi(e) != 0) ? k2_shape(g->f1) : 0;
        // pa_hash_fresh_batch: the seeds' forward half fused into the hash's K2 (developer
        // override PA_K2_FRESH=0: per-key spectra through HBM)
        const char *ef = dev_env("PA_K2_FRESH");
        g->k2fresh = g->k2shape && (!ef || atoi(ef) != 0);
        g->fout = nullptr;
        g->fkey = 0;
        const char *e13 = dev_env("PA_K13_T");
        g->k13 = (!e13 || atoi(e13) != 0) ? k13_shape(g->f2) : 0;
    }
    // K1's first stage straight from the key bits through a 2^R0 x R0 table (radix R0 <= 4 of a
    // shape-specialised K1, see k1_fwd_columns; not when the extra shared memory would cost a CTA
    // per SM).
    // Developer override PA_K1_BITS=0
    {
        // K0 tile (developer overrides PA_K0_RB / PA_K0_CB).  Larger tiles (fewer CTAs) measured
        // slower: C3 64 x 256 / 64 x 512 / 64 x 1024 -> K0 9.7-13.8 / 20.2 us vs 10.3 us at 16 x 256
        const char *er = dev_env("PA_K0_RB"), *ec = dev_env("PA_K0_CB");
        g->k0rb = er ? (uint32_t)atoi(er) : g->N2 >= 2048 ? 64u : 16u;
        g->k0cb = ec ? (uint32_t)atoi(ec) : g->N1 >= 8192 ? 1024u : 256u;
        if (g->k0rb % 16 || g->k0rb > kK0Rows || g->k0rb == 0) g->k0rb = 16;
        if (g->k0cb % 32 || g->k0cb > kK0Cols || g->k0cb == 0) g->k0cb = 256;
    }
    g->ntb = 0;
    {
        const char *e = dev_env("PA_K1_BITS");
        const uint32_t R0 = g->f2.S ? g->f2.st[0].R : 16u;
        if ((!e || atoi(e) != 0) && g->k13 && g->f2.S >= 2 && R0 <= 4) {
            const uint32_t ntb = (1u << R0) * R0, s1 = g->smem1 + ntb * 16;
            if (s1 <= kSmemLimit && (2 * g->smem1 > kSmemLimit || 2 * s1 <= kSmemLimit)) {
                g->ntb = ntb;
                g->smem1 = s1;
            }
        }
    }
    // row blocks for K2's output / K3's input (opt-in PA_LR=1): 128-byte K3 runs for 2- and
    // 4-column groups.  Bit-exact, but K2's stores become 32-byte pieces: C4 K3 725 -> 627, K2
    // 1119 -> 1208 us (net 0), C5d -1.8%, so row-major stays the default
    {
        const char *e = dev_env("PA_LR");
        const uint32_t lr = g->C == 2 ? 2u : g->C == 4 ? 1u : 0u;
        g->lr = e && atoi(e) == 1 && g->N2 % (1u << lr) == 0 ? lr : 0u;
    }
    // K3T (TMEM-staged K3): opt-in, PA_K3T=1.  Bit-exact, but measured slower than K3 (C4 K3
    // 723 -> 1019 us): its loader warps keep ~2 k row pieces in flight against K3's 12 k
    // cp.async (registers bound them; shared memory has no room for staging), see DESIGN.md
    {
        const char *e = dev_env("PA_K3T");
        g->k3t = e && atoi(e) == 1 && g->C == 2 && g->t1 == PA_TMAX && g->N2 <= 8192 &&
                 g->N1 / g->C > 2 * 148u && g->smem1 + 1024 <= kSmemLimit;
    }
    // developer overrides of the thread counts: accepted only as multiples of 32 (k3_epilogue's
    // ballot runs need whole warps, and warps a multiple of C) within [64, PA_TMAX]
    auto threads_ok = [](const char *e) {
        const int v = e ? atoi(e) : 0;
        return v >= 64 && v <= (PA_K2MAX > PA_TMAX ? PA_K2MAX : PA_TMAX) && v % 32 == 0;
    };
    if (const char *e = dev_env("PA_FORCE_T1"); threads_ok(e)) g->t1 = (uint32_t)atoi(e);
    // K2 whose grid (rows x keys) fits one wave of one CTA per SM runs 512 threads even where two
    // CTAs per SM would fit: nothing shares the SM, so the row's latency chain is all there is
    // (C5a single key, 144 rows: 34.3 -> 30.3 us; at C2's 160 rows two CTAs per SM stay faster)
    g->t2one = PA_TMAX;
    if (const char *e = dev_env("PA_FORCE_T2"); threads_ok(e)) g->t2 = g->t2one = (uint32_t)atoi(e);
    // K3's column groups: half of K1's when K1's tile allows one CTA per SM and the half tile
    // two -- a second CTA's loads overlap the first one's stages, worth more than the longer
    // 16-byte row pieces (C4: K3 721 -> 630 us; K1 itself measured slower at C = 1, 778 -> 919
    // us, so it keeps C).  Needs the row-major K2 -> K3 array (lr = 0; wcol is C-specific).
    // Developer override PA_K3_HALF=0.
    {
        // K1's last stage stores straight to global from C = 2 up (32-byte row pieces; same-box
        // C4 2481 -> 2459 us, C5c 336.9 -> 333.8, C5d 1030 -> 1026); developer override
        const char *e = dev_env("PA_K1_GOUT_MINC");
        g->k1gout = e ? (uint32_t)atoi(e) : 2u;
    }
    // K2: L2 prefetch of the CTA's own spectrum row at its start, under the forward stages, when
    // one CTA runs per SM (C4 2453 -> 2421 us, C5d -0.7%; at two CTAs per SM it measured slower,
    // C3 187 -> 193 us).  Developer override PA_PFS=0/1
    {
        const char *e = dev_env("PA_PFS");
        g->pfs = e ? (uint32_t)atoi(e) : g->t2 == PA_TMAX ? 1u : 0u;
    }
    // K1P (persistent K1, finished tiles written behind through TMEM, k1p_fwd_columns): one CTA of
    // 512 threads per SM, a multi-wave grid, column groups of C >= 2 (at C = 1 its 16-byte drain
    // stores are partial-sector writes nothing merges: a 12288 x 12288 plan's K1 took 6.37 ms
    // against 2.48 ms for the plain K1), a shape-specialised plan ending in radix 16 whose
    // last-stage outputs fit the 512 TMEM columns (<= 2 butterflies per thread), and K0's bit
    // streams (not the C = 16 direct gather).  Developer override PA_K1P=0.
    g->k1p_kmax = 0;
    g->smem1p = g->smem1 + g->kbw * 4;
    {
        const char *e = dev_env("PA_K1P");
        const char *et = dev_env("PA_K1P_T");  // developer override of K1P's threads (multiple of 128)
        const int tv = et ? atoi(et) : 0;
        g->k1p_t = tv >= 256 && tv <= PA_TMAX && tv % 128 == 0 ? (uint32_t)tv : PA_TMAX;
        // two CTAs per SM (256 threads, 256 TMEM columns each) when the tiles are small enough --
        // developer opt-in PA_K1P2=1 while it is measured
        const char *e2 = dev_env("PA_K1P2");
        const bool two = e2 && atoi(e2) == 1 && g->t1 == PA_TMAX / 2 && 2 * (g->smem1p + 64) <= kSmemLimit;
        if (two) g->k1p_t = PA_TMAX / 2;
        g->k1p_tcols = two ? 256u : 512u;
        // outputs per drain piece (developer override PA_K1P_PIECE = 2 / 4 / 8)
        const char *ep = dev_env("PA_K1P_PIECE");
        const int pv = ep ? atoi(ep) : 2;
        g->k1p_piece = pv == 4 || pv == 8 ? (uint32_t)pv : 2u;
        const uint32_t nbl = g->f2.S ? (g->f2.st[g->f2.S - 1].nb << g->logC) : 0;
        const uint32_t kmax = (nbl + g->k1p_t - 1) / g->k1p_t;
        if ((!e || atoi(e) != 0) && g->k13 && g->f2.S >= 3 && g->f2.st[g->f2.S - 1].R == 16 &&
            (g->t1 == PA_TMAX || two) && g->C >= 2 && g->C < 16 && kmax >= 1 &&
            (g->k1p_t / 128) * kmax * 64 <= g->k1p_tcols && g->smem1p + 64 <= kSmemLimit &&
            g->N1 / g->C >= 2 * 148u * (two ? 2u : 1u))
            g->k1p_kmax = kmax;
    }
    g->C3 = g->C;
    {
        const char *e = dev_env("PA_K3_HALF");
        if ((!e || atoi(e) != 0) && g->lr == 0 && !g->k3t && g->C >= 2 && 2 * g->smem1 > kSmemLimit &&
            2 * smem_k13(g->N2, g->C / 2, g->f2) <= kSmemLimit)
            g->C3 = g->C / 2;
    }
    g->logC3 = 0;
    while ((1u << g->logC3) < g->C3) ++g->logC3;
    // K3's staged tile in parts (see k3_inv_columns); the part boundaries must fall on
    // butterflies of the first inverse stage (16-row groups): N2 a multiple of 16 * parts
    {
        // measured (round 2): C4 K3 587 (1 part) / 592 (2) / 620 us (4), C5d 207.5 / 217 / 228 us --
        // the per-part barriers cost more than the overlap gains (two CTAs per SM already overlap
        // one tile's load with the other's stages); off by default, developer override PA_K3_PARTS
        const char *e = dev_env("PA_K3_PARTS");
        const int pv = e ? atoi(e) : 1;
        g->k3parts = pv >= 1 && pv <= 4 && g->N2 % (16u * (uint32_t)pv) == 0 ? (uint32_t)pv : 1u;
    }
    g->tile3 = tile_bytes((uint64_t)g->N2 * g->C3) / 16;
    g->smem3 = smem_k13(g->N2, g->C3, g->f2);
    g->t3 = g->C3 == g->C ? g->t1 : 2 * g->smem3 <= kSmemLimit ? PA_TMAX / 2 : PA_TMAX;
    return PA_OK;
}

// K3 runs on its own column groups (C3): the same geometry with K1's group fields replaced
static Geometry k3_geometry(const Geometry &g)
{
    Geometry r = g;
    r.C = g.C3;
    r.logC = g.logC3;
    r.t1 = g.t3;
    r.tile1 = g.tile3;
    r.smem1 = g.smem3;
    return r;
}

static size_t ntables(const Geometry &g)
{
    return 64 + g.f1.nhi + g.f1.ntw + 64 + g.f2.nhi + g.f2.ntw + 64 + g.f2.nhi + (size_t)g.N2 * (64 + g.f1.nhi) +
           g.ntb;
}
static size_t kb_bytes(const Geometry &g) { return (size_t)(g.N1 / g.C) * g.kbw * 4; }

// Persistent block: spec [M] | tables | rev2 [N2] | resid.  Work block: buf [cap][M] |
// kb [cap][...].  Both 256-byte carved, so pa_workspace_size can add them up exactly.
size_t ra_persist_bytes(const Geometry &g)
{
    return al256(g.M * sizeof(double2)) + al256(ntables(g) * sizeof(double2)) + al256(g.N2 * 4u) + al256(8);
}
// work block: buf [cap][M] | kb [cap][...] | buf2 [cap][M] (only with the row-block layout)
size_t ra_work_bytes(const Geometry &g, uint32_t cap)
{
    const size_t b = al256((size_t)cap * g.M * sizeof(double2));
    return b + al256((size_t)cap * kb_bytes(g)) + (g.lr ? b : 0);
}

static void carve_work(RouteA &a, char *blk, uint32_t cap)
{
    const size_t b = al256((size_t)cap * a.g.M * sizeof(double2));
    a.wblk = blk;
    a.buf = reinterpret_cast<double2 *>(blk);
    a.kb = reinterpret_cast<uint32_t *>(blk + b);
    a.buf2 = a.g.lr ? reinterpret_cast<double2 *>(blk + b + al256((size_t)cap * kb_bytes(a.g))) : a.buf;
    a.cap = cap;
    ++a.wgen;
}

// K1 reads the key itself (no K0) when its column groups are at least `min C` wide:
// C = 16 (2-byte runs) saves K0 on the small transforms (C2 38.9 -> 37.9 us cold)
static bool k1_direct(const Geometry &g)
{
    static const uint32_t cmin = [] {
        const char *e = dev_env("PA_K1_DIRECT_MINC");  // developer override (0 = never)
        return e ? (uint32_t)atoi(e) : 16u;  // C = 8 measured slower (C3 K1 66 -> 80 us)
    }();
    return cmin && g.C >= cmin;
}

pa_status ra_create(pa_ctx *h, const uint32_t *seed, cudaStream_t s)
{
    char err[256];
    Geometry &g = h->a.g;
    pa_status st = ra_plan(h->n, h->m, &g, err, sizeof err, h->max_len, h->has_force ? &h->force : nullptr);
    if (st != PA_OK) {
        set_error("%s", err);
        return st;
    }
    RouteA &a = h->a;
    RouteTables &T = a.T;
    char *pb = nullptr, *wb = nullptr;
    // fixed work-buffer capacity for workspace handles and for the column blocks of a split
    // handle (they share block 0's buffers, which therefore must never be reallocated)
    const uint32_t cap = (h->arena || h->parent) && h->batch_opt ? h->batch_opt : 1;
    if ((st = dev_alloc(h, (void **)&pb, ra_persist_bytes(g), "route (a) spectrum + tables"))) return st;
    a.pblk = pb;
    if (h->share_w && ra_work_bytes(g, cap) <= h->share_w_bytes) {
        // a later column block of a split handle: blocks run one after another in stream
        // order, so they share the first block's work buffers
        carve_work(a, h->share_w, cap);
        a.shared_w = true;
    } else {
        if ((st = dev_alloc(h, (void **)&wb, ra_work_bytes(g, cap), "route (a) work buffers"))) return st;
        carve_work(a, wb, cap);
    }
    a.spec = reinterpret_cast<double2 *>(pb);
    pb += al256(g.M * sizeof(double2));
    a.tables = reinterpret_cast<double2 *>(pb);
    pb += al256(ntables(g) * sizeof(double2));
    T.rev2 = reinterpret_cast<uint32_t *>(pb);
    pb += al256(g.N2 * 4u);
    a.resid = reinterpret_cast<unsigned long long *>(pb);
    double2 *p = a.tables;
    T.W1lo = p; p += 64;
    T.W1hi = p; p += g.f1.nhi + g.f1.ntw;  // stage tables follow hi[] (one contiguous copy)
    T.W2lo = p; p += 64;
    T.W2hi = p; p += g.f2.nhi + g.f2.ntw;
    T.thlo = p; p += 64;
    T.thhi = p; p += g.f2.nhi;
    T.rho = p; p += (size_t)g.N2 * (64 + g.f1.nhi);
    T.tb = g.ntb ? p : nullptr; p += g.ntb;

    cudaError_t e;
    if ((e = cudaMemsetAsync(a.resid, 0, sizeof(unsigned long long), s)) != cudaSuccess)
        return cuda_fail(e, "route (a) residual reset");
    uint64_t tot = std::max<uint64_t>(std::max<uint64_t>(g.N1, g.N2), 64);
    k_tables<<<(unsigned)std::min<uint64_t>((tot + 255) / 256, 4096), 256, 0, s>>>(g, T);
    k_rho_tables<<<g.N2, 128, 0, s>>>(g, T);
    k_stage_tables<<<4, 256, 0, s>>>(g.f1, T.W1hi);
    k_stage_tables<<<4, 256, 0, s>>>(g.f2, T.W2hi);
    if (g.ntb) k_bits_table<<<1, 256, 0, s>>>(g.f2.st[0].R, T.tb);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "route (a) table launch");
    h->kernels_per_hash = k1_direct(g) ? 3 : 4;
    return ra_seed(h, seed, s);
}

// Seed spectrum: K0 + K1 + forward half of K2 on the seed, scaled by 1/M.  Uses the
// hash work buffers as scratch (stream-ordered with the hashes).
template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args);

// K2's threads for a grid of `count` keys x N2 rows (Geometry::t2one)
static uint32_t k2_threads(const Geometry &g, uint32_t count)
{
    return (uint64_t)g.N2 * count <= 148u ? g.t2one : g.t2;
}

// The seed half of the path for `count` seeds (a0, create time or a fresh seed): K0 -> K1 (K1P
// where the hash uses it) -> K2 forward half, spectrum / M of seed k at spec + k spec_stride.
static void ra_seed_transform(pa_ctx *h, const uint32_t *seeds, uint64_t seed_stride, uint32_t count,
                              double2 *spec, uint64_t spec_stride, cudaStream_t s, double2 *k1_out = nullptr)
{
    // k1_out: stop after K1, its output for seed k at k1_out + k M (the fresh-seed K2's input)
    RouteA &a = h->a;
    const Geometry &g = a.g;
    const dim3 g0((g.N1 + k0_cols(g) - 1) / k0_cols(g), (g.N2 + k0_rows(g) - 1) / k0_rows(g), count);
    launch_pdl(k0_bits_transpose, g0, dim3(256), 0, s, seeds, h->off, h->L, a.kb, g, seed_stride);
    if (g.k1p_kmax) {
        const uint32_t tiles = (g.N1 / g.C) * count;
        const uint32_t slots = g.k1p_tcols == 256 ? 2 * 148 : 148;
        launch_pdl(kK13[g.k13].k1p, dim3(tiles < slots ? tiles : slots), dim3(g.k1p_t), g.smem1p, s,
                   (const uint32_t *)a.kb, k1_out ? k1_out : a.buf, g, a.T, (uint32_t *)nullptr, (uint64_t)0,
                   (uint64_t)0, count);
    } else {
        launch_pdl(kK13[g.k13].k1, dim3(g.N1 / g.C, count), g.t1, g.smem1, s, (const uint32_t *)a.kb,
                   k1_out ? k1_out : a.buf, g, a.T, (uint32_t *)nullptr, (uint64_t)0, (uint64_t)0,
                   (const uint32_t *)nullptr, (uint64_t)0, (uint64_t)0);
    }
    if (k1_out) return;
    if (g.k2shape)
        launch_pdl(kK2[g.k2shape].seed, dim3(count, g.N2), k2_threads(g, count), g.smem2, s, a.buf, a.buf, spec, g,
                   a.T, spec_stride);
    else
        launch_pdl(k2_rows, dim3(count, g.N2), k2_threads(g, count), g.smem2, s, a.buf, a.buf, spec, g, a.T, 1,
                   1.0 / (double)g.M, spec_stride);
}

pa_status ra_seed(pa_ctx *h, const uint32_t *seed, cudaStream_t s)
{
    RouteA &a = h->a;
    cudaError_t e;
    // the attribute is per device (a process may drive several): set once per device
    static std::atomic<uint64_t> attr_done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = dev < 64 ? 1ull << dev : 0;
    if (bit && (attr_done.load() & bit)) goto launch;
    for (const K13 &f : kK13)
        if ((e = cudaFuncSetAttribute(f.k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLimit)) !=
                cudaSuccess ||
            (e = cudaFuncSetAttribute(f.k1p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLimit - 64)) !=
                cudaSuccess ||
            (e = cudaFuncSetAttribute(f.k3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLimit)) !=
                cudaSuccess)
            return cuda_fail(e, "route (a) cudaFuncSetAttribute");
    if (
        (e = cudaFuncSetAttribute(k2_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kSmemLimit)) != cudaSuccess ||

        (e = cudaFuncSetAttribute(k3t_inv_columns, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kSmemLimit - 1024)) != cudaSuccess)  // K3T has static smem too
        return cuda_fail(e, "route (a) cudaFuncSetAttribute");
    for (const K2Shape &f : kK2)
        if (f.fn && ((e = cudaFuncSetAttribute(f.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemLimit)) !=
                         cudaSuccess ||
                     (e = cudaFuncSetAttribute(f.seed, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)kSmemLimit)) != cudaSuccess ||
                     (e = cudaFuncSetAttribute(f.fresh, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)kSmemLimit)) != cudaSuccess))
            return cuda_fail(e, "route (a) cudaFuncSetAttribute");
    attr_done.fetch_or(bit);
launch:
    ra_seed_transform(h, seed, 0, 1, a.spec, 0, s);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "route (a) seed transform launches");
    return PA_OK;
}

template <typename... KArgs, typename... Args>
static cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// Work buffers for `count` keys in flight (grown on demand, kept for the next call).
// A caller workspace is never grown: pa_hash_batch chunks by its capacity.
static pa_status ra_reserve(pa_ctx *h, uint32_t count, cudaStream_t s)
{
    RouteA &a = h->a;
    if (count <= a.cap) return PA_OK;
    if (h->arena || h->parent) {
        set_error("route (a): %u keys in flight exceed the workspace's %u (pa_options.batch_keys)", count,
                  a.cap);
        return PA_ERR_NOMEM;
    }
    char *nb = nullptr;
    const size_t bytes = ra_work_bytes(a.g, count);
    cudaError_t e = cudaMalloc(&nb, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        set_error("route (a): cannot allocate work buffers for %u keys (%llu bytes): %s", count,
                  (unsigned long long)bytes, cudaGetErrorString(e));
        return PA_ERR_NOMEM;
    }
    // the old buffers may still be in use by work enqueued on s: freed once s passes this point
    h->ws_bytes += bytes - ra_work_bytes(a.g, a.cap);
    defer_free(h, a.wblk, s);
    carve_work(a, nb, count);
    return PA_OK;
}

uint32_t ra_batch_keys(const pa_ctx *h)
{
    if (h->arena || h->parent) return h->a.cap;  // fixed-size (workspace or shared) buffers
    if (h->batch_opt) return h->batch_opt;
    // keys per launch: as many as 4 GiB of work buffers hold, up to 64 -- more keys per launch
    // overlap more (measured: C5a 53 -> 59 Gbit/s from 5 to 64 keys, C5c 50.9 -> 52.9 at 14+)
    const Geometry &g = h->a.g;
    const double per_key = (double)ra_work_bytes(g, 1);
    const uint32_t by_mem = (uint32_t)std::max(1.0, std::floor(4.0 * (1u << 30) / per_key));
    return std::min<uint32_t>(64, by_mem);
}

pa_status ra_hash_batch(pa_ctx *h, const uint32_t *keys, uint64_t key_stride, uint32_t *outs,
                        uint64_t out_stride, uint32_t count, uint64_t zero_words, cudaStream_t s,
                        const double2 *spec, uint64_t spec_stride, bool fresh)
{
    // fresh: `spec` holds the seeds' K1 output (k2_rows_t<..., kFresh>), not spectra
    pa_status st = ra_reserve(h, count, s);
    if (st != PA_OK) return st;
    RouteA &a = h->a;
    const Geometry &g = a.g;
    const dim3 g0((g.N1 + k0_cols(g) - 1) / k0_cols(g), (g.N2 + k0_rows(g) - 1) / k0_rows(g), count);
    const bool direct = k1_direct(g);
    if (!direct) {
        prof_begin(h, 4, s);
        launch_pdl(k0_bits_transpose, g0, dim3(256), 0, s, keys, (uint64_t)0, h->n, a.kb, g, key_stride);
        prof_end(h, s);
    }
    prof_begin(h, 0, s);
    if (g.k1p_kmax && !direct) {
        const uint32_t tiles = (g.N1 / g.C) * count;
        const uint32_t slots = g.k1p_tcols == 256 ? 2 * 148 : 148;
        launch_pdl(kK13[g.k13].k1p, dim3(tiles < slots ? tiles : slots), dim3(g.k1p_t), g.smem1p, s,
                   (const uint32_t *)a.kb, a.buf, g, a.T, outs, zero_words, out_stride, count);
    } else {
        launch_pdl(kK13[g.k13].k1, dim3(g.N1 / g.C, count), g.t1, g.smem1, s, a.kb, a.buf, g, a.T, outs, zero_words,
                   out_stride, direct ? keys : (const uint32_t *)nullptr, key_stride, h->n);
    }
    prof_end(h, s);
    prof_begin(h, 1, s);
    {
        const dim3 g2(count, g.N2);
        const double2 *sp = spec ? spec : a.spec;  // fresh seeds: one spectrum per key
        const uint64_t ss = spec ? spec_stride : 0;
        if (fresh) {
            Geometry gf = g;  // the last key's spectrum row also lands in the handle's spectrum
            gf.fout = a.spec;
            gf.fkey = count - 1;
            launch_pdl(kK2[g.k2shape].fresh, g2, k2_threads(g, count), g.smem2 + 16, s, a.buf, a.buf2,
                       const_cast<double2 *>(sp), gf, a.T, ss);
        }
        else if (g.k2shape)
            launch_pdl(kK2[g.k2shape].fn, g2, k2_threads(g, count), g.smem2, s, a.buf, a.buf2, const_cast<double2 *>(sp), g, a.T, ss);
        else
            launch_pdl(k2_rows, g2, k2_threads(g, count), g.smem2, s, a.buf, a.buf2, const_cast<double2 *>(sp), g, a.T, 0, 1.0, ss);
    }
    prof_end(h, s);
    prof_begin(h, 2, s);
    if (g.k3t) {
        const uint32_t tiles = (g.N1 / g.C) * count;
        launch_pdl(k3t_inv_columns, dim3(tiles < 148 ? tiles : 148), dim3(PA_TMAX), g.smem1, s, a.buf2, g, a.T,
                   h->n, h->m, outs, a.resid, out_stride, count);
    } else {
        const Geometry g3 = k3_geometry(g);
        launch_pdl(kK13[g.k13].k3, dim3(g3.N1 / g3.C, count), g3.t1, g3.smem1, s, a.buf2, g3, a.T, h->n, h->m, outs,
                   a.resid, out_stride);
    }
    prof_end(h, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "route (a) hash launches");
    return PA_OK;
}

pa_status ra_hash(pa_ctx *h, const uint32_t *key, uint32_t *out, uint64_t zero_words, cudaStream_t s)
{
    return ra_hash_batch(h, key, 0, out, 0, 1, zero_words, s);
}

// Fresh seed per key, batched (pa_hash_fresh_batch): for chunks of the work buffers' capacity,
// the chunk's seeds are transformed as one batch (K0 -> K1 -> K2 mode 1, grid over keys) into
// per-key spectra, then its keys are hashed as one batch against them.  Afterwards the handle's
// own spectrum is the last seed's (one device copy).  PA_ERR_UNSUPPORTED: caller loops instead.
pa_status ra_fresh_batch(pa_ctx *h, const uint32_t *seeds, uint64_t seed_stride, const uint32_t *keys,
                         uint64_t key_stride, uint32_t *outs, uint64_t out_stride, uint32_t count,
                         uint64_t zero_words, cudaStream_t s)
{
    RouteA &a = h->a;
    const Geometry &g = a.g;
    const uint32_t chunk = std::min(count, ra_batch_keys(h));
    const size_t spec_bytes = (size_t)g.M * sizeof(double2);
    if (h->arena || h->parent || chunk < 2 || (size_t)chunk * spec_bytes > (size_t(4) << 30))
        return PA_ERR_UNSUPPORTED;
    pa_status st = ra_reserve(h, chunk, s);
    if (st != PA_OK) return st;
    if (a.fcap < chunk) {
        defer_free(h, a.fspec, s);  // the old spectra may still be read by enqueued hashes
        h->ws_bytes -= (size_t)a.fcap * spec_bytes;
        a.fspec = nullptr;
        a.fcap = 0;
        if ((st = dev_alloc(h, (void **)&a.fspec, (size_t)chunk * spec_bytes, "fresh-seed spectra")) != PA_OK)
            return st;
        a.fcap = chunk;
    }
    for (uint32_t k0 = 0; k0 < count; k0 += chunk) {
        const uint32_t c = std::min(chunk, count - k0);
        // the seed's forward half inside the hash's K2 (spectra in TMEM, never in HBM) where it
        // fits; that K2 also writes the chunk's last spectrum into the handle's (every chunk: the
        // last one's stays)
        const bool fused = g.k2fresh && k2f_fits(g, k2_threads(g, c));
        ra_seed_transform(h, seeds + k0 * seed_stride, seed_stride, c, a.fspec, g.M, s, fused ? a.fspec : nullptr);
        if ((st = ra_hash_batch(h, keys + k0 * key_stride, key_stride, outs + k0 * out_stride, out_stride, c,
                                zero_words, s, a.fspec, g.M, fused)) != PA_OK)
            return st;
        if (!fused && k0 + c == count) {
            cudaError_t e = cudaMemcpyAsync(a.spec, a.fspec + (size_t)(c - 1) * g.M, spec_bytes,
                                            cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) return cuda_fail(e, "fresh-seed spectrum copy");
        }
    }
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? PA_OK : cuda_fail(e, "fresh-seed batch launches");
}

#ifdef PA_TIMING
extern "C" int pa_debug_k2_clocks(unsigned long long *out)
{
    return (int)cudaMemcpyFromSymbol(out, g_k2_clk, sizeof(g_k2_clk));
}
extern "C" int pa_debug_trace(unsigned long long *out)
{
    return (int)cudaMemcpyFromSymbol(out, g_trace, sizeof(g_trace));
}
#endif

void ra_destroy(pa_ctx *h)
{
    RouteA &a = h->a;
    dev_free(h, a.pblk);
    if (!a.shared_w) dev_free(h, a.wblk);
    dev_free(h, a.fspec);
    a = RouteA{};
}

}  // namespace pa

namespace pa {
// The cost model's distinct candidate plans for (n, m), cheapest first (measured planning).
bool ra_plan_specialised(const Geometry &g)
{
    FftPlan p1, p2, p2a;
    if (!make_plan(g.N1, &p1) || !make_plan(g.N2, &p2)) return false;
    return k2_shape(p1) && (k13_shape(p2) || (make_plan(g.N2, &p2a, 16, true) && k13_shape(p2a)));
}

int ra_plan_candidates(uint64_t n, uint64_t m, uint64_t max_len, PlanChoice *out, int max)
{
    Geometry g;
    char err[256];
    g_ncand = 0;
    g_cand_on = true;
    ra_plan(n, m, &g, err, sizeof err, max_len);
    g_cand_on = false;
    std::sort(g_cand, g_cand + g_ncand, [](const PlanCand &a, const PlanCand &b) { return a.cost < b.cost; });
    int k = 0;
    for (int i = 0; i < g_ncand && k < max; ++i) {
        bool dup = false;
        for (int j = 0; j < k; ++j)
            dup |= out[j].N1 == g_cand[i].N1 && out[j].N2 == g_cand[i].N2 && out[j].C == g_cand[i].C;
        if (!dup) {
            out[k].N1 = g_cand[i].N1;
            out[k].N2 = g_cand[i].N2;
            out[k].C = g_cand[i].C;
            ++k;
        }
    }
    return k;
}
}  // namespace pa

#ifdef PA_DEV
// Developer build only: the cost model's candidates for (n, m), cheapest first (cost in
// seconds, N1, N2, C), for plan-calibration sweeps (tools/dev/plan_calib.py).
extern "C" int pa_dev_plan_candidates(uint64_t n, uint64_t m, double *cost, uint32_t *n1, uint32_t *n2, uint32_t *c,
                                      int max)
{
    using namespace pa;
    Geometry g;
    char err[256];
    g_ncand = 0;
    g_cand_on = true;
    ra_plan(n, m, &g, err, sizeof err, 0);
    g_cand_on = false;
    std::sort(g_cand, g_cand + g_ncand, [](const PlanCand &a, const PlanCand &b) { return a.cost < b.cost; });
    const int k = g_ncand < max ? g_ncand : max;
    for (int i = 0; i < k; ++i) {
        cost[i] = g_cand[i].cost;
        n1[i] = g_cand[i].N1;
        n2[i] = g_cand[i].N2;
        c[i] = g_cand[i].C;
    }
    return k;
}
// the same candidates with the cost model's features, 13 doubles each:
// cost, N1, N2, C, thr13, lat13, thr2, lat2, spec13, spec2, k1p, occ13, occ2
extern "C" int pa_dev_plan_features(uint64_t n, uint64_t m, double *out, int max)
{
    using namespace pa;
    Geometry g;
    char err[256];
    g_ncand = 0;
    g_cand_on = true;
    ra_plan(n, m, &g, err, sizeof err, 0);
    g_cand_on = false;
    std::sort(g_cand, g_cand + g_ncand, [](const PlanCand &a, const PlanCand &b) { return a.cost < b.cost; });
    const int k = g_ncand < max ? g_ncand : max;
    for (int i = 0; i < k; ++i) {
        double *o = out + 13 * i;
        o[0] = g_cand[i].cost;
        o[1] = g_cand[i].N1;
        o[2] = g_cand[i].N2;
        o[3] = g_cand[i].C;
        for (int j = 0; j < 9; ++j) o[4 + j] = g_cand[i].f[j];
    }
    return k;
}
#endif
