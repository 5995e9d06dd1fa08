// fft_core.cuh -- FP64 complex mixed-radix (2,3,4,5,7,8,16) FFT building blocks for
// libpa route (a).  In-place stages on a batch of C interleaved sequences held in
// padded shared memory; the first and last stage of a pass may load from / store
// to anything (bits, global memory, the parity epilogue) through functors.
#pragma once
#include <stdint.h>

namespace pa {

constexpr int kMaxStages = 24;

// One radix-R stage of a length-Lt transform: span L = R * Ls, twiddle stride
// G = Lt / L (omega_L^{jk} = omega_Lt^{jkG}), nb = Lt / R butterflies per sequence.
struct StageDesc {
    uint32_t R, L, Ls, G, nb;
    uint32_t toff;   // G > 1: this stage's own table of omega_L^j at whi + toff (see butterfly)
    uint64_t magic;  // ceil(2^40 / Ls): t / Ls == (t * magic) >> 40 for t < 2^24
};

struct FftPlan {
    int S;              // number of stages (0 when Lt == 1)
    uint32_t Lt;        // transform length
    uint32_t nhi;       // two-level twiddle table: omega_Lt^e = hi[e >> 6] * lo[e & 63]
    uint32_t ntw;       // entries of the per-stage tables that follow hi[] (stages with G > 1)
    StageDesc st[kMaxStages];
};

__device__ __forceinline__ uint32_t pidx(uint32_t e) { return e + (e >> 4); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b)  // a * conj(b)
{
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }
__device__ __forceinline__ double2 mul_pi(double2 a) { return make_double2(-a.y, a.x); }

// ---- small DFTs: X_k = sum_r v_r w^{rk}, w = exp(-2 pi i / R) (forward) or conj (INV)
template <int R, bool INV> struct Dft;

template <bool INV> struct Dft<2, INV> {
    __device__ __forceinline__ static void run(double2 *v)
    {
        double2 a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    }
};

template <bool INV> struct Dft<4, INV> {
    __device__ __forceinline__ static void run(double2 *v)
    {
        double2 t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
        double2 t2 = cadd(v[1], v[3]), d = csub(v[1], v[3]);
        double2 t3 = INV ? mul_pi(d) : mul_mi(d);
        v[0] = cadd(t0, t2);
        v[2] = csub(t0, t2);
        v[1] = cadd(t1, t3);
        v[3] = csub(t1, t3);
    }
};

template <bool INV> struct Dft<8, INV> {
    __device__ __forceinline__ static void run(double2 *v)
    {
        const double h = 0.70710678118654752440;  // sqrt(1/2)
        double2 e[4] = {v[0], v[2], v[4], v[6]};
        double2 o[4] = {v[1], v[3], v[5], v[7]};
        Dft<4, INV>::run(e);
        Dft<4, INV>::run(o);
        double2 o1 = INV ? make_double2(h * (o[1].x - o[1].y), h * (o[1].x + o[1].y))
                         : make_double2(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
        double2 o2 = INV ? mul_pi(o[2]) : mul_mi(o[2]);
        double2 o3 = INV ? make_double2(-h * (o[3].x + o[3].y), h * (o[3].x - o[3].y))
                         : make_double2(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
        v[0] = cadd(e[0], o[0]);
        v[4] = csub(e[0], o[0]);
        v[1] = cadd(e[1], o1);
        v[5] = csub(e[1], o1);
        v[2] = cadd(e[2], o2);
        v[6] = csub(e[2], o2);
        v[3] = cadd(e[3], o3);
        v[7] = csub(e[3], o3);
    }
};

// radix 16 as 4 x 4: n = 4 n2 + n1, k = k1 + 4 k2,
// X[k1 + 4 k2] = sum_n1 w4^{n1 k2} w16^{n1 k1} sum_n2 w4^{n2 k1} v[4 n2 + n1]
template <bool INV> struct Dft<16, INV> {
    __device__ __forceinline__ static double2 w16(int e)
    {
        const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, h = 0.70710678118654752440;
        double2 w;
        switch (e) {  // exp(-2 pi i e / 16), e in {1,2,3,4,6,9}
        case 1: w = make_double2(c1, -s1); break;
        case 2: w = make_double2(h, -h); break;
        case 3: w = make_double2(s1, -c1); break;
        case 4: w = make_double2(0.0, -1.0); break;
        case 6: w = make_double2(-h, -h); break;
        default: w = make_double2(-c1, s1); break;  // 9
        }
        if (INV) w.y = -w.y;
        return w;
    }
    __device__ __forceinline__ static void run(double2 *v)
    {
        double2 y[4][4];
#pragma unroll
        for (int n1 = 0; n1 < 4; ++n1) {
            double2 q[4] = {v[n1], v[4 + n1], v[8 + n1], v[12 + n1]};
            Dft<4, INV>::run(q);
#pragma unroll
            for (int k1 = 0; k1 < 4; ++k1) y[n1][k1] = q[k1];
        }
#pragma unroll
        for (int n1 = 1; n1 < 4; ++n1)
#pragma unroll
            for (int k1 = 1; k1 < 4; ++k1) {
                const int e = n1 * k1;
                if (e == 4) y[n1][k1] = INV ? mul_pi(y[n1][k1]) : mul_mi(y[n1][k1]);
                else y[n1][k1] = cmul(y[n1][k1], w16(e));
            }
#pragma unroll
        for (int k1 = 0; k1 < 4; ++k1) {
            double2 q[4] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1]};
            Dft<4, INV>::run(q);
#pragma unroll
            for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = q[k2];
        }
    }
};

// cos/sin(2 pi t / R), t = 1..R-1, odd R (20 significant digits)
template <int R> struct Trig;
template <> struct Trig<3> {
    __device__ static constexpr double c(int) { return -0.5; }
    __device__ static constexpr double s(int t) { return t == 1 ? 0.86602540378443864676 : -0.86602540378443864676; }
};
template <> struct Trig<5> {
    __device__ static constexpr double c(int t) { return (t == 1 || t == 4) ? 0.30901699437494742410 : -0.80901699437494742410; }
    __device__ static constexpr double s(int t)
    {
        return t == 1 ? 0.95105651629515357212 : t == 2 ? 0.58778525229247312917
               : t == 3 ? -0.58778525229247312917 : -0.95105651629515357212;
    }
};
template <> struct Trig<7> {
    __device__ static constexpr double c(int t)
    {
        return (t == 1 || t == 6) ? 0.62348980185873353053
               : (t == 2 || t == 5) ? -0.22252093395631440429 : -0.90096886790241912624;
    }
    __device__ static constexpr double s(int t)
    {
        return t == 1 ? 0.78183148246802980871 : t == 2 ? 0.97492791218182360702
               : t == 3 ? 0.43388373911755812048 : t == 4 ? -0.43388373911755812048
               : t == 5 ? -0.97492791218182360702 : -0.78183148246802980871;
    }
};

// odd R: X_k = v0 + sum_r (v_r + v_{R-r}) cos(2 pi rk/R) -+ i sum_r (v_r - v_{R-r}) sin(2 pi rk/R)
template <int R, bool INV> struct DftOdd {
    __device__ __forceinline__ static void run(double2 *v)
    {
        constexpr int H = (R - 1) / 2;
        double2 sum[H + 1], dif[H + 1];
#pragma unroll
        for (int r = 1; r <= H; ++r) {
            sum[r] = cadd(v[r], v[R - r]);
            dif[r] = csub(v[r], v[R - r]);
        }
        double2 out[R];
        out[0] = v[0];
#pragma unroll
        for (int r = 1; r <= H; ++r) out[0] = cadd(out[0], sum[r]);
#pragma unroll
        for (int k = 1; k <= H; ++k) {
            double2 re = v[0], im = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 1; r <= H; ++r) {
                const int t = (r * k) % R;
                re.x = fma(sum[r].x, Trig<R>::c(t), re.x);
                re.y = fma(sum[r].y, Trig<R>::c(t), re.y);
                im.x = fma(dif[r].x, Trig<R>::s(t), im.x);
                im.y = fma(dif[r].y, Trig<R>::s(t), im.y);
            }
            double2 minus = make_double2(re.x + im.y, re.y - im.x);  // re - i*im
            double2 plus = make_double2(re.x - im.y, re.y + im.x);   // re + i*im
            out[k] = INV ? plus : minus;
            out[R - k] = INV ? minus : plus;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = out[r];
    }
};
template <bool INV> struct Dft<3, INV> : DftOdd<3, INV> {};
template <bool INV> struct Dft<5, INV> : DftOdd<5, INV> {};
template <bool INV> struct Dft<7, INV> : DftOdd<7, INV> {};

// omega_Lt^e from the two-level table (shared memory)
__device__ __forceinline__ double2 twiddle(const double2 *lo, const double2 *hi, uint32_t e)
{
    return cmul(hi[e >> 6], lo[e & 63]);
}

// v[k] *= w1^k (or conj) for k = 1..R-1.  Powers 2..4 from w1, then a running
// B = w1^{4a} and w1^{4a+b} = B * w1^b: the same multiply count as a running
// product, at most ~5 complex multiplies deep (latency, and the DESIGN.md error
// bound), and only six complex temporaries live (registers).
template <int R, bool INV>
__device__ __forceinline__ void apply_twiddles(double2 *v, double2 w1)
{
    double2 p[4];
    p[1] = w1;
    if (R > 2) p[2] = cmul(w1, w1);
    if (R > 3) p[3] = cmul(p[2], w1);
#pragma unroll
    for (int b = 1; b < 4 && b < R; ++b) v[b] = INV ? cmulc(v[b], p[b]) : cmul(v[b], p[b]);
    if (R > 4) {
        const double2 w4 = cmul(p[2], p[2]);
        double2 B = w4;
#pragma unroll
        for (int a = 1; 4 * a < R; ++a) {
            if (a > 1) B = cmul(B, w4);
#pragma unroll
            for (int b = 0; b < 4 && 4 * a + b < R; ++b) {
                const double2 w = b ? cmul(B, p[b]) : B;
                v[4 * a + b] = INV ? cmulc(v[4 * a + b], w) : cmul(v[4 * a + b], w);
            }
        }
    }
}

// omega_L^j of a stage.  G = 1: the plan's two-level table at e = j (consecutive lanes,
// consecutive entries).  G > 1: reading the plan's table at e = jG would stride the
// 64-entry low table by G (bank conflicts: up to 8-way for G = 40), so such a stage has
// its own table indexed by j: lo[j & 63] (* hi[j >> 6] when Ls > 64), both exact
// roundings of exp(-2 pi i e / Lt) computed at create time.
__device__ __forceinline__ double2 stage_twiddle(const StageDesc &sd, uint32_t j, const double2 *wlo,
                                                 const double2 *whi)
{
    if (sd.G == 1) return twiddle(wlo, whi, j);
    const double2 *t = whi + sd.toff;
    return sd.Ls > 64 ? cmul(t[64 + (j >> 6)], t[j & 63]) : t[j];
}

template <int R, bool INV>
__device__ __forceinline__ void butterfly(double2 *v, uint32_t j, const StageDesc &sd, const double2 *wlo,
                                          const double2 *whi)
{
    if (!INV) Dft<R, false>::run(v);
    if (j) apply_twiddles<R, INV>(v, stage_twiddle(sd, j, wlo, whi));
    if (INV) Dft<R, true>::run(v);
}

// Where a stage's inputs come from and its outputs go (K2 fuses its row twist into
// the first forward and the last inverse stage):
//   MODE_PLAIN     smem -> smem
//   MODE_TAU_IN    smem * rho^idx -> smem                   (K2 first forward stage)
//   MODE_TAU_OUT   smem -> conj(rho^idx) * . -> gout[idx]   (K2 last inverse stage)
//   MODE_GCOL      gin[row * ld + c] -> smem               (K3 first inverse stage)
//   MODE_GCOL_OUT  smem -> gout[row * ld + c]              (K1 last forward stage)
enum { MODE_PLAIN = 0, MODE_TAU_IN = 1, MODE_TAU_OUT = 2, MODE_GCOL = 3, MODE_GCOL_OUT = 4 };
struct StageCtx {
    const double2 *rlo = nullptr, *rhi = nullptr;    // rho^e two-level tables (K2 row)
    double2 *gout = nullptr;                         // K2 row in global memory
    const double2 *gin = nullptr;                    // MODE_TAU_IN / MODE_GCOL: global input
    uint32_t ld = 0;                                 // MODE_GCOL(_OUT): row(-block) pitch in elements
    uint32_t nth = 0;                                // threads sharing the stage (0 = blockDim.x)
    uint32_t q0 = 0, q1 = 0;                         // butterfly range [q0, q1) (q1 = 0: all)
    // work-array layout (route_a.cu widx): rows in blocks of 2^lr, column groups of 2^lc
    uint32_t lr = 0, lc = 0;
};

// MODE_GCOL(_OUT): element (row, c) of a column group at gin/gout + gcol_off
__device__ __forceinline__ uint64_t gcol_off(const StageCtx &x, uint32_t row, uint32_t c)
{
    return (uint64_t)(row >> x.lr) * x.ld + ((row & ((1u << x.lr) - 1)) << x.lc) + c;
}
// MODE_TAU_IN / MODE_TAU_OUT: element a of a work-array row at gin/gout + grow_off
__device__ __forceinline__ uint32_t grow_off(const StageCtx &x, uint32_t a)
{
    return ((a >> x.lc) << (x.lc + x.lr)) + (a & ((1u << x.lc) - 1));
}

// K2's row twist on a butterfly's inputs v[r] (element idx0 + r Ls): rho^{idx0 + r Ls} =
// rho^{idx0} * rho^{r Ls}, and when 64 | Ls the second factor is the single entry rhi[r Ls / 64]
// (the same for every lane: a broadcast), so a radix-16 butterfly reads one two-level lookup
// instead of 16 -- the lookups' shared-memory wavefronts, not their FP64 work, are what the pass
// pays for (C5b K2 20.8 -> 19.7 us; at radix 5, C4, it measured neutral to
// 0.2% slower and keeps the per-element lookups).  The factor is a product of three correctly
// rounded entries (Sec. 5).
template <int R>
__device__ __forceinline__ bool twist_factored(uint32_t Ls) { return R >= 16 && (Ls & 63) == 0; }

template <int R>
__device__ __forceinline__ void twist_in(double2 *v, const StageCtx &x, uint32_t idx0, uint32_t Ls)
{
    if (twist_factored<R>(Ls)) {
        const double2 t0 = twiddle(x.rlo, x.rhi, idx0);
        v[0] = cmul(v[0], t0);
#pragma unroll
        for (int r = 1; r < R; ++r) v[r] = cmul(v[r], cmul(t0, x.rhi[(r * Ls) >> 6]));
    } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = cmul(v[r], twiddle(x.rlo, x.rhi, idx0 + r * Ls));
    }
}

// One in-place stage over all butterflies of a batch of 2^logC sequences held
// in padded shared memory (element idx of sequence c at pidx((idx << logC) + c)).
//   DIF (forward): v = DFT_R(v); v_k *= omega_L^{jk}
//   DIT (inverse): v_k *= conj omega_L^{jk}; v = IDFT_R(v)
// Not inlined: one copy per (R, direction, mode) per kernel keeps the code in
// the instruction cache.
template <int R, bool INV, int MODE>
__device__ __forceinline__ void stage_inl(double2 *sm, const StageDesc &sd, uint32_t logC, const double2 *wlo,
                                          const double2 *whi, const StageCtx &x)
{
    const uint32_t nb = sd.nb << logC;
    const uint32_t cm = (1u << logC) - 1;
    const uint32_t stride = sd.Ls << logC;
    const uint32_t nth = x.nth ? x.nth : blockDim.x;
    if constexpr (MODE == MODE_TAU_IN && R <= 8) {
        // K2's first stage from global with several butterflies per thread (10240-point rows):
        // the next butterfly's row loads are issued before this one's arithmetic
        if (x.gin) {
            auto first = [&](uint32_t q) {
                const uint32_t t = q >> logC, g = (uint32_t)(((uint64_t)t * sd.magic) >> 40);
                return g * sd.L + (t - g * sd.Ls);
            };
            double2 nv[R];
            uint32_t q = threadIdx.x;
            if (q < nb) {
                const uint32_t i0 = first(q);
#pragma unroll
                for (int r = 0; r < R; ++r) nv[r] = x.gin[grow_off(x, i0 + r * sd.Ls)];
            }
            for (; q < nb; q += nth) {
                const uint32_t c = q & cm, t = q >> logC;
                const uint32_t g = (uint32_t)(((uint64_t)t * sd.magic) >> 40);
                const uint32_t j = t - g * sd.Ls;
                const uint32_t idx0 = g * sd.L + j;
                const uint32_t base = (idx0 << logC) + c;
                double2 v[R];
#pragma unroll
                for (int r = 0; r < R; ++r) v[r] = nv[r];
                if (q + nth < nb) {
                    const uint32_t i1 = first(q + nth);
#pragma unroll
                    for (int r = 0; r < R; ++r) nv[r] = x.gin[grow_off(x, i1 + r * sd.Ls)];
                }
                twist_in<R>(v, x, idx0, sd.Ls);
                butterfly<R, INV>(v, j, sd, wlo, whi);
#pragma unroll
                for (int r = 0; r < R; ++r) sm[pidx(base + r * stride)] = v[r];
            }
            return;
        }
    }
    const uint32_t qend = x.q1 ? x.q1 : nb;
    for (uint32_t q = x.q0 + threadIdx.x; q < qend; q += nth) {
        const uint32_t c = q & cm, t = q >> logC;
        const uint32_t g = (uint32_t)(((uint64_t)t * sd.magic) >> 40);
        const uint32_t j = t - g * sd.Ls;
        const uint32_t idx0 = g * sd.L + j;
        const uint32_t base = (idx0 << logC) + c;
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (MODE == MODE_TAU_IN && x.gin) v[r] = x.gin[grow_off(x, idx0 + r * sd.Ls)];
            else if (MODE == MODE_GCOL) v[r] = x.gin[gcol_off(x, idx0 + r * sd.Ls, c)];
            else v[r] = sm[pidx(base + r * stride)];
        }
        if (MODE == MODE_TAU_IN) twist_in<R>(v, x, idx0, sd.Ls);
        butterfly<R, INV>(v, j, sd, wlo, whi);
        double2 t0;
        if (MODE == MODE_TAU_OUT && twist_factored<R>(sd.Ls)) t0 = twiddle(x.rlo, x.rhi, idx0);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (MODE == MODE_TAU_OUT) {
                const uint32_t idx = idx0 + r * sd.Ls;
                x.gout[grow_off(x, idx)] =
                    cmulc(v[r], twist_factored<R>(sd.Ls) ? (r ? cmul(t0, x.rhi[(r * sd.Ls) >> 6]) : t0)
                                                         : twiddle(x.rlo, x.rhi, idx));
            } else if (MODE == MODE_GCOL_OUT) {
                x.gout[gcol_off(x, idx0 + r * sd.Ls, c)] = v[r];
            } else {
                sm[pidx(base + r * stride)] = v[r];
            }
        }
    }
}

// The same stage as a call (one copy per kernel for the general kernels' radix switch; the
// shape-specialised kernels may inline stage_inl instead).
template <int R, bool INV, int MODE>
__device__ __noinline__ void stage_smem(double2 *sm, StageDesc sd, uint32_t logC, const double2 *wlo,
                                        const double2 *whi, StageCtx x)
{
    stage_inl<R, INV, MODE>(sm, sd, logC, wlo, whi, x);
}

template <bool INV, int MODE = MODE_PLAIN>
__device__ __forceinline__ void stage_any(double2 *sm, const StageDesc &sd, uint32_t logC, const double2 *wlo,
                                          const double2 *whi, const StageCtx &x = StageCtx{})
{
    switch (sd.R) {
    case 2: stage_smem<2, INV, MODE>(sm, sd, logC, wlo, whi, x); break;
    case 3: stage_smem<3, INV, MODE>(sm, sd, logC, wlo, whi, x); break;
    case 4: stage_smem<4, INV, MODE>(sm, sd, logC, wlo, whi, x); break;
    case 5: stage_smem<5, INV, MODE>(sm, sd, logC, wlo, whi, x); break;
    case 7: stage_smem<7, INV, MODE>(sm, sd, logC, wlo, whi, x); break;
    case 8: stage_smem<8, INV, MODE>(sm, sd, logC, wlo, whi, x); break;
    default: stage_smem<16, INV, MODE>(sm, sd, logC, wlo, whi, x); break;
    }
}

// Stages [i0, i1) of the forward DIF (natural -> digit-reversed), barrier after each.
__device__ __forceinline__ void dif_stages(double2 *sm, const FftPlan &P, int i0, int i1, uint32_t logC,
                                           const double2 *wlo, const double2 *whi)
{
    for (int i = i0; i < i1; ++i) {
        stage_any<false>(sm, P.st[i], logC, wlo, whi);
        __syncthreads();
    }
}

// Stages i1-1 down to i0 of the inverse DIT (digit-reversed -> natural), barrier after each.
__device__ __forceinline__ void dit_stages(double2 *sm, const FftPlan &P, int i0, int i1, uint32_t logC,
                                           const double2 *wlo, const double2 *whi)
{
    for (int i = i1 - 1; i >= i0; --i) {
        stage_any<true>(sm, P.st[i], logC, wlo, whi);
        __syncthreads();
    }
}

}  // namespace pa
