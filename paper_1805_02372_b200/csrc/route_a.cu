// route_a.cu -- route (a): exact integer convolution by an FP64 transform.
//
// The paper recasts r = uT as a polynomial product (Sec. 3 Steps 1-3,
// P:128-136): zero-pad, FFT both, multiply, IFFT, take the window
// [n-1, n+m-1) (one-based "nth to (n+k-1)th") and reduce mod 2.  Here:
//
//  * Length (reading R4): a wrap-free window needs only N >= n+m-1 real points
//    (not the paper's 2n+l-2), and the NEGACYCLIC product mod X^N + 1 is as good
//    as the cyclic one (wrapped terms land below n-1).  A real negacyclic
//    product of length N = 2M is a complex cyclic product of length M of the
//    "right-angle" packed, twisted sequence
//        z[u] = (x[u] + i x[u+M]) * zeta^u,   zeta = exp(i pi / N),  u < M,
//    so every transform is a plain complex DFT of length M (no real-to-complex
//    post-pass), 16 bytes per 2 real points.
//  * Four-step split M = N1 * N2, u = a + N1 b (a < N1 contiguous), frequency
//    k = N2 k_a + k_b:
//        K1  strided pass: per column a, DIF over b (N2 points) of the twisted
//            bits, then twiddle tau(a, k_b) = zeta^a * omega_M^{a k_b}; writes the
//            [N2][N1] work array (row = DIF output position p, k_b = rev2[p]).
//        K2  row pass: per row, DIF over a (N1 points, natural -> digit-reversed
//            order), pointwise * seed spectrum (stored in the same order, scaled
//            by 1/M), DIT inverse (digit-reversed -> natural).  In place.
//        K3  strided pass: * conj tau, DIT inverse over k_b -> natural b, untwist
//            by conj(theta_b) = zeta^{-N1 b}, keep t in [n-1, n+m-1): Re part is
//            c[u], Im part is c[u+M]; rint, &1, set the output bit.  Records
//            max |v - rint(v)| (the FP64 error tripwire, PA_ERR_PRECISION).
//  * The seed goes through K1 and K2's forward half once at create (spectrum
//    cached: the seed is bound at pa_create, BASELINE.json north_star (1)).
//  * Shared memory holds C columns x N2 (K1/K3) or one N1 row (K2) of complex
//    doubles, in-place mixed-radix (2,3,4,5,7,8) butterflies, padded index
//    e + e/16 so strided butterfly accesses stay bank-conflict free.
#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <vector>

#include "bits.cuh"
#include "pa_internal.h"

namespace pa {
namespace {

constexpr uint32_t kSmemLimit = 232448;  // 227 KB opt-in dynamic shared memory per CTA

__device__ __forceinline__ uint32_t pidx(uint32_t e) { return e + (e >> 4); }

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
// a * b
__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b)
{
    return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
// a * (-i) and a * (+i)
__device__ __forceinline__ double2 mul_mi(double2 a) { return make_double2(a.y, -a.x); }
__device__ __forceinline__ double2 mul_pi(double2 a) { return make_double2(-a.y, a.x); }

// ---- small DFTs in registers: X_k = sum_r v_r w^{rk}, w = exp(-+2 pi i / R)
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
        // o_k *= w8^k  (w8 = exp(-+ i pi / 4))
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

// cos/sin(2 pi t / R), t = 1..R-1, for odd R (values to 20 significant digits)
template <int R> struct Trig;
template <> struct Trig<3> {
    __device__ static constexpr double c(int t) { return -0.5; }
    __device__ static constexpr double s(int t) { return t == 1 ? 0.86602540378443864676 : -0.86602540378443864676; }
};
template <> struct Trig<5> {
    __device__ static constexpr double c(int t)
    {
        return (t == 1 || t == 4) ? 0.30901699437494742410 : -0.80901699437494742410;
    }
    __device__ static constexpr double s(int t)
    {
        return t == 1 ? 0.95105651629515357212
               : t == 2 ? 0.58778525229247312917
               : t == 3 ? -0.58778525229247312917
                        : -0.95105651629515357212;
    }
};
template <> struct Trig<7> {
    __device__ static constexpr double c(int t)
    {
        return (t == 1 || t == 6) ? 0.62348980185873353053
               : (t == 2 || t == 5) ? -0.22252093395631440429
                                    : -0.90096886790241912624;
    }
    __device__ static constexpr double s(int t)
    {
        return t == 1 ? 0.78183148246802980871
               : t == 2 ? 0.97492791218182360702
               : t == 3 ? 0.43388373911755812048
               : t == 4 ? -0.43388373911755812048
               : t == 5 ? -0.97492791218182360702
                        : -0.78183148246802980871;
    }
};

// odd R: pair r with R-r.  X_k = v0 + sum_r (v_r + v_{R-r}) cos(2 pi rk/R)
//                                   -+ i sum_r (v_r - v_{R-r}) sin(2 pi rk/R)
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
            // forward: X_k = re - i*im, X_{R-k} = re + i*im
            double2 minus = make_double2(re.x + im.y, re.y - im.x);
            double2 plus = make_double2(re.x - im.y, re.y + im.x);
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

// One in-place stage on a batch of C (power of two) interleaved sequences of
// length Lt in padded shared memory (element t of sequence c at t*C + c).
// Span L = R * Ls.  DIF (forward): DFT_R then twiddle omega_L^{jk};
// DIT (inverse): conj twiddle then inverse DFT_R.  W[e] = omega_Lt^e.
template <int R, bool INV>
__device__ __forceinline__ void stage(double2 *__restrict__ sm, uint32_t Lt, uint32_t logC,
                                      uint32_t L, const double2 *__restrict__ W)
{
    const uint32_t Ls = L / R;
    const uint32_t G = Lt / L;
    const uint32_t C = 1u << logC;
    const uint32_t nb = (Lt / R) << logC;
    for (uint32_t q = threadIdx.x; q < nb; q += blockDim.x) {
        const uint32_t c = q & (C - 1);
        const uint32_t t = q >> logC;
        const uint32_t j = t % Ls, g = t / Ls;
        const uint32_t base = g * L + j;
        double2 v[R];
#pragma unroll
        for (int r = 0; r < R; ++r) v[r] = sm[pidx(((base + r * Ls) << logC) + c)];
        if (!INV) {
            Dft<R, false>::run(v);
            if (j) {
#pragma unroll
                for (int k = 1; k < R; ++k) v[k] = cmul(v[k], __ldg(W + j * k * G));
            }
        } else {
            if (j) {
#pragma unroll
                for (int k = 1; k < R; ++k) v[k] = cmulc(v[k], __ldg(W + j * k * G));
            }
            Dft<R, true>::run(v);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) sm[pidx(((base + r * Ls) << logC) + c)] = v[r];
    }
}

template <bool INV>
__device__ __forceinline__ void stage_dispatch(int R, double2 *sm, uint32_t Lt, uint32_t logC,
                                               uint32_t L, const double2 *W)
{
    switch (R) {
    case 2: stage<2, INV>(sm, Lt, logC, L, W); break;
    case 3: stage<3, INV>(sm, Lt, logC, L, W); break;
    case 4: stage<4, INV>(sm, Lt, logC, L, W); break;
    case 5: stage<5, INV>(sm, Lt, logC, L, W); break;
    case 7: stage<7, INV>(sm, Lt, logC, L, W); break;
    default: stage<8, INV>(sm, Lt, logC, L, W); break;
    }
}

// Forward DIF: natural order in, digit-reversed out.
__device__ void fft_dif(double2 *sm, uint32_t Lt, uint32_t logC, const RadixPlan &P,
                        const double2 *W)
{
    uint32_t L = Lt;
    for (int i = 0; i < P.S; ++i) {
        stage_dispatch<false>(P.R[i], sm, Lt, logC, L, W);
        L /= (uint32_t)P.R[i];
        __syncthreads();
    }
}

// Inverse DIT (unscaled): digit-reversed in, natural order out.
__device__ void ifft_dit(double2 *sm, uint32_t Lt, uint32_t logC, const RadixPlan &P,
                         const double2 *W)
{
    uint32_t L = 1;
    for (int i = P.S - 1; i >= 0; --i) {
        L *= (uint32_t)P.R[i];
        stage_dispatch<true>(P.R[i], sm, Lt, logC, L, W);
        __syncthreads();
    }
}

__device__ __forceinline__ double2 tau(const Geometry &g, const double2 *__restrict__ lo,
                                       const double2 *__restrict__ hi, uint64_t a, uint64_t kb)
{
    // E = a * (1 - 4 kb) mod 4M
    int64_t e = (int64_t)a * (1 - 4 * (int64_t)kb);
    int64_t M4 = (int64_t)g.M4;
    e %= M4;
    if (e < 0) e += M4;
    return cmul(__ldg(hi + e / g.taus), __ldg(lo + e % g.taus));
}

// ------------------------------------------------------------------ tables
__global__ void k_tables(Geometry g, double2 *W1, double2 *W2, double2 *theta, double2 *tlo,
                         double2 *thi, int *rev2, uint64_t nhi)
{
    uint64_t tot = max(max((uint64_t)g.N1, (uint64_t)g.N2), max((uint64_t)g.taus, nhi));
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < tot;
         e += (uint64_t)gridDim.x * blockDim.x) {
        double s, c;
        if (e < g.N1) {
            sincospi((double)(2 * e) / (double)g.N1, &s, &c);
            W1[e] = make_double2(c, -s);
        }
        if (e < g.N2) {
            sincospi((double)(2 * e) / (double)g.N2, &s, &c);
            W2[e] = make_double2(c, -s);
            sincospi((double)e / (double)(2 * (uint64_t)g.N2), &s, &c);
            theta[e] = make_double2(c, s);
            // DIF output position e -> frequency index
            uint32_t rem = (uint32_t)e, L = g.N2, mult = 1, k = 0;
            for (int i = 0; i < g.p2.S; ++i) {
                uint32_t Ls = L / (uint32_t)g.p2.R[i];
                k += (rem / Ls) * mult;
                rem %= Ls;
                mult *= (uint32_t)g.p2.R[i];
                L = Ls;
            }
            rev2[e] = (int)k;
        }
        if (e < g.taus) {
            sincospi((double)e / (double)(2 * g.M), &s, &c);
            tlo[e] = make_double2(c, s);
        }
        if (e < nhi) {
            sincospi((double)(e * g.taus) / (double)(2 * g.M), &s, &c);
            thi[e] = make_double2(c, s);
        }
    }
}

// ------------------------------------------------------------------ K1
// bits: the real sequence (key or seed) = bits [off, off+nbits) of `w`,
// zero padded to N = 2M.  Writes buf[p][a] for a in this CTA's C columns.
__global__ void k1_fwd_columns(const uint32_t *__restrict__ w, uint64_t off, uint64_t nbits,
                               double2 *__restrict__ buf, Geometry g,
                               const double2 *__restrict__ W2, const double2 *__restrict__ theta,
                               const double2 *__restrict__ tlo, const double2 *__restrict__ thi,
                               const int *__restrict__ rev2, uint32_t *__restrict__ zero_out,
                               uint64_t zero_words)
{
    extern __shared__ double2 sm[];
    const uint32_t C = g.C, logC = __ffs(C) - 1;
    const uint64_t a0 = (uint64_t)blockIdx.x * C;
    const int64_t lo = (int64_t)off, hi = (int64_t)(off + nbits);

    if (zero_out) {  // the output bits of this hash are OR-ed in by K3
        for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < zero_words;
             i += (uint64_t)gridDim.x * blockDim.x)
            zero_out[i] = 0u;
    }
    // load: z(b, c) = (x[a + N1 b] + i x[a + N1 b + M]) * theta_b
    for (uint32_t b = threadIdx.x; b < g.N2; b += blockDim.x) {
        int64_t P = (int64_t)(a0 + (uint64_t)g.N1 * b) + lo;
        uint32_t re = bits32(w, P, lo, hi);
        uint32_t im = bits32(w, P + (int64_t)g.M, lo, hi);
        double2 th = __ldg(theta + b);
        for (uint32_t c = 0; c < C; ++c) {
            double xr = (double)((re >> c) & 1u), xi = (double)((im >> c) & 1u);
            // (xr + i xi)(th.x + i th.y)
            sm[pidx((b << logC) + c)] = make_double2(xr * th.x - xi * th.y, xr * th.y + xi * th.x);
        }
    }
    __syncthreads();
    fft_dif(sm, g.N2, logC, g.p2, W2);
    // twiddle and store rows p (k_b = rev2[p])
    const uint32_t tot = g.N2 << logC;
    for (uint32_t e = threadIdx.x; e < tot; e += blockDim.x) {
        uint32_t p = e >> logC, c = e & (C - 1);
        uint64_t a = a0 + c;
        double2 v = cmul(sm[pidx(e)], tau(g, tlo, thi, a, (uint64_t)__ldg(rev2 + p)));
        buf[(uint64_t)p * g.N1 + a] = v;
    }
}

// ------------------------------------------------------------------ K2
// mode 0 (hash): DIF, * spec, DIT, store back in place.
// mode 1 (create): DIF, * scale, store to spec.
__global__ void k2_rows(double2 *__restrict__ buf, const double2 *__restrict__ spec_in,
                        double2 *__restrict__ spec_out, Geometry g,
                        const double2 *__restrict__ W1, int mode, double scale)
{
    extern __shared__ double2 sm[];
    const uint32_t N1 = g.N1;
    for (uint32_t row = blockIdx.x; row < g.N2; row += gridDim.x) {
        double2 *rp = buf + (uint64_t)row * N1;
        for (uint32_t e = threadIdx.x; e < N1; e += blockDim.x) sm[pidx(e)] = rp[e];
        __syncthreads();
        fft_dif(sm, N1, 0, g.p1, W1);
        if (mode == 1) {
            double2 *sp = spec_out + (uint64_t)row * N1;
            for (uint32_t e = threadIdx.x; e < N1; e += blockDim.x) {
                double2 v = sm[pidx(e)];
                sp[e] = make_double2(v.x * scale, v.y * scale);
            }
            __syncthreads();
            continue;
        }
        const double2 *sp = spec_in + (uint64_t)row * N1;
        for (uint32_t e = threadIdx.x; e < N1; e += blockDim.x)
            sm[pidx(e)] = cmul(sm[pidx(e)], __ldg(sp + e));
        __syncthreads();
        ifft_dit(sm, N1, 0, g.p1, W1);
        for (uint32_t e = threadIdx.x; e < N1; e += blockDim.x) rp[e] = sm[pidx(e)];
        __syncthreads();
    }
}

// ------------------------------------------------------------------ K3
__global__ void k3_inv_columns(const double2 *__restrict__ buf, Geometry g,
                               const double2 *__restrict__ W2, const double2 *__restrict__ theta,
                               const double2 *__restrict__ tlo, const double2 *__restrict__ thi,
                               const int *__restrict__ rev2, uint64_t n, uint64_t m,
                               uint32_t *__restrict__ out, unsigned long long *__restrict__ resid)
{
    extern __shared__ double2 sm[];
    const uint32_t C = g.C, logC = __ffs(C) - 1;
    const uint64_t a0 = (uint64_t)blockIdx.x * C;
    const uint32_t tot = g.N2 << logC;
    for (uint32_t e = threadIdx.x; e < tot; e += blockDim.x) {
        uint32_t p = e >> logC, c = e & (C - 1);
        uint64_t a = a0 + c;
        double2 v = buf[(uint64_t)p * g.N1 + a];
        sm[pidx(e)] = cmulc(v, tau(g, tlo, thi, a, (uint64_t)__ldg(rev2 + p)));
    }
    __syncthreads();
    ifft_dit(sm, g.N2, logC, g.p2, W2);
    const uint64_t t0 = n - 1, t1 = n + m - 1;  // output window [t0, t1)
    double rmax = 0.0;
    for (uint32_t e = threadIdx.x; e < tot; e += blockDim.x) {
        uint32_t b = e >> logC, c = e & (C - 1);
        uint64_t u = a0 + c + (uint64_t)g.N1 * b;
        double2 wv = cmulc(sm[pidx(e)], __ldg(theta + b));
        uint64_t tr = u, ti = u + g.M;
        if (tr >= t0 && tr < t1) {
            double r = rint(wv.x);
            rmax = fmax(rmax, fabs(wv.x - r));
            if (((long long)r) & 1) {
                uint64_t i = tr - t0;
                atomicOr(out + (i >> 5), 1u << (i & 31));
            }
        }
        if (ti >= t0 && ti < t1) {
            double r = rint(wv.y);
            rmax = fmax(rmax, fabs(wv.y - r));
            if (((long long)r) & 1) {
                uint64_t i = ti - t0;
                atomicOr(out + (i >> 5), 1u << (i & 31));
            }
        }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xFFFFFFFFu, rmax, d));
    if ((threadIdx.x & 31) == 0 && rmax > 0.0)
        atomicMax(resid, (unsigned long long)__double_as_longlong(rmax));
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

bool radix_plan(uint32_t L, RadixPlan *P)
{
    int e2 = 0, e3 = 0, e5 = 0, e7 = 0;
    while (L % 2 == 0) { L /= 2; ++e2; }
    while (L % 3 == 0) { L /= 3; ++e3; }
    while (L % 5 == 0) { L /= 5; ++e5; }
    while (L % 7 == 0) { L /= 7; ++e7; }
    if (L != 1) return false;
    int S = 0;
    auto push = [&](int r) { if (S < kMaxStages) P->R[S++] = r; };
    while (e2 >= 3) { push(8); e2 -= 3; }
    if (e2 == 2) push(4);
    if (e2 == 1) push(2);
    for (int i = 0; i < e5; ++i) push(5);
    for (int i = 0; i < e3; ++i) push(3);
    for (int i = 0; i < e7; ++i) push(7);
    P->S = S;
    return S < kMaxStages;
}

uint32_t smem_bytes(uint64_t elems) { return (uint32_t)((elems + (elems >> 4) + 1) * 16); }

}  // namespace

pa_status ra_plan(uint64_t n, uint64_t m, Geometry *g, char *err, size_t errlen)
{
    const uint64_t L = n + m - 1;
    const uint64_t Mmin = (L + 1) / 2;
    const uint32_t N1MAX = 12288, N2MAX = 14000;
    static const std::vector<uint32_t> sm = smooth_numbers(16384);
    double best = 1e300;
    bool found = false;
    for (uint32_t N1 : sm) {
        if (N1 > N1MAX) break;
        if (smem_bytes(N1) > kSmemLimit) break;
        uint64_t need = (Mmin + N1 - 1) / N1;
        auto it = std::lower_bound(sm.begin(), sm.end(), (uint32_t)std::min<uint64_t>(need, 1u << 30));
        if (it == sm.end() || *it > N2MAX || need > N2MAX) continue;
        uint32_t N2 = *it;
        uint32_t C = 0;
        for (uint32_t c = 16; c >= 1; c >>= 1)
            if (N1 % c == 0 && smem_bytes((uint64_t)N2 * c) <= kSmemLimit) { C = c; break; }
        if (!C) continue;
        uint64_t M = (uint64_t)N1 * N2;
        double pen = C >= 8 ? 0.0 : C == 4 ? 0.02 : C == 2 ? 0.06 : 0.25;
        if (N1 / C < 148 && M > 100000) pen += 0.05;  // strided passes underfill the GPU
        if (N2 < 16 && M > 100000) pen += 0.05;       // row pass underfills
        double cost = (double)M * (1.0 + pen);
        if (cost < best) {
            best = cost;
            found = true;
            g->M = M;
            g->N1 = N1;
            g->N2 = N2;
            g->C = C;
        }
    }
    if (!found) {
        snprintf(err, errlen,
                 "route (a): n+m-1 = %llu needs a complex transform of length >= %llu, beyond the "
                 "two-pass plan's %u x %u limit",
                 (unsigned long long)L, (unsigned long long)Mmin, N1MAX, N2MAX);
        return PA_ERR_UNSUPPORTED;
    }
    radix_plan(g->N1, &g->p1);
    radix_plan(g->N2, &g->p2);
    g->M4 = 4 * g->M;
    uint32_t B = 1;
    while ((uint64_t)B * B < g->M4) B <<= 1;
    g->taus = B;
    g->t1 = 256;
    uint32_t t2 = 64;
    while (t2 < 512 && t2 * 8 < g->N1) t2 <<= 1;
    g->t2 = t2;
    g->smem1 = smem_bytes((uint64_t)g->N2 * g->C);
    g->smem2 = smem_bytes(g->N1);
    return PA_OK;
}

static pa_status alloc(void **p, size_t bytes, pa_ctx *h, const char *what)
{
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) {
        *p = nullptr;
        set_error("route (a): cudaMalloc(%s, %llu bytes) failed: %s", what,
                  (unsigned long long)bytes, cudaGetErrorString(e));
        return PA_ERR_NOMEM;
    }
    h->ws_bytes += bytes;
    return PA_OK;
}

pa_status ra_create(pa_ctx *h, const uint32_t *seed, cudaStream_t s)
{
    char err[256];
    Geometry &g = h->a.g;
    pa_status st = ra_plan(h->n, h->m, &g, err, sizeof err);
    if (st != PA_OK) {
        set_error("%s", err);
        return st;
    }
    RouteA &a = h->a;
    uint64_t nhi = (g.M4 + g.taus - 1) / g.taus;
    if ((st = alloc((void **)&a.buf, g.M * sizeof(double2), h, "buf"))) return st;
    if ((st = alloc((void **)&a.spec, g.M * sizeof(double2), h, "spec"))) return st;
    if ((st = alloc((void **)&a.W1, g.N1 * sizeof(double2), h, "W1"))) return st;
    if ((st = alloc((void **)&a.W2, g.N2 * sizeof(double2), h, "W2"))) return st;
    if ((st = alloc((void **)&a.theta, g.N2 * sizeof(double2), h, "theta"))) return st;
    if ((st = alloc((void **)&a.tau_lo, g.taus * sizeof(double2), h, "tau_lo"))) return st;
    if ((st = alloc((void **)&a.tau_hi, nhi * sizeof(double2), h, "tau_hi"))) return st;
    if ((st = alloc((void **)&a.rev2, g.N2 * sizeof(int), h, "rev2"))) return st;
    if ((st = alloc((void **)&a.resid, sizeof(unsigned long long), h, "resid"))) return st;

    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k1_fwd_columns, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kSmemLimit)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(k2_rows, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kSmemLimit)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(k3_inv_columns, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)kSmemLimit)) != cudaSuccess)
        return cuda_fail(e, "route (a) cudaFuncSetAttribute");
    if ((e = cudaMemsetAsync(a.resid, 0, sizeof(unsigned long long), s)) != cudaSuccess)
        return cuda_fail(e, "route (a) residual reset");

    uint64_t tot = std::max<uint64_t>(std::max<uint64_t>(g.N1, g.N2), std::max<uint64_t>(g.taus, nhi));
    k_tables<<<(unsigned)std::min<uint64_t>((tot + 255) / 256, 4096), 256, 0, s>>>(
        g, a.W1, a.W2, a.theta, a.tau_lo, a.tau_hi, a.rev2, nhi);
    // seed spectrum: K1 + forward half of K2, scaled by 1/M
    k1_fwd_columns<<<g.N1 / g.C, g.t1, g.smem1, s>>>(seed, h->off, h->L, a.buf, g, a.W2, a.theta,
                                                     a.tau_lo, a.tau_hi, a.rev2, nullptr, 0);
    k2_rows<<<g.N2, g.t2, g.smem2, s>>>(a.buf, nullptr, a.spec, g, a.W1, 1, 1.0 / (double)g.M);
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "route (a) create launches");
    h->kernels_per_hash = 3;
    return PA_OK;
}

pa_status ra_hash(pa_ctx *h, const uint32_t *key, uint32_t *out, uint64_t zero_words,
                  cudaStream_t s)
{
    RouteA &a = h->a;
    const Geometry &g = a.g;
    k1_fwd_columns<<<g.N1 / g.C, g.t1, g.smem1, s>>>(key, 0, h->n, a.buf, g, a.W2, a.theta,
                                                     a.tau_lo, a.tau_hi, a.rev2, out, zero_words);
    k2_rows<<<g.N2, g.t2, g.smem2, s>>>(a.buf, a.spec, nullptr, g, a.W1, 0, 1.0);
    k3_inv_columns<<<g.N1 / g.C, g.t1, g.smem1, s>>>(a.buf, g, a.W2, a.theta, a.tau_lo, a.tau_hi,
                                                     a.rev2, h->n, h->m, out, a.resid);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "route (a) hash launches");
    return PA_OK;
}

void ra_destroy(pa_ctx *h)
{
    RouteA &a = h->a;
    void *ptrs[] = {a.buf, a.spec, a.W1, a.W2, a.theta, a.tau_lo, a.tau_hi, a.rev2, a.resid};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    a = RouteA{};
}

}  // namespace pa
