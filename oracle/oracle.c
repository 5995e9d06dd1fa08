/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU oracle for the one computation on the
 * hot path of arXiv 1805.02372: Toeplitz-hash privacy amplification over
 * GF(2).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this code.  It shares no code, header,
 * table or helper with the CUDA path under paper_1805_02372_b200/.
 *
 * Definition followed (citations are PAPER.md lines, "P:L"):
 *   - Toeplitz matrix, diagonal-constant, 2n-1 (here n+m-1) degrees of
 *     freedom, not necessarily square: Sec. 2.1, Eq. (1).
 *   - r = u T with a uniform seed of length n+l-1: Sec. 2.3 Steps 1-2,
 *     P:88-92 (we write the transpose, y = T x, with T of size m x n).
 *   - Layout (reading R2): T[i][j] = s[i - j + n - 1], i in [0,m)
 *     output rows, j in [0,n) key bits.  This is the layout under which the
 *     paper's Step 3 "results of IFFT from the nth to (n+k-1)th" are
 *     exactly the outputs; the pin tests check that identity independently.
 *
 *   y[i] = XOR_{j=0}^{n-1} ( s[i - j + n - 1] AND x[j] ),   i = 0 .. m-1.
 *
 * Two variants:
 *   oracle_toeplitz_bits   the literal double loop over unpacked 0/1 bytes.
 *   oracle_toeplitz_rows   the same sum, 64 terms at a time, on LSB-first
 *                          packed uint64 words (bit b of the string is bit
 *                          b%64 of word b/64).  With j' = n-1-j and the
 *                          reversed key xr[j'] = x[n-1-j'] the sum reads
 *                          y[i] = XOR_{j'} xr[j'] AND s[i + j'], i.e. a
 *                          64-bit window of s starting at bit i + 64k ANDed
 *                          with word k of xr.  Pinned against the bit
 *                          variant by tests/test_oracle.py.
 * Parity: popcount of the AND/XOR accumulator, mod 2.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Literal definition, one output bit per row, byte-per-bit inputs. */
void oracle_toeplitz_bits(uint64_t n, uint64_t m, const uint8_t *seed,
                          const uint8_t *key, uint8_t *out)
{
    for (uint64_t i = 0; i < m; ++i) {
        uint8_t acc = 0;
        for (uint64_t j = 0; j < n; ++j)
            acc ^= (uint8_t)(seed[i + n - 1 - j] & key[j] & 1u);
        out[i] = acc;
    }
}

/* The literal loop over `count` keys (key c at key + c*n, output at out + c*m),
 * used by the exhaustive brute-force pin. */
void oracle_toeplitz_bits_many(uint64_t n, uint64_t m, const uint8_t *seed,
                               const uint8_t *keys, uint8_t *outs,
                               uint64_t count)
{
    for (uint64_t c = 0; c < count; ++c)
        oracle_toeplitz_bits(n, m, seed, keys + c * n, outs + c * m);
}

static inline uint64_t get_bit(const uint64_t *w, uint64_t b)
{
    return (w[b >> 6] >> (b & 63)) & 1u;
}

/* 64-bit window of the bit string w starting at bit o (w must have one
 * readable word past the window). */
static inline uint64_t window64(const uint64_t *w, uint64_t o)
{
    uint64_t q = o >> 6, r = o & 63;
    if (r == 0)
        return w[q];
    return (w[q] >> r) | (w[q + 1] << (64 - r));
}

/* Word-level oracle on selected rows.
 *   seed_words: ceil((n+m-1)/64) words, key_words: ceil(n/64) words
 *   rows[r] in [0,m) for r < nrows; out[r] receives y[rows[r]] (0/1 byte).
 *   threads <= 0 means "all OpenMP threads".
 * Returns 0, or -1 on allocation failure / bad row index. */
int oracle_toeplitz_rows(uint64_t n, uint64_t m, const uint64_t *seed_words,
                         const uint64_t *key_words, const uint64_t *rows,
                         uint64_t nrows, uint8_t *out, int threads)
{
    uint64_t L = n + m - 1;
    uint64_t kw = (n + 63) / 64;
    uint64_t sw = (L + 63) / 64;
    /* reversed key, zero tail */
    uint64_t *xr = (uint64_t *)calloc(kw, sizeof(uint64_t));
    /* seed copy with two zero words of slack so window64 never reads past */
    uint64_t *s = (uint64_t *)calloc(sw + 2, sizeof(uint64_t));
    if (!xr || !s) {
        free(xr);
        free(s);
        return -1;
    }
    for (uint64_t jp = 0; jp < n; ++jp)
        if (get_bit(key_words, n - 1 - jp))
            xr[jp >> 6] |= (uint64_t)1 << (jp & 63);
    memcpy(s, seed_words, sw * sizeof(uint64_t));
    if (L & 63) /* ignore seed bits beyond L */
        s[sw - 1] &= ((uint64_t)1 << (L & 63)) - 1;
    for (uint64_t r = 0; r < nrows; ++r)
        if (rows[r] >= m) {
            free(xr);
            free(s);
            return -1;
        }
#ifdef _OPENMP
    if (threads > 0)
        omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 64)
#endif
    for (int64_t r = 0; r < (int64_t)nrows; ++r) {
        uint64_t i = rows[r];
        uint64_t acc = 0;
        for (uint64_t k = 0; k < kw; ++k)
            acc ^= xr[k] & window64(s, i + 64 * k);
        out[r] = (uint8_t)(__builtin_popcountll(acc) & 1);
    }
    free(xr);
    free(s);
    return 0;
}

/* Word-level oracle, all rows, packed LSB-first output of ceil(m/64) words
 * (tail bits beyond m written 0). */
int oracle_toeplitz_words(uint64_t n, uint64_t m, const uint64_t *seed_words,
                          const uint64_t *key_words, uint64_t *out_words,
                          int threads)
{
    uint64_t *rows = (uint64_t *)malloc(m * sizeof(uint64_t));
    uint8_t *bits = (uint8_t *)malloc(m);
    if (!rows || !bits) {
        free(rows);
        free(bits);
        return -1;
    }
    for (uint64_t i = 0; i < m; ++i)
        rows[i] = i;
    int rc = oracle_toeplitz_rows(n, m, seed_words, key_words, rows, m, bits,
                                  threads);
    if (rc == 0) {
        memset(out_words, 0, ((m + 63) / 64) * sizeof(uint64_t));
        for (uint64_t i = 0; i < m; ++i)
            if (bits[i])
                out_words[i >> 6] |= (uint64_t)1 << (i & 63);
    }
    free(rows);
    free(bits);
    return rc;
}

int oracle_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
