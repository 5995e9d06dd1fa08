"""Pins for the CPU oracle.  No GPU needed.

Each test fixes the oracle to something other than itself: hand-worked
examples (tests/golden), an independently constructed explicit matrix
(brute force, exhaustive on tiny sizes), GF(2)[t] polynomial multiplication
(the paper's Step 3 window), closed forms, and invariants.
"""
import os

import numpy as np
import pytest

import oracle
import pa_synth as syn


def _bits(s):
    return np.array([int(c) for c in s], dtype=np.uint8)


def _load_golden(golden_dir):
    rows = []
    with open(os.path.join(golden_dir, "hand_examples.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            name, cite, n, m, s, x, y = [t.strip() for t in line.split("|")]
            rows.append((name, cite, int(n), int(m), _bits(s), _bits(x), _bits(y)))
    return rows


def test_golden_hand_examples(golden_dir):
    """P2: hand-worked examples (PAPER Eq. (1))."""
    rows = _load_golden(golden_dir)
    assert len(rows) >= 6
    for name, cite, n, m, s, x, y in rows:
        assert s.size == n + m - 1 and x.size == n and y.size == m, name
        got = oracle.toeplitz_bits(n, m, s, x)
        assert np.array_equal(got, y), (name, cite, got, y)
        got_w = oracle.toeplitz_rows(n, m, oracle.pack(s), oracle.pack(x), np.arange(m))
        assert np.array_equal(got_w, y), (name, cite)


def _explicit_matrix(n, m, s):
    """Build T by the diagonal-constant construction of P:48 (first column and
    first row, then T[i][j] = T[i-1][j-1]); independent of the index formula.
    The first column (key bit 0) is s[n-1 .. n+m-2]; the first row (output 0)
    is s[n-1], s[n-2], ..., s[0]  (reading R2)."""
    T = np.zeros((m, n), dtype=np.uint8)
    for i in range(m):
        T[i, 0] = s[n - 1 + i]
    for j in range(n):
        T[0, j] = s[n - 1 - j]
    for i in range(1, m):
        for j in range(1, n):
            T[i, j] = T[i - 1, j - 1]
    return T


def test_bruteforce_exhaustive_tiny():
    """P1: every seed x every key for n <= 8, m <= min(n, 4)."""
    total = 0
    for n in range(1, 9):
        keys = ((np.arange(1 << n)[:, None] >> np.arange(n)[None, :]) & 1).astype(np.uint8)
        for m in range(1, min(n, 4) + 1):
            L = n + m - 1
            for sv in range(1 << L):
                s = ((sv >> np.arange(L)) & 1).astype(np.uint8)
                T = _explicit_matrix(n, m, s)
                want = (keys.astype(np.int64) @ T.T.astype(np.int64)) & 1
                got = oracle.toeplitz_bits_many(n, m, s, keys)
                assert np.array_equal(got, want), (n, m, sv)
                total += keys.shape[0]
    assert total > 500_000


def _clmul(a: int, b: int) -> int:
    """Carry-less (GF(2)[t]) product of two polynomials held as Python ints."""
    r = 0
    while a:
        low = a & -a
        r ^= b << (low.bit_length() - 1)
        a ^= low
    return r


@pytest.mark.parametrize("n,m", [(1, 1), (5, 3), (64, 64), (65, 7), (127, 33), (300, 299), (1000, 100), (4096, 1024)])
def test_polynomial_window(n, m):
    """The paper's Step 3: the hash is the window [n-1, n+m-1)
    (one-based "nth to (n+k-1)th") of the product x(t)*s(t) reduced mod 2,
    i.e. a GF(2)[t] polynomial product -- computed here with Python integers."""
    sw = syn.random_bits(syn.seed_stream(900 + n), n + m - 1)
    kw = syn.random_bits(syn.key_stream(900 + m, n), n)
    S = int.from_bytes(sw.tobytes(), "little")
    X = int.from_bytes(kw.tobytes(), "little")
    P = _clmul(X, S)
    want = np.array([(P >> (n - 1 + i)) & 1 for i in range(m)], dtype=np.uint8)
    got = oracle.toeplitz_rows(n, m, sw, kw, np.arange(m))
    assert np.array_equal(got, want)
    if n * m <= 1_000_000:
        got_b = oracle.toeplitz_bits(n, m, oracle.unpack(sw, n + m - 1), oracle.unpack(kw, n))
        assert np.array_equal(got_b, want)


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 63, 64, 65, 127, 128, 129, 1000, 4097])
def test_word_variant_matches_literal(n):
    """oracle_toeplitz_rows (64-bit words) == the literal double loop."""
    for m in sorted({1, 31, 64, 65, max(1, n // 10), n}):
        if m > n:
            continue
        sw = syn.random_bits(syn.seed_stream(1000 + n), n + m - 1)
        kw = syn.random_bits(syn.key_stream(1000 + n, m), n)
        lit = oracle.toeplitz_bits(n, m, oracle.unpack(sw, n + m - 1), oracle.unpack(kw, n))
        wrd = oracle.toeplitz_words(n, m, sw, kw)
        assert np.array_equal(oracle.unpack(wrd, m), lit), (n, m)
        # tail bits of the packed output are zero
        assert np.all(oracle.unpack(wrd, wrd.size * 64)[m:] == 0)


def test_ignores_bits_past_lengths():
    n, m = 100, 30
    sw = syn.random_bits(syn.seed_stream(7), n + m - 1)
    kw = syn.random_bits(syn.key_stream(7, 1), n)
    base = oracle.toeplitz_words(n, m, sw, kw)
    sw2, kw2 = sw.copy(), kw.copy()
    sw2[-1] |= np.uint64(0xFFFF_FFFF_FFFF_FFFF) << np.uint64((n + m - 1) % 64)
    kw2[-1] |= np.uint64(0xFFFF_FFFF_FFFF_FFFF) << np.uint64(n % 64)
    assert np.array_equal(oracle.toeplitz_words(n, m, sw2, kw2), base)


def _prefix_xor(bits):
    P = np.zeros(bits.size + 1, dtype=np.uint8)
    P[1:] = np.bitwise_xor.accumulate(bits)
    return P


@pytest.mark.parametrize("n,m", [(1000, 1000), (100_003, 25_000), (262_144, 26_214)])
def test_closed_forms(n, m):
    """P3: all-ones key -> y[i] = P[i+n] ^ P[i] (P = prefix XOR of s);
    all-ones seed -> y[i] = parity(x); unit key e_j -> y = s[n-1-j : n-1-j+m];
    zero key -> 0.  O(n+m) forms, independent of the O(nm) oracle loop."""
    L = n + m - 1
    sw = syn.random_bits(syn.seed_stream(2000 + n), L)
    s = oracle.unpack(sw, L)
    rows = np.unique(np.concatenate([np.arange(min(m, 64)), np.arange(max(0, m - 64), m),
                                     np.random.default_rng(n).integers(0, m, 256)]))
    P = _prefix_xor(s)
    y1 = oracle.toeplitz_rows(n, m, sw, syn.ones_bits(n), rows)
    assert np.array_equal(y1, P[rows + n] ^ P[rows])
    kw = syn.random_bits(syn.key_stream(2000 + n, 0), n)
    par = int(oracle.unpack(kw, n).sum() & 1)
    y2 = oracle.toeplitz_rows(n, m, syn.ones_bits(L), kw, rows)
    assert np.all(y2 == par)
    for j in (0, 1, n // 2, n - 1):
        yj = oracle.toeplitz_rows(n, m, sw, syn.unit_bits(n, j), rows)
        assert np.array_equal(yj, s[n - 1 - j + rows]), j
    assert not oracle.toeplitz_rows(n, m, sw, syn.zero_bits(n), rows).any()


def test_sparse_key_is_xor_of_columns():
    """P4: a key with k set bits hashes to the XOR of k seed windows."""
    n, m = 200_001, 40_000
    L = n + m - 1
    sw = syn.random_bits(syn.seed_stream(3000), L)
    s = oracle.unpack(sw, L)
    kw, pos = syn.sparse_bits(3000, n, 17)
    want = np.zeros(m, dtype=np.uint8)
    for j in pos:
        want ^= s[n - 1 - j: n - 1 - j + m]
    got = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
    assert np.array_equal(got, want)


def test_linearity_and_shift_invariance():
    """P5: T(x ^ x') = Tx ^ Tx'.  P6: with s'[t] = s[t+1] the
    hash shifts by one row, y'[i] = y[i+1] (diagonal-constant)."""
    n, m = 5000, 1234
    L = n + m - 1
    sw = syn.random_bits(syn.seed_stream(4000), L)
    a = syn.random_bits(syn.key_stream(4000, 1), n)
    b = syn.random_bits(syn.key_stream(4000, 2), n)
    ya = oracle.toeplitz_words(n, m, sw, a)
    yb = oracle.toeplitz_words(n, m, sw, b)
    assert np.array_equal(oracle.toeplitz_words(n, m, sw, a ^ b), ya ^ yb)
    s = oracle.unpack(sw, L)
    s_shift = np.concatenate([s[1:], [1]]).astype(np.uint8)
    y_shift = oracle.unpack(oracle.toeplitz_words(n, m, oracle.pack(s_shift), a), m)
    assert np.array_equal(y_shift[:-1], oracle.unpack(ya, m)[1:])


def test_row_and_column_split_identities():
    """P7: a block of output rows [r0, r0+mg) is the hash with the seed window
    s[r0 : r0+mg+n-1]; a block of key bits [c0, c0+ng) contributes the hash
    with seed window s[n-ng-c0 : n-c0+m-1], and the blocks XOR to y
    (the paper's Eq. (4) split and Eq. (7) modulo-2 merge)."""
    n, m = 3001, 777
    L = n + m - 1
    s = oracle.unpack(syn.random_bits(syn.seed_stream(5000), L), L)
    x = oracle.unpack(syn.random_bits(syn.key_stream(5000, 0), n), n)
    y = oracle.toeplitz_bits(n, m, s, x)
    # row split into 3 uneven pieces
    cuts = [0, 100, 500, m]
    parts = [oracle.toeplitz_bits(n, b - a, s[a:a + (b - a) + n - 1], x) for a, b in zip(cuts, cuts[1:])]
    assert np.array_equal(np.concatenate(parts), y)
    # column split into 4 uneven pieces, XOR merge
    cuts = [0, 1, 1000, 2222, n]
    acc = np.zeros(m, dtype=np.uint8)
    for c0, c1 in zip(cuts, cuts[1:]):
        ng = c1 - c0
        off = n - ng - c0
        acc ^= oracle.toeplitz_bits(ng, m, s[off:off + ng + m - 1], x[c0:c1])
    assert np.array_equal(acc, y)


def test_threads_deterministic():
    n, m = 50_000, 5_000
    sw = syn.random_bits(syn.seed_stream(6000), n + m - 1)
    kw = syn.random_bits(syn.key_stream(6000, 0), n)
    assert np.array_equal(oracle.toeplitz_words(n, m, sw, kw, threads=1),
                          oracle.toeplitz_words(n, m, sw, kw, threads=0))


def test_rejects_bad_args():
    with pytest.raises(ValueError):
        oracle.toeplitz_bits(0, 1, [], [])
    with pytest.raises(ValueError):
        oracle.toeplitz_bits(3, 2, [1, 0, 1], [1, 1, 0])
    with pytest.raises(ValueError):
        oracle.toeplitz_rows(10, 5, syn.random_bits(1, 14), syn.random_bits(2, 10), [5])


def test_splitmix64_reference_values():
    """SplitMix64 with state 0: published first outputs (Vigna's splitmix64.c)."""
    w = syn.splitmix64(0, 3)
    assert [int(v) for v in w] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    b = syn.random_bits(123, 100)
    assert b.size == 2 and int(b[1]) >> 36 == 0


# ---------------------------------------------------------------- Eq. (1) form (reading R2)
def test_eq1_matrix_is_the_printed_figure():
    """Eq. (1) as printed, square n x n with symbolic entries t_k = k: first row
    t_0, t_n, t_{n+1}, .., t_{2n-2}; first column t_0 .. t_{n-1}; last row t_{n-1} .. t_1, t_0;
    constant diagonals."""
    n = 6
    T = oracle.eq1_matrix(np.arange(2 * n - 1) % 256, n, n)
    assert list(T[0]) == [0] + list(range(n, 2 * n - 1))
    assert list(T[:, 0]) == list(range(n))
    assert list(T[n - 1]) == list(range(n - 1, -1, -1))
    assert list(T[1, :3]) == [1, 0, n]          # second printed row: t_1 t_0 t_n
    for d in range(-(n - 1), n):
        assert len(set(np.diagonal(T, offset=d))) == 1


def test_eq1_hash_equals_diagonal_layout_after_conversion():
    """The paper's r = u T with Eq. (1) equals this library's y = T x on
    the converted seed, for random t, u and non-square shapes (n x l, l <= n)."""
    rng = np.random.default_rng(1805)
    for n, m in [(1, 1), (2, 1), (3, 2), (5, 5), (8, 3), (17, 9), (40, 13), (64, 64)]:
        for _ in range(5):
            t = rng.integers(0, 2, n + m - 1, dtype=np.uint8)
            u = rng.integers(0, 2, n, dtype=np.uint8)
            r = oracle.eq1_hash(t, u, n, m)
            y = oracle.toeplitz_bits(n, m, oracle.seed_from_eq1(t, n, m), u)
            assert np.array_equal(r, y), (n, m)


def test_seed_from_eq1_is_an_involution_on_the_first_n_bits():
    rng = np.random.default_rng(7)
    t = rng.integers(0, 2, 30, dtype=np.uint8)
    s = oracle.seed_from_eq1(t, 20, 11)
    assert np.array_equal(oracle.seed_from_eq1(s, 20, 11), t)
    assert np.array_equal(s[20:], t[20:])
