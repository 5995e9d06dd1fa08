"""CPU oracle for Toeplitz privacy amplification -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_1805_02372_b200``) never imports it, and this package never imports
the product: the two share no code.  The only shared module is ``pa_synth``
(seeded input generation, which holds none of the method's arithmetic).

What it computes (Sec. 2.1 Eq. (1), Sec. 2.3):

    y[i] = XOR_{j=0}^{n-1} s[i - j + n - 1] AND x[j],   i = 0..m-1

with the seed s of n+m-1 bits, the key x of n bits, output y of m bits
(reading R1/R2 for orientation and diagonal layout).  Bit strings
are LSB-first packed (bit b -> word b//64, bit b%64).

Functions
---------
toeplitz_bits(n, m, seed01, key01)        literal double loop (C), 0/1 arrays
toeplitz_bits_many(n, m, seed01, keys01)  same, many keys (exhaustive pin)
toeplitz_rows(n, m, seed_w, key_w, rows)  64-bit word variant, sampled rows
toeplitz_words(n, m, seed_w, key_w)       word variant, full packed output
unpack(words, nbits) / pack(bits)         the oracle's own (numpy) bit packing
eq1_matrix(t01, n, l)                     Eq. (1)'s n x l Toeplitz matrix, literally
eq1_hash(t01, u01, n, l)                  the paper's r = u T over GF(2)
seed_from_eq1(t01, n, m)                  Eq. (1) symbol order -> the diagonal order above

Parity status: every function here is pinned by tests/test_oracle.py against
brute force, hand-worked examples, closed forms, GF(2) polynomial
multiplication and invariants.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2 -fopenmp).  Returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-march=x86-64-v2",
             "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            u64, p = ctypes.c_uint64, ctypes.c_void_p
            lib.oracle_toeplitz_bits.argtypes = [u64, u64, p, p, p]
            lib.oracle_toeplitz_bits.restype = None
            lib.oracle_toeplitz_bits_many.argtypes = [u64, u64, p, p, p, u64]
            lib.oracle_toeplitz_bits_many.restype = None
            lib.oracle_toeplitz_rows.argtypes = [u64, u64, p, p, p, u64, p, ctypes.c_int]
            lib.oracle_toeplitz_rows.restype = ctypes.c_int
            lib.oracle_toeplitz_words.argtypes = [u64, u64, p, p, p, ctypes.c_int]
            lib.oracle_toeplitz_words.restype = ctypes.c_int
            lib.oracle_max_threads.argtypes = []
            lib.oracle_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _check_nm(n: int, m: int) -> None:
    if n < 1 or m < 1:
        raise ValueError(f"n={n}, m={m}: both must be >= 1")


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def unpack(words: np.ndarray, nbits: int) -> np.ndarray:
    """LSB-first packed words (any unsigned dtype) -> uint8 0/1 array."""
    b = np.ascontiguousarray(words).view(np.uint8)
    bits = np.unpackbits(b, bitorder="little")
    if bits.size < nbits:
        raise ValueError(f"{bits.size} bits available, {nbits} requested")
    return bits[:nbits].copy()


def pack(bits: np.ndarray, word_bits: int = 64) -> np.ndarray:
    """uint8 0/1 array -> LSB-first packed uint64 (or uint32) words."""
    bits = np.asarray(bits, dtype=np.uint8)
    nw = (bits.size + word_bits - 1) // word_bits
    padded = np.zeros(nw * word_bits, dtype=np.uint8)
    padded[: bits.size] = bits & 1
    by = np.packbits(padded, bitorder="little")
    return by.view(np.uint64 if word_bits == 64 else np.uint32).copy()


def toeplitz_bits(n: int, m: int, seed01, key01) -> np.ndarray:
    """Literal double loop. seed01: n+m-1 values in {0,1}; key01: n values."""
    _check_nm(n, m)
    s = np.ascontiguousarray(seed01, dtype=np.uint8)
    x = np.ascontiguousarray(key01, dtype=np.uint8)
    if s.size != n + m - 1 or x.size != n:
        raise ValueError(f"seed has {s.size} bits (need {n + m - 1}), key has {x.size} (need {n})")
    out = np.zeros(m, dtype=np.uint8)
    _load().oracle_toeplitz_bits(n, m, _ptr(s), _ptr(x), _ptr(out))
    return out


def toeplitz_bits_many(n: int, m: int, seed01, keys01) -> np.ndarray:
    """keys01: (count, n) 0/1 array -> (count, m) outputs."""
    _check_nm(n, m)
    s = np.ascontiguousarray(seed01, dtype=np.uint8)
    k = np.ascontiguousarray(keys01, dtype=np.uint8)
    if s.size != n + m - 1 or k.ndim != 2 or k.shape[1] != n:
        raise ValueError("bad shapes")
    out = np.zeros((k.shape[0], m), dtype=np.uint8)
    _load().oracle_toeplitz_bits_many(n, m, _ptr(s), _ptr(k), _ptr(out), k.shape[0])
    return out


def _as_u64(words: np.ndarray, nbits: int) -> np.ndarray:
    w = np.ascontiguousarray(words)
    if w.dtype != np.uint64:
        b = w.view(np.uint8)
        need = ((nbits + 63) // 64) * 8
        pad = np.zeros(max(need, b.size + (-b.size) % 8), dtype=np.uint8)
        pad[: b.size] = b
        w = pad.view(np.uint64)
    if w.size * 64 < nbits:
        raise ValueError(f"{w.size * 64} bits available, {nbits} required")
    return w


def toeplitz_rows(n: int, m: int, seed_words, key_words, rows, threads: int = 0) -> np.ndarray:
    """y[rows] (uint8 0/1) by the 64-bit word variant."""
    _check_nm(n, m)
    s = _as_u64(seed_words, n + m - 1)
    x = _as_u64(key_words, n)
    r = np.ascontiguousarray(rows, dtype=np.uint64)
    out = np.zeros(r.size, dtype=np.uint8)
    rc = _load().oracle_toeplitz_rows(n, m, _ptr(s), _ptr(x), _ptr(r), r.size, _ptr(out), threads)
    if rc != 0:
        raise ValueError("oracle_toeplitz_rows failed (row out of range or OOM)")
    return out


def toeplitz_words(n: int, m: int, seed_words, key_words, threads: int = 0) -> np.ndarray:
    """Full output, LSB-first packed into ceil(m/64) uint64 words, tail zero."""
    _check_nm(n, m)
    s = _as_u64(seed_words, n + m - 1)
    x = _as_u64(key_words, n)
    out = np.zeros((m + 63) // 64, dtype=np.uint64)
    rc = _load().oracle_toeplitz_words(n, m, _ptr(s), _ptr(x), _ptr(out), threads)
    if rc != 0:
        raise MemoryError("oracle_toeplitz_words failed")
    return out


# ---------------------------------------------------------------- the paper's Eq. (1) form
def eq1_matrix(t01, n: int, l: int) -> np.ndarray:
    """Eq. (1) written out, generalised to n x l ("the Toeplitz matrix
    is not necessarily square"; T is n x l in Sec. 2.3):

        T[i, j] = t_{i-j}        for i >= j   (lower triangle and diagonal)
        T[i, j] = t_{j-i+n-1}    for j >  i   (upper triangle)

    t01 holds the n+l-1 symbols t_0 .. t_{n+l-2}."""
    t = np.asarray(t01, dtype=np.uint8)
    if t.size != n + l - 1:
        raise ValueError(f"t has {t.size} symbols, Eq. (1) with n = {n}, l = {l} needs {n + l - 1}")
    T = np.zeros((n, l), dtype=np.uint8)
    for i in range(n):
        for j in range(l):
            T[i, j] = t[i - j] if i >= j else t[j - i + n - 1]
    return T


def eq1_hash(t01, u01, n: int, l: int) -> np.ndarray:
    """r = u T over GF(2) (Sec. 2.3 Step 2): u the n-bit corrected key as a row
    vector, T = eq1_matrix(t01, n, l); returns the l bits of r."""
    u = np.asarray(u01, dtype=np.int64)
    if u.size != n:
        raise ValueError(f"u has {u.size} bits, need {n}")
    return ((u @ eq1_matrix(t01, n, l).astype(np.int64)) & 1).astype(np.uint8)


def seed_from_eq1(t01, n: int, m: int) -> np.ndarray:
    """DESIGN.md reading R2: the diagonal-order seed s with y = T x, T[i][j] = s[i-j+n-1],
    equal to Eq. (1)'s r = u T: s[k] = t_{n-1-k} for k < n, s[k] = t_k for n <= k < n+m-1."""
    t = np.asarray(t01, dtype=np.uint8)
    if t.size != n + m - 1:
        raise ValueError(f"t has {t.size} symbols, need {n + m - 1}")
    s = t.copy()
    s[:n] = t[:n][::-1]
    return s
