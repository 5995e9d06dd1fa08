"""Secondary full-output reference (SURVEY 8(c) pin P11), test infrastructure only.

y = window [n-1, n+m-1) of the integer convolution x * s, mod 2 (Sec. 3 Step 3,
P:128-136), computed with an FP64 real FFT (scipy/pocketfft) of length N >= n+m-1 (reading R4:
no term wraps into the window).  Each window value is an integer count; the function returns
the largest distance to the nearest integer as its own rounding certificate (it must stay
< 0.5; the tests require < 0.25).  It shares no code with libpa or with oracle/, and is itself
checked against the direct oracle in tests/test_fft_ref.py before the GPU tests use it at sizes
the direct oracle cannot finish (C3, C4, C5c full outputs).
"""
from __future__ import annotations

import os

import numpy as np
import scipy.fft as sfft


def _bits(words: np.ndarray, nbits: int) -> np.ndarray:
    b = np.unpackbits(np.ascontiguousarray(words).view(np.uint8), bitorder="little")[:nbits]
    if b.size < nbits:
        raise ValueError(f"{b.size} bits available, {nbits} required")
    return b


def fft_window(n: int, m: int, seed_words, key_words):
    """-> (y as uint8 0/1 [m], max |c - rint(c)| over the window)."""
    L = n + m - 1
    N = sfft.next_fast_len(L, real=True)
    workers = os.cpu_count() or 1
    X = sfft.rfft(_bits(key_words, n).astype(np.float64), N, workers=workers)
    S = sfft.rfft(_bits(seed_words, L).astype(np.float64), N, workers=workers)
    X *= S
    del S
    c = sfft.irfft(X, N, workers=workers)[n - 1:n + m - 1]
    del X
    r = np.rint(c)
    resid = float(np.max(np.abs(c - r))) if m else 0.0
    return (r.astype(np.int64) & 1).astype(np.uint8), resid
