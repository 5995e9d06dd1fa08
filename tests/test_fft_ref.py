"""Pin the secondary FFT reference (tests/fft_ref.py) to the direct oracle, so
that the GPU tests may use it for full outputs at C3/C4/C5c."""
import numpy as np
import pytest

import oracle
import pa_synth as syn
from fft_ref import fft_window


@pytest.mark.parametrize("n,m", [(1, 1), (2, 1), (33, 7), (1000, 1000), (4097, 1023), (65_537, 6_553),
                                 (200_003, 50_000)])
def test_fft_window_equals_direct_oracle(n, m):
    sw = syn.random_bits(syn.seed_stream(90), n + m - 1)
    kw = syn.random_bits(syn.key_stream(90, n), n)
    y, resid = fft_window(n, m, sw, kw)
    assert resid < 0.25
    assert np.array_equal(y, oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m))


def test_fft_window_worst_case_all_ones():
    """All-ones key and seed: every window value is n (closed form y[i] = n mod 2)."""
    n, m = 300_001, 30_000
    ones = syn.ones_bits(n + m - 1)
    y, resid = fft_window(n, m, ones, syn.ones_bits(n))
    assert resid < 1e-6
    assert np.all(y == (n & 1))
