"""pa_blocked_plan: the block shape of the length-compatible split (Eq. (4)-(7),
P:103-141) -- host-only planning, run without a GPU."""
import numpy as np
import pytest

import paper_1805_02372_b200 as pa


def work(n, m, nb, mb):
    return -(-m // mb) * -(-((n + 31) // 32 * 32) // nb) * (nb + mb)


def round1_shape(n, m, lim):
    """Round 1's rule: one row block when m fits half the limit, else square blocks of lim / 2."""
    mr = (m + 31) // 32 * 32
    mb = mr if (mr + 31 <= lim // 2 or (lim > mr and mr + 64 <= lim - mr)) else (lim // 2) // 32 * 32
    nb = min((lim + 1 - mb) // 32 * 32, (n + 31) // 32 * 32)
    return nb, mb


@pytest.mark.parametrize("seed", range(6))
def test_block_shape_invariants(seed):
    rng = np.random.default_rng(seed)
    for _ in range(200):
        n = int(rng.integers(64, 10**9))
        m = int(rng.integers(1, n + 1)) if rng.random() < 0.5 else max(1, n // int(rng.integers(2, 200)))
        lim = int(rng.integers(64, 2 * (n + m)))
        p = pa.pa_blocked_plan(n, m, lim)
        nb, mb = p["nb"], p["mb"]
        assert nb % 32 == 0 and mb % 32 == 0 and nb >= 32 and mb >= 32
        assert nb + mb - 1 <= lim
        assert p["blocks"] == -(-m // mb) * -(-n // nb)
        # never more transform work than round 1's shape for the same limit
        nb1, mb1 = round1_shape(n, m, lim)
        if nb1 >= 32 and mb1 >= 32 and nb1 + mb1 - 1 <= lim:
            assert work(n, m, nb, mb) <= work(n, m, nb1, mb1)


def test_one_row_block_when_it_pays():
    """m = 10^8, limit 1.6 * 10^8: one row block (17 blocks), not square 8 * 10^7 blocks (26)."""
    p = pa.pa_blocked_plan(10**9, 10**8, 160_000_000)
    assert p["mb"] >= 10**8 and p["blocks"] == 17


def test_default_limit_is_one_plan_and_budget_monotone():
    n, m = 10**9, 10**8
    p0 = pa.pa_blocked_plan(n, m)
    assert p0["nb"] + p0["mb"] - 1 <= 2 * 13312 * 13312  # one route-(a) plan per block
    prev = 0
    for gib in (64, 16, 6, 3, 1):
        p = pa.pa_blocked_plan(n, m, 0, gib << 30)
        assert p["blocks"] >= prev  # a smaller budget never gives fewer (longer) blocks
        prev = p["blocks"]
    with pytest.raises(pa.PaError) as e:
        pa.pa_blocked_plan(n, m, 0, 1 << 20)  # 1 MiB cannot hold a block handle
    assert e.value.status == pa.PA_ERR_NOMEM


def test_invalid_arguments():
    for args in ((100, 0), (100, 101)):
        with pytest.raises(pa.PaError) as e:
            pa.pa_blocked_plan(*args)
        assert e.value.status == pa.PA_ERR_INVALID_ARG
    with pytest.raises(pa.PaError):
        pa.pa_blocked_plan(1000, 100, 32)
