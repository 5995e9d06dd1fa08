"""SPEC acceptance criteria run against the GPU path.

SPEC's criteria bind its CPU program; here they are used as test ideas for this library's
hot path: the GPU hash through the C ABI against the CPU oracle.  Criterion 5
(finite-size math) is tests/test_finite_size.py, 7 (1 Gbit under 2 GiB) is in
tests/test_parity_gpu.py, 8 (the two-party session) is out of scope.
"""
import numpy as np
import pytest

import oracle
import pa_synth as syn

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU hosts
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1805_02372_b200 as pa  # noqa: E402

DEV = torch.device("cuda:0")


def dev(words):
    w = np.ascontiguousarray(words).view(np.int32)
    w = np.concatenate([w, np.zeros((-w.size) % 4 + 4, np.int32)])
    return torch.from_numpy(w.copy()).to(DEV)


def bits(t, m):
    return oracle.unpack(t.cpu().numpy().view(np.uint32), m)


def hash_under_plan(n, m, seed_t, key_t, plan, rng):
    """One of the library's plans: route (a) / (b), an Eq. (4) column split, a 2-D blocking."""
    if plan == "blocked":
        lim = int(rng.integers(64, n + m))
        out = torch.zeros(pa.words32(m) + 4, dtype=torch.int32, device=DEV)
        pa.pa_hash_blocked(n, m, seed_t.data_ptr(), key_t.data_ptr(), out.data_ptr(), lim, 0)
        return out
    opts = {"transform": dict(route="transform"), "bitpacked": dict(route="bitpacked"),
            # caps leave room above m for a 128-bit block and a smooth transform length
            "split": dict(route="transform",
                          max_transform_len=int(rng.integers(m + m // 10 + 1024, n + 2 * m + 2048)))}[plan]
    with pa.Hasher(n, m, seed_t, **opts) as h:
        return h.hash(key_t)


def test_criterion1_oracle_equivalence_random_plans():
    """1000 random trials, n in [1, 2^16], l in [1, n], random seeds and a random plan each:
    bit-exact against the oracle."""
    rng = np.random.default_rng(511)
    plans = ["transform", "bitpacked", "split", "blocked"]
    for trial in range(1000):
        n = int(rng.integers(1, (1 << 16) + 1))
        m = int(rng.integers(1, n + 1))
        plan = plans[trial % 4]
        if (plan == "split" and n + m < 300) or (plan == "blocked" and n + m < 80):
            plan = "transform"
        sw = syn.random_bits(syn.seed_stream(5000 + trial), n + m - 1)
        kw = syn.random_bits(syn.key_stream(5000 + trial, 0), n)
        seed_t, key_t = dev(sw), dev(kw)
        out = hash_under_plan(n, m, seed_t, key_t, plan, rng)
        torch.cuda.synchronize()
        want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
        assert np.array_equal(bits(out, m), want), (trial, n, m, plan)


def test_criterion2_plan_invariance_n_2e20():
    """n = 2^20: outputs under the plans (p column blocks, q row blocks) in {(1,1), (2,2),
    (4,1), (1,8)} are bit-identical, for random (u, seed)."""
    n = 1 << 20
    m = n // 10
    rng = np.random.default_rng(514)
    for trial in range(12):
        sw = syn.random_bits(syn.seed_stream(6000 + trial), n + m - 1)
        kw = syn.random_bits(syn.key_stream(6000 + trial, 0), n)
        seed_t, key_t = dev(sw), dev(kw)
        outs = []
        with pa.Hasher(n, m, seed_t) as h:  # (1, 1)
            outs.append(bits(h.hash(key_t), m))
        for p_, q_ in ((2, 2), (4, 1), (1, 8)):
            # column blocks of ~n/p key bits and row blocks of ~m/q bits: n_b + m_b - 1 <= lim
            mb = ((m + q_ - 1) // q_ + 31) // 32 * 32
            nb = (n + p_ - 1) // p_
            lim = nb + mb - 1
            out = torch.zeros(pa.words32(m) + 4, dtype=torch.int32, device=DEV)
            pa.pa_hash_blocked(n, m, seed_t.data_ptr(), key_t.data_ptr(), out.data_ptr(), lim, 0)
            outs.append(bits(out, m))
        with pa.Hasher(n, m, seed_t, route="transform", max_transform_len=n // 2) as h:  # Eq. (4) in-handle
            outs.append(bits(h.hash(key_t), m))
        for o in outs[1:]:
            assert np.array_equal(o, outs[0]), trial
        rows = np.unique(rng.integers(0, m, 64))
        assert np.array_equal(outs[0][rows], oracle.toeplitz_rows(n, m, sw, kw, rows))


@pytest.mark.parametrize("n", range(1, 7))
def test_criterion3_exhaustive_small_on_the_transform_route(n):
    """Every key and every seed for n <= 6, l <= min(n, 4) through the FP64 transform route
    (route (a), forced), against the schoolbook product mod 2: one handle per seed
    (pa_set_seed), all 2^n keys as one batch."""
    for m in range(1, min(n, 4) + 1):
        L = n + m - 1
        keys01 = ((np.arange(1 << n)[:, None] >> np.arange(n)) & 1).astype(np.uint8)
        kws = np.stack([oracle.pack(k, 32) for k in keys01]).astype(np.uint32)
        kt = torch.zeros((1 << n, 4), dtype=torch.int32, device=DEV)
        kt[:, :1] = torch.from_numpy(kws[:, :1].view(np.int32).copy()).to(DEV)
        seed_t = torch.zeros(8, dtype=torch.int32, device=DEV)
        with pa.Hasher(n, m, seed_t, route="transform") as h:
            outs = h.new_out(1 << n)
            for sv in range(1 << L):
                s01 = ((sv >> np.arange(L)) & 1).astype(np.uint8)
                seed_t[0] = int(np.int32(np.uint32(sv)))
                h.set_seed(seed_t)
                h.hash_batch(kt, outs)
                got = np.stack([oracle.unpack(r, m) for r in outs.cpu().numpy().view(np.uint32)])
                T = np.array([[s01[i - j + n - 1] for j in range(n)] for i in range(m)], dtype=np.int64)
                want = (keys01.astype(np.int64) @ T.T) & 1
                assert np.array_equal(got, want.astype(np.uint8)), (n, m, sv)


def test_criterion4_precision_contract():
    """Transform lengths in [2^23, 2^24]: 20 random trials, parities equal the exact
    result (sampled rows vs the oracle) and the recorded residual stays < 0.25 (typed
    PA_ERR_PRECISION otherwise: tests/test_parity_gpu.py fault injection)."""
    rng = np.random.default_rng(516)
    for trial in range(20):
        L = int(rng.integers(1 << 23, (1 << 24) - 64))  # n + m - 1 = transform length bound
        n = int(L * 10 // 11)
        m = L - n + 1
        sw = syn.random_bits(syn.seed_stream(7000 + trial), n + m - 1)
        kw = syn.random_bits(syn.key_stream(7000 + trial, 0), n)
        with pa.Hasher(n, m, dev(sw), route="transform") as h:
            assert (1 << 22) <= h.info["transform_len"] <= (1 << 25)
            y = bits(h.hash(dev(kw)), m)
            torch.cuda.synchronize()
            r = h.residual()
        assert r < 0.25
        rows = np.unique(rng.integers(0, m, 48))
        assert np.array_equal(y[rows], oracle.toeplitz_rows(n, m, sw, kw, rows)), trial


def test_criterion9_linearity_500_trials():
    """hash(a xor b) = hash(a) xor hash(b), 500 random trials, n <= 2^12, both routes."""
    rng = np.random.default_rng(522)
    for trial in range(500):
        n = int(rng.integers(1, (1 << 12) + 1))
        m = int(rng.integers(1, n + 1))
        sw = syn.random_bits(syn.seed_stream(8000 + trial), n + m - 1)
        a = syn.random_bits(syn.key_stream(8000 + trial, 0), n)
        b = syn.random_bits(syn.key_stream(8000 + trial, 1), n)
        route = "transform" if trial % 2 else "bitpacked"
        with pa.Hasher(n, m, dev(sw), route=route) as h:
            ya, yb, yab = (bits(h.hash(dev(k)), m) for k in (a, b, a ^ b))
        assert np.array_equal(yab, ya ^ yb), (trial, n, m, route)
