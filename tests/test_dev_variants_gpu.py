"""Opt-in kernel variants and forced plans, bit-exact against the oracle.

The product library (libpa.so) ignores the environment; these variants are reachable only in
the PA_DEV developer build (libpa_dev.so, built by __graft_entry__.build()).  Each test runs
its body in a child process with PA_LIB pointing at that build and the PA_* overrides set:
  * PA_K3T=1  -- the persistent TMEM-staged K3 (loader warps ld.global -> tcgen05.st, compute
                 warps tcgen05.ld -> shared memory), measured slower, off by default;
  * PA_LR=1   -- the row-block work-array layout between K2 and K3;
  * PA_FORCE_PLAN / PA_K3_HALF -- forced plans that exercise K3's half-width column groups;
  * PA_K1P=0 / PA_K2_FRESH=0 -- the plain K1 and the per-key-spectra fresh-seed path, each
                 bit-identical to the product path it replaces.
"""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - collected on CPU hosts
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DEV_LIB = os.path.join(ROOT, "paper_1805_02372_b200", "libpa_dev.so")


def run_child(body: str, args: dict, env: dict):
    """Run tests/test_dev_variants_gpu.py:<body>(**args) against the developer library."""
    if not os.path.exists(DEV_LIB):
        pytest.fail("libpa_dev.so missing: run __graft_entry__.build()")
    code = (f"import sys; sys.path[:0] = [{ROOT!r}, {os.path.join(ROOT, 'tests')!r}]\n"
            f"import test_dev_variants_gpu as t, json\n"
            f"t.{body}(**json.loads({json.dumps(json.dumps(args))}))\n")
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "PA_LIB": DEV_LIB, **env},
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


# ------------------------------------------------------------------ bodies (child process)
def _helpers():
    import numpy as np

    import oracle
    import paper_1805_02372_b200 as pa
    dev = torch.device("cuda:0")

    def to_dev(w64):
        w = np.ascontiguousarray(w64).view(np.int32)
        pad = (-w.size) % 4
        if pad:
            w = np.concatenate([w, np.zeros(pad, np.int32)])
        return torch.from_numpy(w.copy()).to(dev)

    def from_dev(t, m):
        return oracle.unpack(t.cpu().numpy().view(np.uint32), m)

    def sample_rows(m, seed=0, k=4096):
        rng = np.random.default_rng(seed)
        return np.unique(np.concatenate([np.arange(min(m, 256)), np.arange(max(0, m - 256), m),
                                         rng.integers(0, m, k)]))
    return np, oracle, pa, to_dev, from_dev, sample_rows


def body_k3t(name):
    import pa_synth as syn
    np, oracle, pa, to_dev, from_dev, sample_rows = _helpers()
    assert pa._lib.LIB_PATH == DEV_LIB
    n, m, sw, kw = syn.config_inputs(name)
    with pa.Hasher(n, m, to_dev(sw)) as h:
        got = from_dev(h.hash(to_dev(kw)), m)
        j = n // 3
        unit = from_dev(h.hash(to_dev(syn.unit_bits(n, j))), m)
        torch.cuda.synchronize()
        assert h.residual() < 1e-3
    rows = sample_rows(m, 5)
    assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, sw, kw, rows))
    s01 = oracle.unpack(sw, n + m - 1)
    assert np.array_equal(unit, s01[n - 1 - j:n - 1 - j + m])


def body_row_block(n, m):
    import pa_synth as syn
    np, oracle, pa, to_dev, from_dev, sample_rows = _helpers()
    sw = syn.random_bits(syn.seed_stream(101), n + m - 1)
    kw = syn.random_bits(syn.key_stream(101, 0), n)
    s01 = oracle.unpack(sw, n + m - 1)
    rows = sample_rows(m, 9)
    with pa.Hasher(n, m, to_dev(sw), route="transform") as h:
        got = from_dev(h.hash(to_dev(kw)), m)
        j = (2 * n) // 3
        unit = from_dev(h.hash(to_dev(syn.unit_bits(n, j))), m)
        torch.cuda.synchronize()
        assert h.residual() < 1e-3
    assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, sw, kw, rows))
    assert np.array_equal(unit, s01[n - 1 - j:n - 1 - j + m])


def body_k3_half(n, m, plan, half, out):
    import pa_synth as syn
    np, oracle, pa, to_dev, from_dev, sample_rows = _helpers()
    sw = syn.random_bits(syn.seed_stream(121), n + m - 1)
    kw = syn.random_bits(syn.key_stream(121, 0), n)
    s01 = oracle.unpack(sw, n + m - 1)
    with pa.Hasher(n, m, to_dev(sw), route="transform") as h:
        assert "%d,%d,%d" % (h.info["n1"], h.info["n2"], h.info["cols_per_cta"]) == plan
        assert h.info["k3_cols_per_cta"] == h.info["cols_per_cta"] // (2 if half == "1" else 1)
        got = from_dev(h.hash(to_dev(kw)), m)
        j = n // 2 + 1
        unit = from_dev(h.hash(to_dev(syn.unit_bits(n, j))), m)
        torch.cuda.synchronize()
        assert h.residual() < 1e-3
    assert np.array_equal(unit, s01[n - 1 - j:n - 1 - j + m])
    rows = sample_rows(m, 12)
    assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, sw, kw, rows))
    np.save(out, got)


# ------------------------------------------------------------------ tests
@pytest.mark.parametrize("name", ["C4", "C5d"])
def test_tmem_staged_k3_opt_in(name):
    """PA_K3T=1 (persistent TMEM-staged K3) is bit-exact at the sizes it serves: sampled rows vs
    the oracle plus the full unit-key closed form."""
    run_child("body_k3t", {"name": name}, {"PA_K3T": "1"})


@pytest.mark.parametrize("n,m", [(100_000_000, 20_000_000), (16_777_233, 1_677_723), (300_007, 60_001)])
@pytest.mark.parametrize("k3t", ["0", "1"])
def test_row_block_layout_opt_in(n, m, k3t):
    """PA_LR=1 (R x C blocks of a column group contiguous) through K1/K2/K3 and the seed path,
    with and without the TMEM-staged K3: sampled rows + the full unit-key closed form."""
    run_child("body_row_block", {"n": n, "m": m}, {"PA_LR": "1", "PA_K3T": k3t})


@pytest.mark.parametrize("n,m,plan", [(10_000_000, 1_000_000, "4096,1792,4"), (3_000_000, 300_000, "1024,3600,2"),
                                       (2_000_003, 400_000, "1536,4096,2")])
def test_k3_half_column_groups(n, m, plan, tmp_path):
    """K3 on half of K1's column groups (Geometry::C3) under forced plans: bit-exact against the
    oracle and the unit-key closed form, and identical to K3 on K1's groups (PA_K3_HALF=0)."""
    import numpy as np
    outs = []
    for half in ("1", "0"):
        f = str(tmp_path / f"half{half}.npy")
        run_child("body_k3_half", {"n": n, "m": m, "plan": plan, "half": half, "out": f},
                  {"PA_FORCE_PLAN": plan, "PA_K3_HALF": half})
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


def body_k1p_off(n, m, count, out):
    """Hash `count` keys with K1P disabled (PA_K1P=0: the non-persistent K1) and save them."""
    import numpy as np

    import pa_synth as syn
    np_, oracle, pa, to_dev, from_dev, sample_rows = _helpers()
    sw = syn.random_bits(syn.seed_stream(171), n + m - 1)
    keys = syn.random_bits_torch([syn.key_stream(171, k) for k in range(count)], n, "cuda")
    with pa.Hasher(n, m, to_dev(sw), route="transform") as h:
        outs = h.hash_batch(keys)
        torch.cuda.synchronize()
        np.save(out, outs.cpu().numpy()[:, :pa.words32(m)])  # the output words only (rows are padded)


@pytest.mark.parametrize("count", [1, 3])
def test_k1p_matches_plain_k1(count, tmp_path):
    """K1P (persistent K1, TMEM write-behind; the product path at C4) performs the same FP64
    operations in the same order as the plain K1, so the hashes are identical bit for bit -- one
    key and a batch whose tiles span keys; plus sampled rows of the last key vs the oracle."""
    import numpy as np

    import oracle
    import paper_1805_02372_b200 as pa
    import pa_synth as syn
    n, m = 100_000_000, 20_000_000
    sw = syn.random_bits(syn.seed_stream(171), n + m - 1)
    seed = torch.from_numpy(np.ascontiguousarray(sw).view(np.int32).copy()).cuda()
    keys = syn.random_bits_torch([syn.key_stream(171, k) for k in range(count)], n, "cuda")
    with pa.Hasher(n, m, seed, route="transform") as h:
        assert h.info["cols_per_cta"] == 2  # the C4 plan K1P serves
        outs = h.hash_batch(keys).cpu().numpy()[:, :pa.words32(m)]
    f = str(tmp_path / "plain.npy")
    run_child("body_k1p_off", {"n": n, "m": m, "count": count, "out": f}, {"PA_K1P": "0"})
    assert np.array_equal(outs, np.load(f))
    kk = syn.random_bits(syn.key_stream(171, count - 1), n)
    rows = np.unique(np.random.default_rng(7).integers(0, m, 128))
    got = oracle.unpack(outs[count - 1].view(np.uint32), m)
    assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, sw, kk, rows))


def body_fresh(n, m, count, out):
    """pa_hash_fresh_batch of `count` keys against their own seeds; save outputs + residual."""
    import numpy as np

    import pa_synth as syn
    L = n + m - 1
    seeds = syn.random_bits_torch([syn.seed_stream(190 + k) for k in range(count)], L, "cuda")
    keys = syn.random_bits_torch([syn.key_stream(190, k) for k in range(count)], n, "cuda")
    import paper_1805_02372_b200 as pa
    with pa.Hasher(n, m, seeds[0], route="transform") as h:
        # the ceil(m/32) output words only: new_out's rows are padded to 16 bytes, and the padding
        # words are not part of the output (whatever the allocator left there stays)
        outs = h.hash_fresh_batch(seeds, keys).cpu().numpy()[:, :pa.words32(m)]
        np.save(out, np.concatenate([outs.reshape(-1).view(np.uint32),
                                     np.array([h.residual()]).view(np.uint32)]))


@pytest.mark.parametrize("n,m,count", [(1_000_003, 250_000, 5), (50_000_017, 5_000_001, 2)])
def test_fresh_fused_matches_spectra_path(n, m, count, tmp_path):
    """The fused fresh-seed K2 (seed forward half in the hash's K2, spectrum row in TMEM; product
    path) and the per-key spectra path (PA_K2_FRESH=0: seed K2 writes spectra to HBM, the hash's
    K2 reads them) perform the same FP64 operations in the same order: identical outputs and the
    identical residual, bit for bit."""
    import numpy as np
    f1, f0 = str(tmp_path / "fused.npy"), str(tmp_path / "spectra.npy")
    body_fresh(n, m, count, f1)
    run_child("body_fresh", {"n": n, "m": m, "count": count, "out": f0}, {"PA_K2_FRESH": "0"})
    assert np.array_equal(np.load(f1), np.load(f0))
