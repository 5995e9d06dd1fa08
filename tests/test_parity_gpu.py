"""GPU parity: libpa (through the C ABI) vs the CPU oracle, bit-exact.

Inputs are seeded SplitMix64 bit strings (pa_synth).  Sizes span several
tiles and ragged tails; full outputs are compared where the oracle finishes in
seconds, sampled rows (each an independent O(n) oracle evaluation) plus
closed forms at the BASELINE.json sizes.
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
FULL_LIMIT = 3e10   # n*m bit-products the oracle runs in full (OpenMP, seconds)


def to_dev(words64: np.ndarray) -> torch.Tensor:
    w = np.ascontiguousarray(words64).view(np.int32)
    pad = (-w.size) % 4
    if pad:
        w = np.concatenate([w, np.zeros(pad, np.int32)])
    return torch.from_numpy(w.copy()).to(DEV)


def from_dev(t: torch.Tensor, m: int) -> np.ndarray:
    return oracle.unpack(t.cpu().numpy().view(np.uint32), m)


def sample_rows(m: int, seed: int = 0, k: int = 4096) -> np.ndarray:
    rng = np.random.default_rng(seed)
    r = np.concatenate([np.arange(min(m, 256)), np.arange(max(0, m - 256), m), rng.integers(0, m, k)])
    return np.unique(r)


def check(n, m, sw, kw, route, full=None):
    seed_t, key_t = to_dev(sw), to_dev(kw)
    with pa.Hasher(n, m, seed_t, route=route) as h:
        out = h.hash(key_t)
        torch.cuda.synchronize()
        got = from_dev(out, m)
        # tail bits beyond m are zero
        allbits = oracle.unpack(out.cpu().numpy().view(np.uint32), 32 * ((m + 31) // 32))
        assert not allbits[m:].any()
        res = h.residual()
        info = h.info
    if full is None:
        full = n * m <= FULL_LIMIT
    if full:
        want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, f"n={n} m={m} route={route} {bad.size} wrong bits, first {bad[:8]} info={info}"
    else:
        rows = sample_rows(m, n)
        want = oracle.toeplitz_rows(n, m, sw, kw, rows)
        bad = np.flatnonzero(got[rows] != want)
        assert bad.size == 0, f"n={n} m={m} route={route} sampled rows wrong: {rows[bad[:8]]}"
    if info["route"] == pa.PA_ROUTE_TRANSFORM:
        assert res < 1e-3, res
    return got, info


SWEEP_N = [1, 2, 31, 32, 33, 63, 64, 65, 127, 1000, 4095, 4096, 4097, 65537, 1_000_003]


def _ms(n):
    return sorted({m for m in (1, 32, 33, n // 10, n // 4, n) if 1 <= m <= n})


@pytest.mark.parametrize("route", ["bitpacked", "transform"])
@pytest.mark.parametrize("n", SWEEP_N)
def test_length_sweep(route, n):
    for m in _ms(n):
        if route == "bitpacked" and n * m > 2e11:
            continue
        sw = syn.random_bits(syn.seed_stream(100 + n % 97), n + m - 1)
        kw = syn.random_bits(syn.key_stream(100, n + m), n)
        check(n, m, sw, kw, route)


@pytest.mark.parametrize("name", ["C1", "C2"])
def test_configs_full(name):
    n, m, sw, kw = syn.config_inputs(name)
    for route in ("transform", "bitpacked") if name == "C1" else ("transform",):
        check(n, m, sw, kw, route, full=True)


@pytest.mark.parametrize("name", ["C3", "C4", "C5a", "C5b", "C5c", "C5d"])
def test_configs_sampled_and_closed_forms(name):
    """BASELINE.json sizes, same launch configuration as bench.py: sampled rows
    vs the oracle, plus full-output closed forms (all-ones key, unit keys)."""
    n, m, sw, kw = syn.config_inputs(name)
    check(n, m, sw, kw, "auto", full=False)
    L = n + m - 1
    s = oracle.unpack(sw, L)
    P = np.zeros(L + 1, np.uint8)
    P[1:] = np.bitwise_xor.accumulate(s)
    with pa.Hasher(n, m, to_dev(sw)) as h:
        got = from_dev(h.hash(to_dev(syn.ones_bits(n))), m)
        i = np.arange(m)
        assert np.array_equal(got, P[i + n] ^ P[i])
        for j in (0, n // 3, n - 1):
            got = from_dev(h.hash(to_dev(syn.unit_bits(n, j))), m)
            assert np.array_equal(got, s[n - 1 - j: n - 1 - j + m]), j
        assert h.residual() < 1e-3


def test_routes_agree():
    """P8: the two exact GPU algorithms agree bit for bit."""
    for n, m in ((20_011, 2_001), (100_000, 25_000), (333_333, 3_333)):
        sw = syn.random_bits(syn.seed_stream(7 + n), n + m - 1)
        kw = syn.random_bits(syn.key_stream(7, n), n)
        a, _ = check(n, m, sw, kw, "transform", full=False)
        b, _ = check(n, m, sw, kw, "bitpacked", full=False)
        assert np.array_equal(a, b)


def test_structured_inputs():
    n, m = 50_000, 12_345
    L = n + m - 1
    sw = syn.random_bits(syn.seed_stream(9), L)
    s = oracle.unpack(sw, L)
    for route in ("transform", "bitpacked"):
        with pa.Hasher(n, m, to_dev(sw), route=route) as h:
            assert not from_dev(h.hash(to_dev(syn.zero_bits(n))), m).any()
            kw, pos = syn.sparse_bits(11, n, 25)
            want = np.zeros(m, np.uint8)
            for j in pos:
                want ^= s[n - 1 - j: n - 1 - j + m]
            assert np.array_equal(from_dev(h.hash(to_dev(kw)), m), want)
        with pa.Hasher(n, m, to_dev(syn.ones_bits(L)), route=route) as h:
            kw = syn.random_bits(5, n)
            par = int(oracle.unpack(kw, n).sum() & 1)
            assert np.all(from_dev(h.hash(to_dev(kw)), m) == par)


def test_linearity_and_garbage_tail_bits():
    n, m = 77_777, 7_777
    sw = syn.random_bits(syn.seed_stream(21), n + m - 1)
    a = syn.random_bits(31, n)
    b = syn.random_bits(32, n)
    for route in ("transform", "bitpacked"):
        with pa.Hasher(n, m, to_dev(sw), route=route) as h:
            ya = from_dev(h.hash(to_dev(a)), m)
            yb = from_dev(h.hash(to_dev(b)), m)
            assert np.array_equal(from_dev(h.hash(to_dev(a ^ b)), m), ya ^ yb)
            a2 = a.copy()
            a2[-1] |= np.uint64(0xFFFF_FFFF_FFFF_FFFF) << np.uint64(n % 64)
            assert np.array_equal(from_dev(h.hash(to_dev(a2)), m), ya)


@pytest.mark.parametrize("route", ["transform", "bitpacked"])
def test_seed_offset_row_and_column_shards(route):
    """Row and column shards via pa_options.seed_bit_offset reassemble y (P7,
    the paper's Eq. (4) split and Eq. (7) merge)."""
    n, m = 40_000, 9_000
    L = n + m - 1
    sw = syn.random_bits(syn.seed_stream(33), L)
    kw = syn.random_bits(syn.key_stream(33, 0), n)
    want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
    seed_t = to_dev(sw)
    key_bits = oracle.unpack(kw, n)
    parts = []
    for r0, r1 in ((0, 3000), (3000, 3001), (3001, m)):
        with pa.Hasher(n, r1 - r0, seed_t, route=route, seed_bit_offset=r0) as h:
            parts.append(from_dev(h.hash(to_dev(kw)), r1 - r0))
    assert np.array_equal(np.concatenate(parts), want)
    acc = np.zeros(m, np.uint8)
    for c0, c1 in ((0, 12_345), (12_345, 21_346), (21_346, n)):  # each >= m bits (m <= n_g)
        ng = c1 - c0
        with pa.Hasher(ng, m, seed_t, route=route, seed_bit_offset=n - ng - c0) as h:
            acc ^= from_dev(h.hash(to_dev(oracle.pack(key_bits[c0:c1]))), m)
    assert np.array_equal(acc, want)


def test_batch_and_u64_and_host_paths():
    n, m = 123_457, 30_000
    sw = syn.random_bits(syn.seed_stream(44), n + m - 1)
    keys = [syn.random_bits(syn.key_stream(44, k), n) for k in range(5)]
    kw32 = (n + 31) // 32
    stride = (kw32 + 3) // 4 * 4
    mat = np.zeros((5, stride), np.int32)
    for k, w in enumerate(keys):
        mat[k, :kw32] = w.view(np.int32)[:kw32]
    for route in ("transform", "bitpacked"):
        with pa.Hasher(n, m, to_dev(sw), route=route) as h:
            outs = h.hash_batch(torch.from_numpy(mat).to(DEV))
            torch.cuda.synchronize()
            for k, w in enumerate(keys):
                want = oracle.unpack(oracle.toeplitz_words(n, m, sw, w), m)
                assert np.array_equal(oracle.unpack(outs[k].cpu().numpy().view(np.uint32), m), want)
                # host end-to-end path
                kh = torch.from_numpy(w.view(np.int32).copy()).pin_memory()
                oh = torch.zeros((m + 31) // 32, dtype=torch.int32).pin_memory()
                h.hash_host(kh, oh)
                assert np.array_equal(oracle.unpack(oh.numpy().view(np.uint32), m), want)
        # uint64 aliases: output tail half-word zero-filled
        seed_t = to_dev(sw)
        hh = pa.pa_create_u64(n, m, seed_t.data_ptr(), 0)
        try:
            out = torch.full(((m + 63) // 64 * 2,), -1, dtype=torch.int32, device=DEV)
            key0 = to_dev(keys[0])  # keep alive across the call
            pa.pa_hash_u64(hh, key0.data_ptr(), out.data_ptr(), 0)
            torch.cuda.synchronize()
            allb = oracle.unpack(out.cpu().numpy().view(np.uint32), 64 * ((m + 63) // 64))
            want = oracle.unpack(oracle.toeplitz_words(n, m, sw, keys[0]), m)
            assert np.array_equal(allb[:m], want) and not allb[m:].any()
        finally:
            pa.pa_destroy(hh)


def test_rejects_host_pointer_and_misalignment():
    n, m = 1000, 100
    seed_t = to_dev(syn.random_bits(1, n + m - 1))
    host = torch.zeros(64, dtype=torch.int32)
    with pytest.raises(pa.PaError) as e:
        pa.pa_create(n, m, host.data_ptr(), 0)
    assert e.value.status == pa.PA_ERR_INVALID_ARG
    with pytest.raises(pa.PaError):
        pa.pa_create(n, m, seed_t.data_ptr() + 4, 0)
    with pa.Hasher(n, m, seed_t) as h:
        with pytest.raises(pa.PaError):
            pa.pa_hash(h.handle, host.data_ptr(), h.new_out().data_ptr(), 0)


def test_tiny_transform_edge_cases():
    """Degenerate lengths on the transform route: n = m = 1, m = n, m = 1."""
    for n, m in ((1, 1), (2, 1), (2, 2), (3, 3), (7, 1), (8, 8), (100, 1), (100, 100)):
        for sv in range(3):
            sw = syn.random_bits(1000 + sv, n + m - 1)
            kw = syn.random_bits(2000 + sv, n)
            check(n, m, sw, kw, "transform", full=True)


@pytest.mark.parametrize("n,m,count", [(1_048_576, 104_857, 70), (3_000_000, 300_000, 9), (200_003, 50_000, 1)])
def test_batch_native_many_keys(n, m, count):
    """pa_hash_batch on the transform route runs keys in grid-batched chunks
    (BASELINE.json configs[4] shape); every output equals its own oracle result."""
    sw = syn.random_bits(syn.seed_stream(55), n + m - 1)
    kw32 = (n + 31) // 32
    stride = (kw32 + 3) // 4 * 4
    keys = [syn.random_bits(syn.key_stream(55, k), n) for k in range(count)]
    mat = np.zeros((count, stride), np.int32)
    for k, w in enumerate(keys):
        mat[k, :kw32] = w.view(np.int32)[:kw32]
    with pa.Hasher(n, m, to_dev(sw), route="transform") as h:
        outs = h.hash_batch(torch.from_numpy(mat).to(DEV)).cpu().numpy()
        single = from_dev(h.hash(to_dev(keys[-1])), m)
        assert h.residual() < 1e-3
    rows = sample_rows(m, 3, 512)
    for k in sorted({0, count // 2, count - 1}):
        got = oracle.unpack(outs[k].view(np.uint32), m)
        assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, sw, keys[k], rows)), k
        assert not oracle.unpack(outs[k].view(np.uint32), 32 * ((m + 31) // 32))[m:].any()
    assert np.array_equal(oracle.unpack(outs[-1].view(np.uint32), m), single)


@pytest.mark.parametrize("route", ["transform", "bitpacked"])
def test_fresh_seed_per_key(route):
    """pa_set_seed: a new seed per round gives the same result as a
    handle created on that seed, and hashes queued before the call keep the old one."""
    n, m = 70_001, 17_000
    s1 = syn.random_bits(syn.seed_stream(61), n + m - 1)
    s2 = syn.random_bits(syn.seed_stream(62), n + m - 1)
    kw = syn.random_bits(syn.key_stream(61, 0), n)
    with pa.Hasher(n, m, to_dev(s1), route=route) as h:
        key = to_dev(kw)
        y1 = h.hash(key)
        h.set_seed(to_dev(s2))
        y2 = h.hash(key)
        torch.cuda.synchronize()
        assert np.array_equal(from_dev(y1, m), oracle.unpack(oracle.toeplitz_words(n, m, s1, kw), m))
        assert np.array_equal(from_dev(y2, m), oracle.unpack(oracle.toeplitz_words(n, m, s2, kw), m))


def test_xor_fold_kernel():
    """pa_xor_fold: XOR of G packed partials (the Eq. (7) merge)."""
    rng = np.random.default_rng(5)
    for G, words in ((1, 7), (5, 1027), (8, 4096)):
        stride = (words + 3) // 4 * 4
        src = rng.integers(-2**31, 2**31 - 1, size=(G, stride), dtype=np.int64).astype(np.int32)
        want = np.bitwise_xor.reduce(src[:, :words], axis=0)
        s = torch.from_numpy(src).to(DEV)
        d = torch.full((stride,), 7, dtype=torch.int32, device=DEV)
        pa.pa_xor_fold(d.data_ptr(), s.data_ptr(), words, G, stride, 0)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy()[:words], want)


def test_dist_driver_single_rank_nccl():
    """dist.hash_rows / hash_cols / hash_keys through libpa and NCCL (world size 1 on
    this box; the multi-rank split arithmetic is covered on CPU with gloo)."""
    import os
    import socket
    import torch.distributed as dist
    from paper_1805_02372_b200 import dist as pd
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=DEV)
    try:
        n, m = 300_007, 60_000
        sw = syn.random_bits(syn.seed_stream(71), n + m - 1)
        kw = syn.random_bits(syn.key_stream(71, 0), n)
        want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
        seed_t = to_dev(sw)
        rows = pd.hash_rows(n, m, seed_t, to_dev(kw))
        cols = pd.hash_cols(n, m, seed_t, kw)
        torch.cuda.synchronize()
        assert np.array_equal(from_dev(rows, m), want)
        assert np.array_equal(from_dev(cols, m), want)
        keys = torch.stack([to_dev(syn.random_bits(syn.key_stream(72, k), n)) for k in range(3)])
        idx, outs = pd.hash_keys(n, m, seed_t, keys)
        assert idx == [0, 1, 2]
        for k in idx:
            wk = oracle.unpack(oracle.toeplitz_words(n, m, sw, syn.random_bits(syn.key_stream(72, k), n)), m)
            assert np.array_equal(from_dev(outs[k], m), wk)
        # persistent sharded hashers (bench.py --split rows / cols), repeated calls
        for cls in (pd.RowSplit, pd.ColSplit):
            sh = cls(n, m, seed_t)
            k = to_dev(kw) if cls is pd.RowSplit else sh.key_block(kw, DEV)
            for _ in range(3):
                y = sh(k)
            torch.cuda.synchronize()
            assert np.array_equal(from_dev(y, m), want), cls.__name__
            sh.close()
        # fused Eq. (7) merge (NEXT-1): K3's partial in a peer-mappable buffer, folded by
        # pa_xor_fold_peers through the device pointer table, for several steps and shapes
        for nn, mm in ((n, m), (4096 * 3 + 17, 5_000), (1_000_003, 250_000)):
            s2 = syn.random_bits(syn.seed_stream(73), nn + mm - 1)
            k2 = [syn.random_bits(syn.key_stream(73, k), nn) for k in range(3)]
            sh = pd.ColSplit(nn, mm, to_dev(s2), fused=True)
            for kk in k2:
                y = sh(sh.key_block(kk, DEV))
                torch.cuda.synchronize()
                assert np.array_equal(from_dev(y, mm), oracle.unpack(oracle.toeplitz_words(nn, mm, s2, kk), mm))
            sh.close()
        # the one-shot auto entry point: key on the source rank, cost-model split
        split, y = pd.hash(n, m, seed_t, to_dev(kw))
        torch.cuda.synchronize()
        assert split == "rows" and np.array_equal(from_dev(y, m), want)
    finally:
        dist.destroy_process_group()


def test_xor_fold_peers_pointer_table():
    """pa_xor_fold_peers over a device table of pointers (here all local): dst = XOR of the
    slices [first, first + words) of every source, ragged lengths and offsets."""
    rng = np.random.default_rng(5)
    for G, words, first in ((1, 7, 0), (3, 1000, 4), (8, 4097, 12), (5, 3, 8)):
        srcs = [torch.from_numpy(rng.integers(-2**31, 2**31, first + words + 5, dtype=np.int64).astype(np.int32))
                .to(DEV) for _ in range(G)]
        table = torch.tensor([t.data_ptr() for t in srcs], dtype=torch.int64, device=DEV)
        dst = torch.full((words + 4,), -1, dtype=torch.int32, device=DEV)
        pa.pa_xor_fold_peers(dst.data_ptr(), table.data_ptr(), G, first, words, 0)
        torch.cuda.synchronize()
        want = np.zeros(words, np.int32)
        for t in srcs:
            want ^= t.cpu().numpy()[first:first + words]
        assert np.array_equal(dst.cpu().numpy()[:words], want)
        assert (dst.cpu().numpy()[words:] == -1).all()
    ptr = pa.pa_peer_alloc(4096)
    try:
        assert len(pa.pa_peer_export(ptr)) == 64
    finally:
        pa.pa_peer_free(ptr)


def test_host_async_graph_repoints_buffers():
    """pa_hash_host_async / pa_hash_host replay one captured CUDA graph; new host
    buffers are patched into its copy nodes."""
    n, m = 1_000_003, 250_000
    sw = syn.random_bits(syn.seed_stream(81), n + m - 1)
    keys = [syn.random_bits(syn.key_stream(81, k), n) for k in range(3)]
    with pa.Hasher(n, m, to_dev(sw)) as h:
        outs = []
        for k, w in enumerate(keys):
            kh = torch.from_numpy(w.view(np.int32).copy()).pin_memory()
            oh = torch.zeros((m + 31) // 32, dtype=torch.int32).pin_memory()
            (h.hash_host_async if k % 2 == 0 else h.hash_host)(kh, oh)
            outs.append((kh, oh))
        torch.cuda.synchronize()
        rows = sample_rows(m, 9, 512)
        for (kh, oh), w in zip(outs, keys):
            got = oracle.unpack(oh.numpy().view(np.uint32), m)
            assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, sw, w, rows))


def test_host_copy_modes_pinned_pageable_misaligned():
    """pa_hash_host moves a small key / output with copy kernels over mapped pinned pages and
    falls back to the copy engines for pageable buffers; switching between the two (and
    4-byte-aligned host pointers, the kernels' scalar path) re-builds or re-points the graph
    and every result stays exact."""
    n, m = 1_000_003, 250_000
    kw_, ow = pa.words32(n), pa.words32(m)
    sw = syn.random_bits(syn.seed_stream(83), n + m - 1)
    keys = [syn.random_bits(syn.key_stream(83, k), n) for k in range(6)]
    rows = sample_rows(m, 11, 512)
    with pa.Hasher(n, m, to_dev(sw)) as h:
        for k, w in enumerate(keys):
            kind = ("pinned", "pageable", "pinned+4", "pinned", "pageable+4", "pinned+4")[k]
            pin = kind.startswith("pinned")
            off = 1 if kind.endswith("+4") else 0
            kbuf = torch.zeros(kw_ + 4, dtype=torch.int32)
            obuf = torch.full((ow + 4,), -1, dtype=torch.int32)
            if pin:
                kbuf, obuf = kbuf.pin_memory(), obuf.pin_memory()
            kbuf[off:off + kw_] = torch.from_numpy(w.view(np.int32)[:kw_].copy())
            kh, oh = kbuf[off:off + kw_], obuf[off:off + ow]
            assert (kh.data_ptr() % 16 != 0) == bool(off)
            (h.hash_host if k % 2 else h.hash_host_async)(kh, oh)
            torch.cuda.synchronize()
            got = oracle.unpack(oh.numpy().view(np.uint32), 32 * ow)
            assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, sw, w, rows)), kind
            assert not got[m:].any(), kind
            assert (obuf[:off] == -1).all() and (obuf[off + ow:] == -1).all(), kind  # nothing outside


@pytest.mark.parametrize("n,m,maxb", [(20_000, 7_000, 5_000), (50_001, 20_000, 16_384), (3001, 3000, 700),
                                      (100_000, 10_000, 0)])
def test_length_compatible_blocked(n, m, maxb):
    """pa_hash_blocked: row x column block division with the Eq. (7) XOR merge equals
    the single-transform hash (plan invariance)."""
    sw = syn.random_bits(syn.seed_stream(91 + n), n + m - 1)
    kw = syn.random_bits(syn.key_stream(91, n), n)
    out = torch.full(((m + 31) // 32 + 3,), -1, dtype=torch.int32, device=DEV)
    seed_t, key_t = to_dev(sw), to_dev(kw)  # keep the tensors alive across the call
    pa.pa_hash_blocked(n, m, seed_t.data_ptr(), key_t.data_ptr(), out.data_ptr(), maxb, 0)
    torch.cuda.synchronize()
    want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
    allb = oracle.unpack(out.cpu().numpy().view(np.uint32), 32 * ((m + 31) // 32))
    assert np.array_equal(allb[:m], want)
    assert not allb[m:].any()


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_worst_case_rounding_all_ones(name):
    """All-ones key and seed maximise |x|_2 |s|_2 in the FP64 error bound (DESIGN.md
    Sec. 5): every count is exactly n, so y[i] = n mod 2 for all i, and the recorded
    residual must stay far below 0.5."""
    n, m = syn.CONFIGS[name]["n"], syn.CONFIGS[name]["m"]
    with pa.Hasher(n, m, to_dev(syn.ones_bits(n + m - 1))) as h:
        got = from_dev(h.hash(to_dev(syn.ones_bits(n))), m)
        res = h.residual()
    assert np.all(got == (n & 1))
    assert res < 1e-3, res


# ---------------------------------------------------------------- caller-owned workspace
@pytest.mark.parametrize("route,n,m,split", [("bitpacked", 4096, 1024, 0), ("transform", 300_007, 60_001, 0),
                                             ("transform", 300_007, 60_001, 200_000)])
def test_workspace_owned_by_caller(route, n, m, split):
    """pa_create_ws: the handle's device memory is the caller's tensor -- nothing else is
    allocated (device free memory unchanged), the bytes match pa_workspace_size and the
    result matches the oracle, for single keys, batches (chunked at batch_keys) and the
    host path."""
    sw = syn.random_bits(syn.seed_stream(61), n + m - 1)
    keys = [syn.random_bits(syn.key_stream(61, k), n) for k in range(7)]
    opts = dict(route=route, batch_keys=3, max_transform_len=split)
    need = pa.workspace_size(n, m, **opts)
    # every torch buffer first, so the free-memory check below sees libpa alone
    seed_t = to_dev(sw)
    ws = torch.empty(need, dtype=torch.uint8, device=DEV)
    kt = torch.stack([to_dev(k) for k in keys])
    w4 = ((m + 31) // 32 + 3) // 4 * 4
    outs = torch.empty((len(keys), w4), dtype=torch.int32, device=DEV)
    one = torch.empty(w4, dtype=torch.int32, device=DEV)
    kh = kt[1].cpu().pin_memory()
    oh = torch.zeros(w4, dtype=torch.int32).pin_memory()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    with pa.Hasher(n, m, seed_t, workspace=ws, **opts) as h:
        h.hash_batch(kt, outs)
        h.hash(kt[0], one)
        h.hash_host(kh, oh)
        torch.cuda.synchronize()
        free1 = torch.cuda.mem_get_info()[0]
        assert h.info["workspace_bytes"] == need
        assert (h.info["column_blocks"] > 1) == bool(split)
        assert h.residual() < 1e-3
    assert abs(free0 - free1) <= (2 << 20), (free0, free1)  # no hidden cudaMalloc
    for k, kw in enumerate(keys):
        want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
        assert np.array_equal(from_dev(outs[k], m), want), k
    assert np.array_equal(from_dev(one, m), oracle.unpack(oracle.toeplitz_words(n, m, sw, keys[0]), m))
    assert np.array_equal(oracle.unpack(oh.numpy().view(np.uint32), m),
                          oracle.unpack(oracle.toeplitz_words(n, m, sw, keys[1]), m))


def test_workspace_too_small_is_nomem():
    n, m = 100_000, 10_000
    seed_t = to_dev(syn.random_bits(syn.seed_stream(62), n + m - 1))
    need = pa.workspace_size(n, m, route="transform")
    ws = torch.empty(need - 4096, dtype=torch.uint8, device=DEV)
    with pytest.raises(pa.PaError) as e:
        pa.Hasher(n, m, seed_t, route="transform", workspace=ws)
    assert e.value.status == pa.PA_ERR_NOMEM and "workspace" in pa.pa_last_error()


# ---------------------------------------------------------------- Eq. (4) split in a handle
@pytest.mark.parametrize("n,m,maxlen", [(300_007, 60_001, 200_000), (500_009, 100_000, 350_000),
                                        (65_537, 60_000, 61_000), (4_099, 4_000, 4_300)])
def test_max_transform_len_split_matches_unsplit_and_oracle(n, m, maxlen):
    """Plan invariance: the column-split handle (Eq. (4) blocks on seed windows
    n - n_g - c0, partial outputs XOR-merged in place, Eq. (7)) reproduces y exactly, through
    pa_hash, pa_hash_batch, pa_hash_u64 and pa_set_seed."""
    sw = syn.random_bits(syn.seed_stream(63), n + m - 1)
    sw2 = syn.random_bits(syn.seed_stream(64), n + m - 1)
    keys = [syn.random_bits(syn.key_stream(63, k), n) for k in range(3)]
    with pa.Hasher(n, m, to_dev(sw), route="transform", max_transform_len=maxlen) as h:
        info = h.info
        assert info["column_blocks"] > 1 and info["transform_len"] <= maxlen, info
        y = [h.hash(to_dev(k)) for k in keys]
        kt = torch.stack([to_dev(k) for k in keys])
        yb = h.hash_batch(kt)
        k64 = to_dev(keys[0])
        o64 = torch.full((2 * ((m + 63) // 64) + 4,), -1, dtype=torch.int32, device=DEV)
        pa.pa_hash_u64(h.handle, k64.data_ptr(), o64.data_ptr(), 0)
        h.set_seed(to_dev(sw2))
        y2 = h.hash(to_dev(keys[0]))
        torch.cuda.synchronize()
        assert h.residual() < 1e-3
    for k, kw in enumerate(keys):
        want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
        assert np.array_equal(from_dev(y[k], m), want), ("hash", k)
        assert np.array_equal(from_dev(yb[k], m), want), ("batch", k)
    w64 = o64.cpu().numpy().view(np.uint32)
    assert np.array_equal(oracle.unpack(w64, m), oracle.unpack(oracle.toeplitz_words(n, m, sw, keys[0]), m))
    assert not oracle.unpack(w64[: 2 * ((m + 63) // 64)], 64 * ((m + 63) // 64))[m:].any()
    assert np.array_equal(from_dev(y2, m), oracle.unpack(oracle.toeplitz_words(n, m, sw2, keys[0]), m))


def test_max_transform_len_too_small_is_unsupported():
    n, m = 10_000, 5_000
    seed_t = to_dev(syn.random_bits(syn.seed_stream(65), n + m - 1))
    with pytest.raises(pa.PaError) as e:
        pa.Hasher(n, m, seed_t, route="transform", max_transform_len=m + 100)
    assert e.value.status == pa.PA_ERR_UNSUPPORTED


# ---------------------------------------------------------------- fresh seed per key
@pytest.mark.parametrize("route,maxlen,count", [("bitpacked", 0, 5), ("transform", 0, 5), ("transform", 150_000, 5),
                                                ("transform", 0, 70), ("transform", 0, 1)])
def test_hash_fresh_batch_per_key_seeds(route, maxlen, count):
    """NEXT-2: key k hashed with its own seed k, three transforms per key.  Unsplit route
    (a) transforms a chunk's seeds as one batch into per-key spectra and hashes the chunk against
    them (70 keys: two chunks, the second ragged); afterwards the handle holds the last seed."""
    n, m = (3_001, 1_000) if route == "bitpacked" else (120_001, 30_000)
    seeds = [syn.random_bits(syn.seed_stream(70 + k), n + m - 1) for k in range(count)]
    keys = [syn.random_bits(syn.key_stream(70, k), n) for k in range(count)]
    st, kt = torch.stack([to_dev(s) for s in seeds]), torch.stack([to_dev(k) for k in keys])
    probe = syn.random_bits(syn.key_stream(71, 0), n)
    with pa.Hasher(n, m, st[0], route=route, max_transform_len=maxlen) as h:
        outs = h.hash_fresh_batch(st, kt)
        after = from_dev(h.hash(to_dev(probe)), m)
        torch.cuda.synchronize()
    for k in range(count):
        want = oracle.unpack(oracle.toeplitz_words(n, m, seeds[k], keys[k]), m)
        assert np.array_equal(from_dev(outs[k], m), want), k
    assert np.array_equal(after, oracle.unpack(oracle.toeplitz_words(n, m, seeds[-1], probe), m))


@pytest.mark.parametrize("n,m,count", [(250_007, 62_000, 3), (20_000_003, 4_000_000, 2), (50_000_017, 5_000_001, 2),
                                     (1_048_576, 104_857, 70)])
def test_hash_fresh_batch_fused_k2_shapes(n, m, count):
    """The fresh-seed K2 (each seed's forward half in the hash's K2, its spectrum row held in
    TMEM) on the row shapes 2048 = [8, 16, 16] (two CTAs per SM, 256 TMEM columns each),
    6144 = [3, 8, 16, 16] and 10240 = [5, 8, 16, 16] (one CTA per SM, 512 columns, two last-stage
    butterflies per thread): every key against its own seed, and the handle afterwards holds the
    last seed (the spectrum row the last key's CTAs wrote; 70 keys: two chunks, each chunk's
    last key rewrites it).  Full outputs at the small shape, sampled rows (both ends + random) at
    the large ones."""
    L = n + m - 1
    seeds = [syn.random_bits(syn.seed_stream(150 + k), L) for k in range(count)]
    keys = [syn.random_bits(syn.key_stream(150, k), n) for k in range(count)]
    probe = syn.random_bits(syn.key_stream(151, 0), n)
    st, kt = torch.stack([to_dev(s) for s in seeds]), torch.stack([to_dev(k) for k in keys])
    with pa.Hasher(n, m, to_dev(syn.random_bits(syn.seed_stream(149), L)), route="transform") as h:
        outs = h.hash_fresh_batch(st, kt)
        after = from_dev(h.hash(to_dev(probe)), m)
        assert h.residual() < 0.25
        torch.cuda.synchronize()
    full = n * m <= 2 * 10**10
    rows = sample_rows(m, 29, 384)
    for k in range(count):
        got = from_dev(outs[k], m)
        if full:
            assert np.array_equal(got, oracle.unpack(oracle.toeplitz_words(n, m, seeds[k], keys[k]), m)), k
        else:
            assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, seeds[k], keys[k], rows)), k
    if full:
        assert np.array_equal(after, oracle.unpack(oracle.toeplitz_words(n, m, seeds[-1], probe), m))
    else:
        assert np.array_equal(after[rows], oracle.toeplitz_rows(n, m, seeds[-1], probe, rows))


@pytest.mark.parametrize("n,m,off,count,kwargs", [(120_001, 30_000, 77, 9, {}), (1_000_003, 250_000, 5, 4, {}),
                                                   (50_001, 9_000, 3, 6, {"batch_keys": 2})])
def test_hash_fresh_batch_seed_offset_and_workspace(n, m, off, count, kwargs):
    """Fresh seeds at a seed_bit_offset (each row's window starts `off` bits in; the batched seed
    transform reads it through K0's offset), on a large shape (sampled rows) and on a
    workspace-backed handle (one key at a time)."""
    L = n + m - 1
    raw = [syn.random_bits(syn.seed_stream(130 + k), off + L) for k in range(count)]
    win = [oracle.pack(oracle.unpack(r, off + L)[off:], 32) for r in raw]  # the window, re-based
    keys = [syn.random_bits(syn.key_stream(130, k), n) for k in range(count)]
    st, kt = torch.stack([to_dev(r) for r in raw]), torch.stack([to_dev(k) for k in keys])
    ws = None
    opts = dict(kwargs)
    if "batch_keys" in opts:
        nbytes = pa.workspace_size(n, m, route="transform", seed_bit_offset=off, batch_keys=opts["batch_keys"])
        ws = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
        opts["workspace"] = ws
    with pa.Hasher(n, m, st[0], route="transform", seed_bit_offset=off, **opts) as h:
        outs = h.hash_fresh_batch(st, kt)
        torch.cuda.synchronize()
    rows = sample_rows(m, 13, 512)
    for k in range(count):
        got = from_dev(outs[k], m)
        assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, win[k], keys[k], rows)), k


# ---------------------------------------------------------------- Eq. (1) seed converter
@pytest.mark.parametrize("n,m", [(1, 1), (3, 2), (31, 2), (32, 32), (33, 7), (100, 61), (4096, 1024),
                                 (100_003, 9_999)])
def test_seed_from_paper_eq1_matches_oracle(n, m):
    """pa_seed_from_paper_eq1 == the oracle's reading-R2 conversion bit for bit (garbage
    past n+m-1 in the source is not copied), and hashing the converted seed equals the
    paper's literal r = u T with Eq. (1) on small shapes."""
    L = n + m - 1
    rng = np.random.default_rng(n * 7 + m)
    t01 = rng.integers(0, 2, L, dtype=np.uint8)
    tw = oracle.pack(t01, 32)
    tw = np.concatenate([tw, np.full(4, 0xFFFFFFFF, np.uint32)])  # garbage tail words
    if L % 32:
        tw[L // 32] |= np.uint32((0xFFFFFFFF << (L % 32)) & 0xFFFFFFFF)  # garbage bits past L
    t_dev = torch.from_numpy(tw.view(np.int32).copy()).to(DEV)
    s_dev = pa.seed_from_paper_eq1(t_dev, n, m)
    torch.cuda.synchronize()
    got = s_dev.cpu().numpy().view(np.uint32)
    want = oracle.seed_from_eq1(t01, n, m)
    assert np.array_equal(oracle.unpack(got, L), want)
    assert not oracle.unpack(got[: (L + 31) // 32], 32 * ((L + 31) // 32))[L:].any()
    if n * m <= 1 << 14:
        u01 = rng.integers(0, 2, n, dtype=np.uint8)
        with pa.Hasher(n, m, s_dev) as h:
            y = from_dev(h.hash(to_dev(oracle.pack(u01))), m)
        assert np.array_equal(y, oracle.eq1_hash(t01, u01, n, m))


def test_seed_from_paper_eq1_rejects_overlap():
    buf = torch.zeros(64, dtype=torch.int32, device=DEV)
    with pytest.raises(pa.PaError) as e:
        pa.pa_seed_from_paper_eq1(buf.data_ptr(), buf[4:].data_ptr(), 500, 100, 0)
    assert e.value.status == pa.PA_ERR_INVALID_ARG


@pytest.mark.parametrize("n,m,count", [(4096, 1024, 300), (33, 7, 70_000), (20_000, 3_000, 9), (5_000, 5_000, 3)])
def test_bitpacked_batch_native(n, m, count):
    """Route (b) batches on grid.z (chunks of 65535 keys) with strided zeroing; every key vs
    the oracle (sampled keys for the 70k batch)."""
    kw32 = (n + 31) // 32
    stride = (kw32 + 3) // 4 * 4
    sw = syn.random_bits(syn.seed_stream(81), n + m - 1)
    rng = np.random.default_rng(81)
    keys = rng.integers(0, 2**32, (count, stride), dtype=np.uint64).astype(np.uint32)
    with pa.Hasher(n, m, to_dev(sw), route="bitpacked") as h:
        kt = torch.from_numpy(keys.view(np.int32)).to(DEV)
        outs = h.new_out(count)
        outs.fill_(-1)
        h.hash_batch(kt, outs)
        torch.cuda.synchronize()
        got = outs.cpu().numpy().view(np.uint32)
    check_k = range(count) if count <= 300 else np.unique(np.r_[0, 65534, 65535, count - 1,
                                                                 rng.integers(0, count, 50)])
    for k in check_k:
        kk = keys[k].copy()
        want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kk), m)
        assert np.array_equal(oracle.unpack(got[k], m), want), k
        assert not oracle.unpack(got[k][: (m + 31) // 32], 32 * ((m + 31) // 32))[m:].any()


# ---------------------------------------------------------------- full outputs at scale (P11)
@pytest.mark.parametrize("name", ["C3", "C5c", "C4"])
def test_full_output_vs_fft_reference(name):
    """Every output bit at the BASELINE sizes, in the bench's launch configuration, against
    the FP64 pocketfft reference (tests/fft_ref.py, pinned to the direct oracle in
    tests/test_fft_ref.py; its own rounding certificate must be < 0.25)."""
    from fft_ref import fft_window
    n, m, sw, kw = syn.config_inputs(name)
    with pa.Hasher(n, m, to_dev(sw)) as h:
        out = h.hash(to_dev(kw))
        torch.cuda.synchronize()
        got = from_dev(out, m)
        res = h.residual()
    want, cert = fft_window(n, m, sw, kw)
    assert cert < 0.25, cert
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, f"{name}: {bad.size} wrong bits, first {bad[:8]}"
    assert res < 1e-3


# ---------------------------------------------------------------- confirmation digest (NEXT-4)
def test_confirmation_digest():
    """a second, independently seeded Toeplitz hash to 64 bits; equal keys
    confirm, every one of 100 single-bit flips is detected, digest == oracle."""
    from paper_1805_02372_b200.confirm import confirmation_digest, digests_match
    l, tag = 250_000, 64
    key = syn.random_bits(syn.key_stream(95, 0), l)
    tseed = syn.random_bits(syn.seed_stream(95), l + tag - 1)
    ts = to_dev(tseed)
    da = confirmation_digest(to_dev(key), l, ts, tag)
    db = confirmation_digest(to_dev(key.copy()), l, ts, tag)
    assert digests_match(da, db, tag)
    assert np.array_equal(from_dev(da, tag), oracle.unpack(oracle.toeplitz_words(l, tag, tseed, key), tag))
    rng = np.random.default_rng(95)
    kb = key.view(np.uint32).copy()
    missed = 0
    for j in rng.choice(l, 100, replace=False):
        flipped = kb.copy()
        flipped[j // 32] ^= np.uint32(1 << (j % 32))
        if digests_match(da, confirmation_digest(to_dev(flipped.view(np.uint64)), l, ts, tag), tag):
            missed += 1
    assert missed == 0
    with pytest.raises(ValueError):
        confirmation_digest(to_dev(key), l, ts, 32)


# ---------------------------------------------------------------- keys beyond one transform
def test_auto_split_gigabit_key():
    """n ~ 10^9 (the paper's 50-100 km regime): no single transform plans, so
    pa_create splits the key into Eq. (4) column blocks by itself (plain pa_create, default
    options).  Sampled rows vs the oracle for a random key; every output bit vs the all-ones
    closed form y[i] = P[i+n] xor P[i] (P = prefix XOR of the seed)."""
    n, m = 1_000_000_007, 100_000_003
    sw = syn.random_bits(syn.seed_stream(97), n + m - 1)
    kw = syn.random_bits(syn.key_stream(97, 0), n)
    with pa.Hasher(n, m, to_dev(sw)) as h:
        assert h.info["column_blocks"] > 1 and h.route == "transform", h.info
        out = h.hash(to_dev(kw))
        ones = h.hash(to_dev(syn.ones_bits(n)))
        torch.cuda.synchronize()
        assert h.residual() < 1e-3
        got = from_dev(out, m)
        got_ones = from_dev(ones, m)
    rows = sample_rows(m, 97, k=512)
    assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, sw, kw, rows))
    s01 = oracle.unpack(sw, n + m - 1)
    P = np.zeros(n + m, dtype=np.uint8)
    np.bitwise_xor.accumulate(s01, out=P[1:])
    want = P[n:n + m] ^ P[:m]
    bad = np.flatnonzero(got_ones != want)
    assert bad.size == 0, f"{bad.size} wrong bits, first {bad[:8]}"


@pytest.mark.parametrize("n,m", [(400_000_007, 4_000_001), (300_000_011, 30_000_007)])
def test_auto_split_priced_block_length(n, m):
    """Keys just beyond one plan: the automatic Eq. (4) split takes the block length the cost
    model prices cheapest (shorter blocks with the shape-specialised kernels, not the longest
    one-column plans).  Every output bit of the all-ones key against the prefix-XOR closed form,
    sampled rows of a random key against the oracle."""
    sw = syn.random_bits(syn.seed_stream(98), n + m - 1)
    kw = syn.random_bits(syn.key_stream(98, 0), n)
    with pa.Hasher(n, m, to_dev(sw)) as h:
        assert h.info["column_blocks"] > 1 and h.route == "transform", h.info
        got = from_dev(h.hash(to_dev(kw)), m)
        got_ones = from_dev(h.hash(to_dev(syn.ones_bits(n))), m)
        torch.cuda.synchronize()
        assert h.residual() < 1e-3
    rows = sample_rows(m, 98, k=384)
    assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, sw, kw, rows))
    s01 = oracle.unpack(sw, n + m - 1)
    P = np.zeros(n + m, dtype=np.uint8)
    np.bitwise_xor.accumulate(s01, out=P[1:])
    assert np.array_equal(got_ones, P[n:n + m] ^ P[:m])


def test_key_and_output_must_not_overlap():
    n, m = 1_000_003, 250_000
    with pa.Hasher(n, m, to_dev(syn.random_bits(syn.seed_stream(99), n + m - 1))) as h:
        buf = torch.zeros(pa.words32(n) + 64, dtype=torch.int32, device=DEV)
        with pytest.raises(pa.PaError) as e:
            pa.pa_hash(h.handle, buf.data_ptr(), buf[16:].data_ptr(), 0)
        assert e.value.status == pa.PA_ERR_INVALID_ARG and "overlap" in pa.pa_last_error()
        keys = torch.zeros((4, (pa.words32(n) + 3) // 4 * 4), dtype=torch.int32, device=DEV)
        with pytest.raises(pa.PaError):
            pa.pa_hash_batch(h.handle, keys.data_ptr(), keys.shape[1], keys[1].data_ptr(), keys.shape[1], 2, 0)



def _path_cases(count=24, seed=4242):
    rng = np.random.default_rng(seed)
    cases = []
    for i in range(count):
        kind = ["fresh", "batch", "blocked", "blocked_host"][i % 4]
        n = int(np.exp(rng.uniform(np.log(2e4), np.log(3e6))))
        m = max(1, int(n * rng.uniform(0.02, 0.9)))
        cases.append((kind, n, m, int(rng.integers(2, 6)), int(rng.integers(0, 3))))
    return cases


@pytest.mark.parametrize("kind,n,m,count,variant", _path_cases())
def test_random_paths_fuzz(kind, n, m, count, variant):
    """Seeded random shapes through the batched, fresh-seed (fused K2 + the handle's last seed
    afterwards) and blocked (device / host-streamed, random block limits and budgets) paths;
    sampled rows (both ends + random) against the oracle."""
    L = n + m - 1
    rows = sample_rows(m, n % 1000, k=96)
    if kind in ("fresh", "batch"):
        seeds = [syn.random_bits(syn.seed_stream(300 + k), L) for k in range(count)]
        keys = [syn.random_bits(syn.key_stream(300, k), n) for k in range(count)]
        kt = torch.stack([to_dev(k) for k in keys])
        with pa.Hasher(n, m, to_dev(seeds[0]), route="transform") as h:
            if kind == "fresh":
                outs = h.hash_fresh_batch(torch.stack([to_dev(s) for s in seeds]), kt)
                after = from_dev(h.hash(to_dev(keys[0])), m)
            else:
                outs = h.hash_batch(kt)
            torch.cuda.synchronize()
        for k in range(count):
            sk = seeds[k] if kind == "fresh" else seeds[0]
            assert np.array_equal(from_dev(outs[k], m)[rows], oracle.toeplitz_rows(n, m, sk, keys[k], rows)), k
        if kind == "fresh":
            assert np.array_equal(after[rows], oracle.toeplitz_rows(n, m, seeds[-1], keys[0], rows))
        return
    sw = syn.random_bits(syn.seed_stream(301), L)
    kw = syn.random_bits(syn.key_stream(301, 0), n)
    lim = [0, max(n // 3 + m, 4096), max(m + 64, (n + m) // 5)][variant]
    if kind == "blocked":
        sd, kd = to_dev(sw), to_dev(kw)
        out = torch.zeros(pa.words32(m) + 4, dtype=torch.int32, device=DEV)
        pa.pa_hash_blocked(n, m, sd.data_ptr(), kd.data_ptr(), out.data_ptr(), lim, 0)
        got = from_dev(out, m)
    else:
        sh = torch.from_numpy(np.ascontiguousarray(sw).view(np.int32).copy()).pin_memory()
        kh = torch.from_numpy(np.ascontiguousarray(kw).view(np.int32).copy()).pin_memory()
        oh = torch.zeros(pa.words32(m), dtype=torch.int32).pin_memory()
        pa.pa_hash_blocked_host(n, m, sh.data_ptr(), kh.data_ptr(), oh.data_ptr(), lim, [0, 256 << 20, 1 << 30][variant], 0)
        got = oracle.unpack(oh.numpy().view(np.uint32), m)
    assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, sw, kw, rows))


def _fuzz_shapes(count=48, seed=1805):
    rng = np.random.default_rng(seed)
    shapes = []
    for _ in range(count):
        n = int(np.exp(rng.uniform(0, np.log(3e6))))
        m = int(rng.integers(1, n + 1)) if rng.random() < 0.8 else max(1, n // int(rng.integers(100, 5000)))
        shapes.append((n, m))
    return shapes


@pytest.mark.parametrize("n,m", _fuzz_shapes())
def test_random_shapes_fuzz(n, m):
    """Seeded random (n, m) across every planner regime (route choice, smooth lengths, N1 x N2
    splits, column-group widths, direct K1 gather), both routes where route (b) is affordable;
    full outputs or sampled rows vs the oracle."""
    sw = syn.random_bits(syn.seed_stream(n % 1000 + 7), n + m - 1)
    kw = syn.random_bits(syn.key_stream(m % 1000 + 7, 0), n)
    got, info = check(n, m, sw, kw, "transform")
    if n * m <= 2e9:
        got_b, _ = check(n, m, sw, kw, "bitpacked", full=False)
        assert np.array_equal(got, got_b)


def test_no_device_memory_leak_across_handles():
    """200 create / hash / destroy cycles over both routes, split, workspace-backed and host-path
    handles return device memory to its starting level (libpa cudaMallocs are all freed)."""
    shapes = [(4096, 1024, {}), (1_000_003, 250_000, {}), (300_007, 60_001, {"max_transform_len": 200_000}),
              (65_537, 6_553, {"route": "bitpacked"})]
    inputs = [(to_dev(syn.random_bits(syn.seed_stream(110 + i), n + m - 1)),
               to_dev(syn.random_bits(syn.key_stream(110, i), n))) for i, (n, m, _) in enumerate(shapes)]
    kh = torch.zeros(pa.words32(1_000_003), dtype=torch.int32).pin_memory()
    oh = torch.zeros(pa.words32(250_000), dtype=torch.int32).pin_memory()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for it in range(50):
        for i, (n, m, opts) in enumerate(shapes):
            with pa.Hasher(n, m, inputs[i][0], **opts) as h:
                h.hash(inputs[i][1])
                if n == 1_000_003:
                    h.hash_host(kh, oh)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 <= (4 << 20), (free0, free1)


def test_concurrent_handles_on_streams():
    """Independent handles on separate streams, interleaved, each bit-exact (one hash in flight
    per handle, several handles in flight at once)."""
    cases = [(1_000_003, 250_000), (300_007, 30_001), (4096, 1024), (2_000_001, 200_000)]
    hs, keys, outs, streams, wants = [], [], [], [], []
    for i, (n, m) in enumerate(cases):
        sw = syn.random_bits(syn.seed_stream(120 + i), n + m - 1)
        kw = syn.random_bits(syn.key_stream(120, i), n)
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            h = pa.Hasher(n, m, to_dev(sw), stream=s)
        hs.append(h)
        keys.append(to_dev(kw))
        outs.append(h.new_out())
        streams.append(s)
        wants.append(oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m) if n * m <= 5e11 else None)
    torch.cuda.synchronize()
    for rep in range(5):
        for h, k, o, s in zip(hs, keys, outs, streams):
            h.hash(k, o, stream=s)
    torch.cuda.synchronize()
    for (n, m), h, o, w in zip(cases, hs, outs, wants):
        assert np.array_equal(from_dev(o, m), w), (n, m)
        h.close()


# ---------------------------------------------------------------- fault injection (SURVEY aux table)
def test_fault_injection_flipped_output_bit_is_detected():
    """The parity check is sensitive: one flipped output bit is reported at exactly its row."""
    n, m = 1_000_003, 250_000
    sw = syn.random_bits(syn.seed_stream(130), n + m - 1)
    kw = syn.random_bits(syn.key_stream(130, 0), n)
    with pa.Hasher(n, m, to_dev(sw)) as h:
        out = h.hash(to_dev(kw))
        torch.cuda.synchronize()
    words = out.cpu().numpy().view(np.uint32).copy()
    i = 123_457
    words[i // 32] ^= np.uint32(1 << (i % 32))
    want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
    bad = np.flatnonzero(oracle.unpack(words, m) != want)
    assert list(bad) == [i]


def test_fault_injection_corrupted_spectrum_trips_precision():
    """The FP64 tripwire: scribbling over a handle's seed spectrum (reachable here because the
    workspace is the caller's: spectrum first after the staging block) makes the window values
    non-integers, and pa_residual reports PA_ERR_PRECISION."""
    n, m = 1_000_003, 250_000
    al = lambda b: (b + 255) // 256 * 256  # noqa: E731
    need = pa.workspace_size(n, m, route="transform")
    ws = torch.zeros(need, dtype=torch.uint8, device=DEV)
    seed_t = to_dev(syn.random_bits(syn.seed_stream(131), n + m - 1))
    with pa.Hasher(n, m, seed_t, route="transform", workspace=ws) as h:
        key = to_dev(syn.random_bits(syn.key_stream(131, 0), n))
        h.hash(key)
        assert h.residual() < 1e-3
        stage = al(4 * pa.words32(n)) + al(4 * pa.words32(m))
        M = h.info["transform_len"] // 2
        spec = ws[stage:stage + 16 * M].view(torch.float64)
        spec.copy_(torch.rand(spec.numel(), dtype=torch.float64, device=DEV) * 1e-6)
        h.hash(key)
        with pytest.raises(pa.PaError) as e:
            h.residual()
        assert e.value.status == pa.PA_ERR_PRECISION and "residual" in pa.pa_last_error()


def test_gigabit_under_2gib_budget_and_plan_consistency():
    """SPEC acceptance criterion 7: a 1 Gbit input (2^30 key bits, m = n/10) amplifies
    under a 2 GiB device-memory budget via the planner (pa_hash_blocked: row x column blocks of
    <= 9e7 bits, one handle alive at a time; peak use sampled through NVML, inputs included),
    sampled rows vs the oracle; and a 64 Mbit prefix hashed through two different plans agrees
    with the single-transform hash."""
    import threading
    import pynvml
    n = 1 << 30
    m = n // 10
    sw = syn.random_bits(syn.seed_stream(140), n + m - 1)
    kw = syn.random_bits(syn.key_stream(140, 0), n)
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    base = pynvml.nvmlDeviceGetMemoryInfo(hnd).used
    peak = [base]
    stop = threading.Event()

    def sample():
        while not stop.is_set():
            peak[0] = max(peak[0], pynvml.nvmlDeviceGetMemoryInfo(hnd).used)
            stop.wait(0.0005)
    th = threading.Thread(target=sample)
    th.start()
    try:
        seed_t, key_t = to_dev(sw), to_dev(kw)
        out = torch.zeros(pa.words32(m) + 4, dtype=torch.int32, device=DEV)
        pa.pa_hash_blocked(n, m, seed_t.data_ptr(), key_t.data_ptr(), out.data_ptr(), 90_000_000, 0)
        torch.cuda.synchronize()
    finally:
        stop.set()
        th.join()
    used = peak[0] - base
    assert used <= 2 * 2**30, f"peak device memory {used / 2**30:.2f} GiB"
    rows = sample_rows(m, 140, k=256)
    assert np.array_equal(from_dev(out, m)[rows], oracle.toeplitz_rows(n, m, sw, kw, rows))
    del seed_t, key_t, out
    # 64 Mbit prefix: the same data and seed through two plans and one transform
    n2 = 1 << 26
    m2 = n2 // 10
    sw2, kw2 = sw[: (n2 + m2 - 1 + 63) // 64], kw[: n2 // 64]
    seed2, key2 = to_dev(sw2), to_dev(kw2)
    outs = []
    for lim in (20_000_000, 7_000_001):
        o = torch.zeros(pa.words32(m2) + 4, dtype=torch.int32, device=DEV)
        pa.pa_hash_blocked(n2, m2, seed2.data_ptr(), key2.data_ptr(), o.data_ptr(), lim, 0)
        outs.append(from_dev(o, m2))
    with pa.Hasher(n2, m2, seed2) as h:
        outs.append(from_dev(h.hash(key2), m2))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    pa.pa_hash_blocked_release()


@pytest.mark.parametrize("n,m,count,kwargs", [(1_048_576, 104_857, 64, {}), (4096, 1024, 500, {}),
                                              (300_007, 60_001, 5, {"max_transform_len": 200_000}),
                                              (1_048_576, 104_857, 150, {}),
                                              (300_007, 60_001, 133, {"max_transform_len": 200_000}),
                                              (4096, 1024, 9000, {})])
def test_hash_host_batch(n, m, count, kwargs):
    """pa_hash_host_batch: pinned host keys (strided rows) -> chunks of keys pipelined through two
    staging slots (H2D / hash / D2H overlapped; several chunks with a ragged last one for the
    larger counts); every output vs the oracle (sampled above 64 keys), tail bits zero, and
    nothing written past each output row."""
    sw = syn.random_bits(syn.seed_stream(150), n + m - 1)
    kw32 = pa.words32(n)
    rng = np.random.default_rng(150)
    keys = rng.integers(0, 2**32, (count, kw32 + 3), dtype=np.uint64).astype(np.uint32)
    kh = torch.from_numpy(keys.view(np.int32)).pin_memory()
    oh = torch.full((count, pa.words32(m) + 5), -1, dtype=torch.int32).pin_memory()
    with pa.Hasher(n, m, to_dev(sw), **kwargs) as h:
        h.hash_host_batch(kh, oh)
    got = oh.numpy().view(np.uint32)
    check_k = range(count) if count <= 64 else np.unique(np.r_[0, count - 1, rng.integers(0, count, 40)])
    for k in check_k:
        want = oracle.unpack(oracle.toeplitz_words(n, m, sw, keys[k, :kw32].copy()), m)
        assert np.array_equal(oracle.unpack(got[k], m), want), k
        assert not oracle.unpack(got[k][: pa.words32(m)], 32 * pa.words32(m))[m:].any()
    assert (oh[:, pa.words32(m):] == -1).all()


def test_host_graph_recaptured_after_work_buffers_move():
    """pa_hash_host caches a CUDA graph holding the work-buffer pointers.  A fresh-seed batch
    (count >= 2) regrows those buffers (stream-ordered, the old block freed once the stream
    passes it); the next pa_hash_host on the same host buffers must re-capture, not replay stale
    pointers.  Every output is checked against the oracle."""
    n, m = 1_000_003, 250_000
    sw = syn.random_bits(syn.seed_stream(131), n + m - 1)
    kw = syn.random_bits(syn.key_stream(131, 0), n)
    key_h = torch.from_numpy(np.ascontiguousarray(kw).view(np.int32).copy()).pin_memory()
    out_h = torch.zeros(pa.words32(m), dtype=torch.int32).pin_memory()
    want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
    count = 4
    seeds = syn.random_bits_torch([syn.seed_stream(140 + k) for k in range(count)], n + m - 1, DEV)
    keys = syn.random_bits_torch([syn.key_stream(141, k) for k in range(count)], n, DEV)
    with pa.Hasher(n, m, to_dev(sw)) as h:
        h.hash_host(key_h, out_h)
        assert np.array_equal(oracle.unpack(out_h.numpy().view(np.uint32), m), want)
        outs = h.hash_fresh_batch(seeds, keys)
        h.set_seed(to_dev(sw))
        out_h.zero_()
        h.hash_host(key_h, out_h)
        assert np.array_equal(oracle.unpack(out_h.numpy().view(np.uint32), m), want)
        for k in (0, count - 1):
            s_k = syn.random_bits(syn.seed_stream(140 + k), n + m - 1)
            k_k = syn.random_bits(syn.key_stream(141, k), n)
            rows = sample_rows(m, k, 256)
            assert np.array_equal(from_dev(outs[k], m)[rows], oracle.toeplitz_rows(n, m, s_k, k_k, rows))
        # a larger plain batch moves them again
        big = h.hash_batch(syn.random_bits_torch([syn.key_stream(142, k) for k in range(8)], n, DEV))
        out_h.zero_()
        h.hash_host_async(key_h, out_h)
        torch.cuda.synchronize()
        assert np.array_equal(oracle.unpack(out_h.numpy().view(np.uint32), m), want)
        k7 = syn.random_bits(syn.key_stream(142, 7), n)
        rows = sample_rows(m, 7, 256)
        assert np.array_equal(from_dev(big[7], m)[rows], oracle.toeplitz_rows(n, m, sw, k7, rows))


def test_fresh_batch_rejects_overlapping_outputs():
    n, m = 100_003, 20_000
    with pa.Hasher(n, m, to_dev(syn.random_bits(syn.seed_stream(150), n + m - 1))) as h:
        W = (pa.words32(n + m) + 3) // 4 * 4
        buf = torch.zeros((4, W), dtype=torch.int32, device=DEV)
        for outs_p in (buf[0, 8:].data_ptr(), buf[2, 8:].data_ptr()):  # inside the seed / the key
            with pytest.raises(pa.PaError) as e:
                pa.pa_hash_fresh_batch(h.handle, buf[0].data_ptr(), W, buf[2].data_ptr(), W, outs_p, W, 1, 0)
            assert e.value.status == pa.PA_ERR_INVALID_ARG and "overlap" in pa.pa_last_error()


def test_explicit_device_option():
    """pa_options.device: an explicit ordinal binds the handle to that device and
    later calls run there; an ordinal past the visible devices is rejected."""
    n, m = 4096, 1024
    sw = syn.random_bits(syn.seed_stream(151), n + m - 1)
    kw = syn.random_bits(syn.key_stream(151, 0), n)
    seed_t, key_t = to_dev(sw), to_dev(kw)
    o = pa.make_options(route="transform", device=0)
    h = pa.pa_create_ex(n, m, seed_t.data_ptr(), o, 0)
    try:
        assert pa.pa_get_info(h)["device"] == 0
        out = torch.zeros(pa.words32(m) + 3, dtype=torch.int32, device=DEV)
        pa.pa_hash(h, key_t.data_ptr(), out.data_ptr(), 0)
        torch.cuda.synchronize()
        assert np.array_equal(from_dev(out, m), oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m))
    finally:
        pa.pa_destroy(h)
    o.device = torch.cuda.device_count()
    with pytest.raises(pa.PaError) as e:
        pa.pa_create_ex(n, m, seed_t.data_ptr(), o, 0)
    assert e.value.status == pa.PA_ERR_INVALID_ARG and "device" in pa.pa_last_error()


@pytest.mark.parametrize("n,m,maxb,pinned", [(20_000, 7_000, 5_000, True), (50_001, 20_000, 16_384, False),
                                             (3001, 3000, 700, True), (100_000, 10_000, 0, True),
                                             (1_000_003, 250_000, 300_001, True)])
def test_length_compatible_blocked_host(n, m, maxb, pinned):
    """pa_hash_blocked_host: seed, key and output in host memory (pinned or
    pageable), row x column blocks streamed through two staging slots, Eq. (7) XOR merge -- the
    full output equals the oracle's, and nothing is written past ceil(m/32) words."""
    sw = syn.random_bits(syn.seed_stream(93 + n), n + m - 1)
    kw = syn.random_bits(syn.key_stream(93, n), n)
    seed_h = torch.from_numpy(np.ascontiguousarray(sw).view(np.int32).copy())
    key_h = torch.from_numpy(np.ascontiguousarray(kw).view(np.int32).copy())
    out_h = torch.full((pa.words32(m) + 3,), -1, dtype=torch.int32)
    if pinned:
        seed_h, key_h, out_h = seed_h.pin_memory(), key_h.pin_memory(), out_h.pin_memory()
    pa.pa_hash_blocked_host(n, m, seed_h.data_ptr(), key_h.data_ptr(), out_h.data_ptr(), maxb, 0, 0)
    want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
    allb = oracle.unpack(out_h.numpy()[: pa.words32(m)].view(np.uint32), 32 * pa.words32(m))
    assert np.array_equal(allb[:m], want)
    assert not allb[m:].any()
    assert (out_h.numpy()[pa.words32(m):] == -1).all()


def test_blocked_host_4gbit_under_16gib_budget():
    """NEXT-3 at the paper's scale: n = 4*10^9 key bits and the seed stay in pinned
    host memory; pa_hash_blocked_host streams them through a 16 GiB device budget (peak device
    use sampled with NVML).  Random key: 64 sampled rows vs the oracle.  All-ones key: every
    output bit against the closed form y[i] = parity(s[i .. i+n-1]) (y[i+1] = y[i] ^ s[i] ^
    s[i+n]), computed from the seed alone."""
    import threading
    import pynvml
    n, m = 4 * 10**9, 10**7
    budget = 16 * 2**30
    sw = syn.random_bits(syn.seed_stream(160), n + m - 1)
    kw = syn.random_bits(syn.key_stream(160, 0), n)
    seed_h = torch.from_numpy(sw.view(np.int32)).pin_memory()
    key_h = torch.from_numpy(kw.view(np.int32)).pin_memory()
    out_h = torch.zeros(pa.words32(m), dtype=torch.int32).pin_memory()
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    base = pynvml.nvmlDeviceGetMemoryInfo(hnd).used
    peak = [base]
    stop = threading.Event()

    def sample():
        while not stop.is_set():
            peak[0] = max(peak[0], pynvml.nvmlDeviceGetMemoryInfo(hnd).used)
            stop.wait(0.0005)
    th = threading.Thread(target=sample)
    th.start()
    try:
        pa.pa_hash_blocked_host(n, m, seed_h.data_ptr(), key_h.data_ptr(), out_h.data_ptr(), 0, budget, 0)
        got = oracle.unpack(out_h.numpy().view(np.uint32), m)
        ones_h = torch.from_numpy(syn.ones_bits(n).view(np.int32)).pin_memory()
        pa.pa_hash_blocked_host(n, m, seed_h.data_ptr(), ones_h.data_ptr(), out_h.data_ptr(), 0, budget, 0)
        got_ones = oracle.unpack(out_h.numpy().view(np.uint32), m)
    finally:
        stop.set()
        th.join()
    pa.pa_hash_blocked_release()
    assert peak[0] - base <= budget, f"peak device memory {(peak[0] - base) / 2**30:.2f} GiB"
    rows = sample_rows(m, 160, k=32)[:64]
    assert np.array_equal(got[rows], oracle.toeplitz_rows(n, m, sw, kw, rows))
    assert n % 64 == 0  # parity of s[0..n): the popcount parity of the XOR of its words
    y0 = bin(int(np.bitwise_xor.reduce(sw[: n // 64]))).count("1") & 1
    lo = np.unpackbits(sw[: (m + 63) // 64].view(np.uint8), bitorder="little")
    hi = np.unpackbits(sw[n // 64: (n + m + 63) // 64].view(np.uint8), bitorder="little")
    d = np.bitwise_xor(lo[: m - 1], hi[: m - 1])
    want = np.concatenate([[y0], np.bitwise_xor.accumulate(d) ^ y0]).astype(np.uint8)
    assert np.array_equal(got_ones, want)


@pytest.mark.parametrize("n,m", [(1_067_928, 266_982), (300_007, 60_001), (1_000_003, 250_000)])
def test_measured_planning(n, m):
    """PA_PLAN_MEASURE: the planner's best candidates are built and timed at create and the
    fastest kept (remembered per shape): the hash stays bit-exact against the oracle, the plan is
    a valid split of a transform >= n + m - 1, and a second handle of the shape reuses it."""
    import time
    sw = syn.random_bits(syn.seed_stream(181), n + m - 1)
    kw = syn.random_bits(syn.key_stream(181, 0), n)
    seed = to_dev(sw)
    with pa.Hasher(n, m, seed, route="transform", plan="measure") as h:
        info = h.info
        got = from_dev(h.hash(to_dev(kw)), m)
        torch.cuda.synchronize()
        assert h.residual() < 1e-3
    assert info["transform_len"] >= n + m - 1 and info["n1"] * info["n2"] * 2 == info["transform_len"]
    assert np.array_equal(got, oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m))
    t0 = time.perf_counter()
    with pa.Hasher(n, m, seed, route="transform", plan="measure") as h2:
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        assert (h2.info["n1"], h2.info["n2"], h2.info["cols_per_cta"]) == (info["n1"], info["n2"],
                                                                          info["cols_per_cta"])
    assert dt < 0.5  # remembered: no second round of trial handles
