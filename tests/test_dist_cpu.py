"""Multi-process (gloo, world_size 2 and 3, CPU) tests of the multi-GPU split logic in
paper_1805_02372_b200.dist: row split + all-gather, column split + XOR merge, and
independent-key dealing reassemble exactly the single-device hash.  The per-rank
hash is injected (the CPU oracle) -- this tests the partition arithmetic and the
collectives, the GPU kernels are covered by tests/test_parity_gpu.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import pa_synth as syn


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def oracle_hash(n, m, seed_t, seed_off, key_t):
    """hash_fn with libpa's calling convention, computed by the oracle on the CPU."""
    from paper_1805_02372_b200.dist import extract_bits
    sw = extract_bits(seed_t.numpy().view(np.uint32), seed_off, n + m - 1)
    kw = extract_bits(key_t.numpy().view(np.uint32), 0, n)
    y = oracle.toeplitz_words(n, m, sw, kw)
    w = (m + 31) // 32
    return torch.from_numpy(y.view(np.int32)[:w].copy())


def _worker(rank, world, port, n, m, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1805_02372_b200 import dist as pd
        sw = syn.random_bits(syn.seed_stream(77), n + m - 1)
        kw = syn.random_bits(syn.key_stream(77, 0), n)
        seed_t = torch.from_numpy(sw.view(np.int32).copy())
        key_t = torch.from_numpy(kw.view(np.int32).copy())
        rows = pd.hash_rows(n, m, seed_t, key_t, hash_fn=oracle_hash)
        cols = pd.hash_cols(n, m, seed_t, kw, hash_fn=oracle_hash, device=torch.device("cpu"))
        keys = torch.stack([torch.from_numpy(syn.random_bits(syn.key_stream(78, k), n).view(np.int32).copy())
                            for k in range(5)])
        idx, outs = pd.hash_keys(n, m, seed_t, keys, hash_fn=oracle_hash)
        # persistent splitters with per-step source-rank distribution (rank 0 holds the key):
        # row split broadcasts the key, column split scatters 128-bit-aligned key blocks
        src_key = key_t.clone() if rank == 0 else torch.zeros_like(key_t)
        rs = pd.RowSplit(n, m, seed_t, hash_fn=oracle_hash)
        rows2 = rs(src_key, src=0).clone()
        rows3 = rs(src_key, src=0).clone()  # a second step reuses the handles and buffers
        cs = pd.ColSplit(n, m, seed_t, hash_fn=oracle_hash, xor_fn=pd._xor_fold_host)
        cols2 = cs(cs.scatter_key(key_t if rank == 0 else None, src=0)).clone()
        auto_split, auto = pd.hash(n, m, seed_t, key_t if rank == 0 else torch.zeros_like(key_t),
                                   hash_fn=oracle_hash, xor_fn=pd._xor_fold_host)
        forced = {s: pd.hash(n, m, seed_t, key_t if rank == 0 else torch.zeros_like(key_t), split=s,
                             hash_fn=oracle_hash, xor_fn=pd._xor_fold_host)[1].numpy().copy()
                  for s in ("rows", "cols")}
        q.put((rank, rows.numpy().copy(), cols.numpy().copy(), idx, outs.numpy().copy(),
               [rows2.numpy().copy(), rows3.numpy().copy(), cols2.numpy().copy(), auto.numpy().copy(),
                forced["rows"], forced["cols"]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,m", [(2, 3001, 700), (2, 4096, 1024), (3, 2000, 1500), (3, 1000, 999),
                                        (2, 300, 999)])
def test_splits_reassemble(world, n, m):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sw = syn.random_bits(syn.seed_stream(77), n + m - 1)
    kw = syn.random_bits(syn.key_stream(77, 0), n)
    want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
    for rank, rows, cols, idx, outs, more in res:
        assert np.array_equal(oracle.unpack(rows.view(np.uint32), m), want), ("rows", rank)
        assert np.array_equal(oracle.unpack(cols.view(np.uint32), m), want), ("cols", rank)
        for j, y in enumerate(more):
            assert np.array_equal(oracle.unpack(y.view(np.uint32), m), want), ("splitter", j, rank)
        for i, k in enumerate(idx):
            wk = oracle.unpack(oracle.toeplitz_words(n, m, sw, syn.random_bits(syn.key_stream(78, k), n)), m)
            assert np.array_equal(oracle.unpack(outs[i].view(np.uint32), m), wk), ("keys", rank, k)
    dealt = sorted(k for r in res for k in r[3])
    assert dealt == list(range(5))


def test_range_helpers():
    from paper_1805_02372_b200 import dist as pd
    for m in (1, 31, 32, 33, 1000, 20_000_000):
        for w in (1, 2, 3, 8):
            rr = pd.row_ranges(m, w)
            assert rr[0][0] == 0 and rr[-1][1] == m
            assert all(a % 32 == 0 or a == b == m for a, b in rr)
            assert all(rr[i][1] == rr[i + 1][0] for i in range(w - 1))
    cr = pd.col_ranges(10, 3, 4)
    assert cr[0][0] == 0 and cr[-1][1] == 10 and sum(b - a for a, b in cr) == 10
    for n in (1, 127, 128, 129, 3001, 10**8):
        for w in (1, 2, 3, 8):
            cr = pd.col_ranges(n, 7, w)
            assert cr[0][0] == 0 and cr[-1][1] == n
            assert all(a % 128 == 0 or a == n for a, _ in cr)
            assert all(cr[i][1] == cr[i + 1][0] for i in range(w - 1))
    assert pd.col_seed_offset(100, 20, 50) == 50


def _corrupt_worker(rank, world, port, n, m, q):
    """Column split whose rank-1 partial has one flipped bit (SPEC S:475 corrupted-merge hook)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1805_02372_b200 import dist as pd
        sw = syn.random_bits(syn.seed_stream(79), n + m - 1)
        kw = syn.random_bits(syn.key_stream(79, 0), n)
        seed_t = torch.from_numpy(sw.view(np.int32).copy())

        def corrupt(nn, mm, s, off, k):
            out = oracle_hash(nn, mm, s, off, k)
            if rank == 1:
                out[7] ^= 1 << 3  # bit 7 * 32 + 3 of this rank's partial
            return out
        cols = pd.hash_cols(n, m, seed_t, kw, hash_fn=corrupt, device=torch.device("cpu"))
        q.put((rank, cols.numpy().copy()))
    finally:
        dist.destroy_process_group()


def test_corrupted_merge_is_detected_at_its_bit():
    """Fault injection into the Eq. (7) merge: the merged output differs from the oracle at
    exactly the corrupted bit, on every rank (the XOR merge uses every partial)."""
    world, n, m = 2, 3001, 700
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_corrupt_worker, args=(r, world, port, n, m, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sw = syn.random_bits(syn.seed_stream(79), n + m - 1)
    kw = syn.random_bits(syn.key_stream(79, 0), n)
    want = oracle.unpack(oracle.toeplitz_words(n, m, sw, kw), m)
    for rank, cols in res:
        bad = np.flatnonzero(oracle.unpack(cols.view(np.uint32), m) != want)
        assert list(bad) == [7 * 32 + 3], (rank, bad[:5])


def test_choose_split_cost_model():
    """the row split barely shrinks each GPU's transform (n + m/G), the column split
    does (n/G + m); at C4 (m/n = 0.2) the columns win for G >= 2, and one GPU never splits."""
    from paper_1805_02372_b200 import dist as pd
    assert pd.choose_split(10**8, 2 * 10**7, 1) == "rows"
    for g in (2, 4, 8):
        assert pd.choose_split(10**8, 2 * 10**7, g) == "cols"
    # m close to n: the column split would leave each GPU ~m points -> rows
    assert pd.choose_split(10**7, 10**7, 8) == "rows"
    # tiny keys: latency of the extra collective dominates -> rows
    assert pd.choose_split(4096, 1024, 8) == "rows"


def test_bench_gpus2_spawns_ranks_cpu_selftest():
    """`bench.py --gpus N` without a torchrun environment re-executes itself under
    torch.distributed.run; --selftest-cpu drives the rank plumbing over gloo (row split with key
    broadcast, column split with key scatter + XOR merge) with the oracle as the per-rank hash."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--selftest-cpu"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([s for s in r.stdout.splitlines() if s.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["rows_split_ok"] and line["cols_split_ok"]
    assert line["choose_split_C4"] == "cols"
