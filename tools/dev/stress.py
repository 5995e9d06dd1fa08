"""Randomised parity stress against the oracle (developer tool, not a test): for T seconds, random
(n, m) through pa_hash_fresh_batch (+ the handle's last seed afterwards), pa_hash_batch,
pa_hash_blocked and pa_hash_blocked_host (random block limits and device budgets), sampled rows
(both ends + random) vs oracle.toeplitz_rows.

    python tools/dev/stress.py SEED SECONDS
"""
import sys, os, time, torch, numpy as np
sys.path.insert(0, os.getcwd())
import pa_synth as syn, oracle
import paper_1805_02372_b200 as pa
rng = np.random.default_rng(int(sys.argv[1])); T = float(sys.argv[2])
def words(w):
    w = np.ascontiguousarray(w).view(np.int32); w = np.concatenate([w, np.zeros((-w.size) % 4, np.int32)])
    return torch.from_numpy(w.copy()).cuda()
t0 = time.time(); bad = 0; cnt = 0; kinds = {}
while time.time() - t0 < T:
    kind = rng.choice(["fresh", "batch", "blocked", "blocked_host"], p=[0.4, 0.3, 0.2, 0.1])
    if kind.startswith("blocked"):
        n = int(np.exp(rng.uniform(np.log(2e4), np.log(3e6)))); m = max(1, int(n * rng.uniform(0.05, 1.0)))
    else:
        n = int(np.exp(rng.uniform(np.log(3e5), np.log(6e7)))); m = max(1, int(n * rng.uniform(0.02, 0.5)))
    count = int(rng.choice([2, 3, 4, 7])) if kind in ("fresh", "batch") else 1
    sw = syn.random_bits(syn.seed_stream(9000 + cnt), n + m - 1)
    seeds = [syn.random_bits(syn.seed_stream(9500 + cnt * 8 + k), n + m - 1) for k in range(count)]
    keys = [syn.random_bits(syn.key_stream(9000 + cnt, k), n) for k in range(count)]
    rows = np.unique(np.concatenate([np.arange(min(m, 48)), np.arange(max(0, m - 48), m), rng.integers(0, m, 48)])).astype(np.uint64)
    outs = []; lim = None
    if kind in ("fresh", "batch"):
        kt = torch.stack([words(k) for k in keys])
        with pa.Hasher(n, m, words(sw), route="transform") as h:
            o = h.hash_fresh_batch(torch.stack([words(s) for s in seeds]), kt) if kind == "fresh" else h.hash_batch(kt)
            o = o.cpu().numpy()
            after = None
            if kind == "fresh":
                after = oracle.unpack(h.hash(words(keys[0])).cpu().numpy().view(np.uint32), m)
        for k in range(count):
            outs.append((seeds[k] if kind == "fresh" else sw, keys[k], oracle.unpack(o[k].view(np.uint32), m)))
        if after is not None:
            outs.append((seeds[-1], keys[0], after))
    else:
        lim = int(rng.choice([0, max(n // 3 + m, 4096), max(m + 64, (n + m) // 5)]))
        out = torch.zeros(pa.words32(m) + 4, dtype=torch.int32, device="cuda")
        if kind == "blocked":
            sd, kd = words(sw), words(keys[0])  # keep the tensors alive across the async call
            pa.pa_hash_blocked(n, m, sd.data_ptr(), kd.data_ptr(), out.data_ptr(), lim, 0)
            torch.cuda.synchronize(); o = out.cpu().numpy()
        else:
            sh = torch.from_numpy(np.ascontiguousarray(sw).view(np.int32).copy()).pin_memory()
            kh = torch.from_numpy(np.ascontiguousarray(keys[0]).view(np.int32).copy()).pin_memory()
            oh = torch.zeros(pa.words32(m), dtype=torch.int32).pin_memory()
            budget = int(rng.choice([0, 64 << 20, 256 << 20]))
            try:
                pa.pa_hash_blocked_host(n, m, sh.data_ptr(), kh.data_ptr(), oh.data_ptr(), lim, budget, 0)
            except pa.PaError as e:
                kinds["nomem"] = kinds.get("nomem", 0) + 1; cnt += 1; continue
            o = oh.numpy()
        outs.append((sw, keys[0], oracle.unpack(o.view(np.uint32), m)))
    for s_, k_, got in outs:
        want = oracle.toeplitz_rows(n, m, s_, k_, rows)
        if not np.array_equal(got[rows.astype(np.int64)], want):
            bad += 1; print("MISMATCH", kind, n, m, count, lim if kind.startswith("blocked") else "", flush=True)
    kinds[kind] = kinds.get(kind, 0) + 1
    cnt += 1
pa.pa_hash_blocked_release()
print(f"stress2: {cnt} cases {kinds}, {bad} mismatches, {time.time()-t0:.0f}s")
