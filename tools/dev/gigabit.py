"""Length-compatible regime: one pa_create / pa_hash at n ~ 1e9 .. 1e10 (auto column split)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import pa_synth as syn, paper_1805_02372_b200 as pa
def dw(w): return torch.from_numpy(np.ascontiguousarray(w).view(np.int32).copy()).cuda()
for n, m in [(10**9, 10**8), (4 * 10**9, 10**7)]:
    sw = syn.random_bits(syn.seed_stream(6), n + m - 1)
    kw = syn.random_bits(syn.key_stream(6, 0), n)
    t0 = time.time()
    h = pa.Hasher(n, m, dw(sw)); torch.cuda.synchronize()
    tc = time.time() - t0
    key = dw(kw); out = h.new_out()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    h.hash(key, out); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); h.hash(key, out); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = float(np.median(ts))
    print(f"n={n} m={m} blocks={h.info['column_blocks']} transform_len={h.info['transform_len']} "
          f"ws={h.info['workspace_bytes']/2**30:.1f}GiB create={tc:.2f}s hash={t:.2f}ms {n/t/1e6:.1f} Gbit/s "
          f"resid={h.residual():.2e}", flush=True)
    h.close(); del key, out, flush; torch.cuda.empty_cache()
