"""Fresh-seed batch vs plain batch vs a single pa_set_seed, per key (developer tool)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import pa_synth as syn, paper_1805_02372_b200 as pa
def dw(w):
    w = np.ascontiguousarray(w).view(np.int32)
    return torch.from_numpy(np.concatenate([w, np.zeros((-w.size) % 4, np.int32)])).cuda()
for name in ("C2", "C5a"):
    n, m, sw, kw = syn.config_inputs(name)
    count = 64
    seeds = torch.stack([dw(syn.random_bits(syn.seed_stream(900 + k), n + m - 1)) for k in range(count)])
    keys = torch.stack([dw(kw)] * count)
    h = pa.Hasher(n, m, seeds[0]); outs = h.new_out(count)
    def t(fn, it=10):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(it): fn()
        e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / it / count * 1e3
    print(name, "fresh batch us/key", round(t(lambda: h.hash_fresh_batch(seeds, keys, outs)), 2),
          "hash batch us/key", round(t(lambda: h.hash_batch(keys, outs)), 2),
          "set_seed us", round(t(lambda: h.set_seed(seeds[1]), 10) * count, 2))
