"""Is the cold-L2 penalty instruction fetch or data?  A: flush -> hash(h1).  B: flush ->
hash(h2) (same plan, other buffers: code hot) -> hash(h1) (h1's data cold)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import pa_synth as syn, paper_1805_02372_b200 as pa

def dw(w):
    return torch.from_numpy(np.ascontiguousarray(w).view(np.int32).copy()).cuda()

for name in sys.argv[1:] or ["C2"]:
    n, m, sw, kw = syn.config_inputs(name)
    h1, h2 = pa.Hasher(n, m, dw(sw)), pa.Hasher(n, m, dw(sw))
    k1, k2 = dw(kw), dw(kw)
    o1, o2 = h1.new_out(), h2.new_out()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        h1.hash(k1, o1); h2.hash(k2, o2)
    res = {"A_cold": [], "B_codehot": [], "warm": []}
    for it in range(30):
        for mode in res:
            flush.zero_()
            if mode == "B_codehot":
                h2.hash(k2, o2)
            if mode == "warm":
                h1.hash(k1, o1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); h1.hash(k1, o1); e1.record(); torch.cuda.synchronize()
            res[mode].append(e0.elapsed_time(e1) * 1e3)
    print(name, {k: round(float(np.median(v)), 1) for k, v in res.items()})
