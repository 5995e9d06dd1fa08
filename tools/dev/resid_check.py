import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import pa_synth as syn, paper_1805_02372_b200 as pa
def dw(w): return torch.from_numpy(np.ascontiguousarray(w).view(np.int32).copy()).cuda()
for name in ("C2", "C3", "C4"):
    n, m, sw, kw = syn.config_inputs(name)
    h = pa.Hasher(n, m, dw(sw)); key = dw(kw); out = h.new_out()
    h.hash(key, out); torch.cuda.synchronize()
    r1 = h.residual()
    for _ in range(5): h.hash(key, out)
    r2 = h.residual()
    print(name, r1, r2, h.info)
