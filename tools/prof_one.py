"""Run `reps` hashes of one config (for ncu / compute-sanitizer captures).

    python tools/prof_one.py C4 [reps] [route]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pa_synth as syn  # noqa: E402
import paper_1805_02372_b200 as pa  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
route = sys.argv[3] if len(sys.argv) > 3 else "auto"
n, m, sw, kw = syn.config_inputs(name)
dw = lambda w: torch.from_numpy(np.ascontiguousarray(w).view(np.int32).copy()).cuda()  # noqa: E731
h = pa.Hasher(n, m, dw(sw), route=route)
key = dw(kw)
out = h.new_out()
for _ in range(reps):
    h.hash(key, out)
torch.cuda.synchronize()
print(name, h.info, "resid", h.residual())
h.close()
