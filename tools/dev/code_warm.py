"""Experiment: how much of a cold (L2-flushed) hash is instruction fetch?  After each flush,
optionally run one hash of ANOTHER handle whose K2 is the same kernel (C5a: 4096 x 144 shares
k2_rows_t<16, 16> with C2's 4096 x 160) -- it warms that kernel's code in L2 but none of C2's
data -- then time the C2 hash with events."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import pa_synth as syn
import paper_1805_02372_b200 as pa


def dw(w):
    return torch.from_numpy(np.ascontiguousarray(w).view(np.int32).copy()).cuda()


def handle(name):
    n, m, sw, kw = syn.config_inputs(name)
    h = pa.Hasher(n, m, dw(sw))
    return h, dw(kw), h.new_out()


main_h, main_k, main_o = handle("C2")
warm_h, warm_k, warm_o = handle(sys.argv[1] if len(sys.argv) > 1 else "C5a")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for mode in ("cold", "code-warm", "cold", "code-warm", "all-warm"):
    ts = []
    for it in range(40):
        if mode != "all-warm":
            flush.zero_()
        if mode == "code-warm":
            warm_h.hash(warm_k, warm_o)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        main_h.hash(main_k, main_o)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    print(f"{mode:10s} C2 hash median {np.median(ts[5:]):.1f} us")
