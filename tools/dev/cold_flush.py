"""Cold-start penalty: is it the flush's dirty L2 lines (write-back) or cold misses?"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import pa_synth as syn, paper_1805_02372_b200 as pa

def dw(w):
    return torch.from_numpy(np.ascontiguousarray(w).view(np.int32).copy()).cuda()

for name in sys.argv[1:] or ["C2"]:
    n, m, sw, kw = syn.config_inputs(name)
    h1 = pa.Hasher(n, m, dw(sw))
    k1 = dw(kw)
    o1 = h1.new_out()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    rd = torch.empty(512 << 20, dtype=torch.uint8, device="cuda").view(torch.int64)
    acc = torch.empty(1, dtype=torch.int64, device="cuda")
    for _ in range(3):
        h1.hash(k1, o1)
    res = {}
    for mode in ("write_flush", "write_flush+spin50us", "read_flush", "write_then_read", "none"):
        ts = []
        for it in range(30):
            if mode.startswith("write"):
                flush.zero_()
            if mode == "read_flush" or mode == "write_then_read":
                torch.sum(rd, dim=0, out=acc.view(()))
            if mode == "write_flush+spin50us":
                torch.cuda._sleep(100000)  # ~50 us of spinning, no memory traffic
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); h1.hash(k1, o1); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res[mode] = round(float(np.median(ts)), 1)
    print(name, res)
