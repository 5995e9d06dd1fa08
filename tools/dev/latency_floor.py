"""Event-timing floor of the bench protocol (256 MiB memset flush, then e0 / op / e1): a
one-kernel torch op vs a route-(b) C1 hash, flushed and warm.

    python tools/dev/latency_floor.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import pa_synth as syn  # noqa: E402
import paper_1805_02372_b200 as pa  # noqa: E402


def t(fn, flush, iters=50):
    ts = []
    for _ in range(iters):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts)


flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
small = torch.zeros(4, device="cuda")
n, m, sw, kw = syn.config_inputs("C1")
w = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int32).copy()).cuda()  # noqa: E731
h = pa.Hasher(n, m, w(sw))
key, out = w(kw), h.new_out()
for name, fn in (("torch add_ (1 kernel)", lambda: small.add_(1)), ("C1 hash", lambda: h.hash(key, out))):
    print(f"{name:24s} flushed {t(fn, flush):6.2f} us   warm {t(fn, None):6.2f} us")
rflush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
print(f"C1 hash after a READ flush (sum of 256 MiB) {t(lambda: h.hash(key, out), None, 1):.2f} us (1 iter)")
ts = []
for _ in range(30):
    rflush.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.hash(key, out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print(f"C1 hash, read-flushed: {np.median(ts):.2f} us")
