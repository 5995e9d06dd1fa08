"""Developer timing sweep (not the bench contract): per-config ms/hash and Gbit/s.

    python tools/quick_time.py [C1 C2 ...]
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pa_synth as syn  # noqa: E402
import paper_1805_02372_b200 as pa  # noqa: E402


def dev_words(w):
    return torch.from_numpy(np.ascontiguousarray(w).view(np.int32).copy()).cuda()


def main(names, iters=20):
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for name in names:
        n, m, sw, kw = syn.config_inputs(name)
        for route in ("auto", "transform", "bitpacked"):
            if route == "bitpacked" and n * m > 1e13:
                continue
            t0 = time.time()
            h = pa.Hasher(n, m, dev_words(sw), route=route)
            torch.cuda.synchronize()
            tc = time.time() - t0
            key = dev_words(kw)
            out = h.new_out()
            for _ in range(3):
                h.hash(key, out)
            torch.cuda.synchronize()
            ts = []
            for _ in range(iters):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                h.hash(key, out)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            # back-to-back (L2-warm) throughput
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(iters):
                h.hash(key, out)
            e1.record()
            torch.cuda.synchronize()
            b2b = e0.elapsed_time(e1) / iters
            pa.pa_profile_enable(h.handle, True)
            pa.pa_profile_read(h.handle)
            for _ in range(iters):
                flush.zero_()
                h.hash(key, out)
            kt = pa.pa_profile_read(h.handle)
            pa.pa_profile_enable(h.handle, False)
            kts = " ".join(f"{k}={v[1] / v[0] * 1e3:.1f}us" for k, v in kt.items())
            med = float(np.median(ts))
            print(f"{name} n={n} m={m} route={h.route} info={h.info} create={tc*1e3:.1f}ms "
                  f"cold median={med*1e3:.1f}us ({n/med/1e6:.1f} Gbit/s) b2b={b2b*1e3:.1f}us "
                  f"({n/b2b/1e6:.1f} Gbit/s) resid={h.residual():.2e} | {kts}", flush=True)
            h.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4"])
