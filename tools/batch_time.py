"""Batched throughput (BASELINE config C5): keys/s and Gbit/s of pa_hash_batch on one GPU.

    python tools/batch_time.py C5a C5b ...
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pa_synth as syn  # noqa: E402
import paper_1805_02372_b200 as pa  # noqa: E402


def main(names):
    for name in names:
        n, m, sw, kw = syn.config_inputs(name)
        count = {"C5a": 256, "C5b": 128, "C5c": 32, "C5d": 8}.get(name, 16)
        kw32 = (n + 31) // 32
        stride = (kw32 + 3) // 4 * 4
        keys = torch.zeros((count, stride), dtype=torch.int32, device="cuda")
        w = torch.from_numpy(np.ascontiguousarray(kw).view(np.int32)[:kw32].copy()).cuda()
        keys[:, :kw32] = w
        seed = torch.from_numpy(np.ascontiguousarray(sw).view(np.int32).copy()).cuda()
        h = pa.Hasher(n, m, seed)
        outs = h.new_out(count)
        h.hash_batch(keys, outs)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            h.hash_batch(keys, outs)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 3 / count
        print(f"{name} n={n} keys={count} {t * 1e3:.1f} us/key  {n / (t * 1e-3) / 1e9:.1f} Gbit/s  "
              f"plan {h.info['n1']}x{h.info['n2']} C={h.info['cols_per_cta']}", flush=True)
        h.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C5a", "C5b", "C5c", "C5d"])
