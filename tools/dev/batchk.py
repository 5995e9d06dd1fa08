"""Batched throughput vs keys per launch (pa_options.batch_keys)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import pa_synth as syn, paper_1805_02372_b200 as pa
for name, count in (("C5a", 256), ("C5b", 128), ("C5c", 32)):
    n, m, sw, kw = syn.config_inputs(name)
    kw32 = (n + 31) // 32; stride = (kw32 + 3) // 4 * 4
    keys = torch.zeros((count, stride), dtype=torch.int32, device="cuda")
    keys[:, :kw32] = torch.from_numpy(np.ascontiguousarray(kw).view(np.int32)[:kw32].copy()).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for bk in (0, 4, 8, 16, 32, 64):
        h = pa.Hasher(n, m, torch.from_numpy(np.ascontiguousarray(sw).view(np.int32).copy()).cuda(), batch_keys=bk)
        outs = h.new_out(count)
        h.hash_batch(keys, outs); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); h.hash_batch(keys, outs); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / count)
        t = float(np.median(ts))
        print(f"{name} batch_keys={bk} {t*1e3:.1f} us/key {n/(t*1e-3)/1e9:.1f} Gbit/s", flush=True)
        h.close()
