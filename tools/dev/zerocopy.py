"""Experiment: key read by the kernels straight from pinned host memory vs H2D copy."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import pa_synth as syn, paper_1805_02372_b200 as pa
for name in ("C2", "C3", "C5a"):
    n, m, sw, kw = syn.config_inputs(name)
    h = pa.Hasher(n, m, torch.from_numpy(np.ascontiguousarray(sw).view(np.int32).copy()).cuda())
    kh = torch.from_numpy(np.ascontiguousarray(kw).view(np.int32).copy()).pin_memory()
    oh = torch.zeros(h.new_out().numel(), dtype=torch.int32).pin_memory()
    od = h.new_out()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    def zc():
        pa.pa_hash(h.handle, kh.data_ptr(), od.data_ptr(), torch.cuda.current_stream().cuda_stream)
        oh.copy_(od, non_blocking=True)
    def cp():
        h.hash_host_async(kh, oh)
    res = {}
    for nm, fn in (("memcpy", cp), ("zerocopy", zc), ("memcpy2", cp), ("zerocopy2", zc)):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(30):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        res[nm] = round(float(np.median(ts)), 1)
    ok = np.array_equal(oh.numpy(), od.cpu().numpy()[:oh.numel()])
    print(name, res, "zc result == memcpy result:", ok)
    h.close()
