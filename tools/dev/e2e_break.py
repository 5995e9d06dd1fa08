import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import pa_synth as syn, paper_1805_02372_b200 as pa
n, m, sw, kw = syn.config_inputs("C2")
def dw(w):
    w = np.ascontiguousarray(w).view(np.int32)
    return torch.from_numpy(np.concatenate([w, np.zeros((-w.size) % 4, np.int32)])).cuda()
h = pa.Hasher(n, m, dw(sw)); key = dw(kw); out = h.new_out()
kh = torch.from_numpy(np.ascontiguousarray(kw).view(np.int32).copy()).pin_memory()
oh = torch.empty(pa.words32(m), dtype=torch.int32).pin_memory()
s = torch.cuda.current_stream()
def ev(fn, it=50):
    ts = []
    for _ in range(5): fn()
    torch.cuda.synchronize()
    for _ in range(it):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter(); e0.record(); fn(); e1.record(); e1.synchronize(); t1 = time.perf_counter()
        ts.append((e0.elapsed_time(e1) * 1e3, (t1 - t0) * 1e6))
    a = np.array(ts); return np.median(a[:, 0]), np.median(a[:, 1])
print("hash only (events, wall us):", ev(lambda: h.hash(key, out)))
print("H2D only:", ev(lambda: key.copy_(kh.to(key.device, non_blocking=True)[:key.numel()] if False else key[:kh.numel()].copy_(kh, non_blocking=True))))
print("D2H only:", ev(lambda: oh.copy_(out[:oh.numel()], non_blocking=True)))
print("pa_hash_host:", ev(lambda: h.hash_host(kh, oh)))
print("H2D+hash+D2H async then sync:", ev(lambda: (key[:kh.numel()].copy_(kh, non_blocking=True), h.hash(key, out), oh.copy_(out[:oh.numel()], non_blocking=True))))
