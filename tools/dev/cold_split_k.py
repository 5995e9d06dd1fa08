"""Per-kernel cold penalty: A flush->hash(h1); B flush->hash(h2)->hash(h1); warm."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import pa_synth as syn, paper_1805_02372_b200 as pa

def dw(w):
    return torch.from_numpy(np.ascontiguousarray(w).view(np.int32).copy()).cuda()

for name in sys.argv[1:] or ["C2"]:
    n, m, sw, kw = syn.config_inputs(name)
    h1, h2 = pa.Hasher(n, m, dw(sw)), pa.Hasher(n, m, dw(sw))
    k1, k2 = dw(kw), dw(kw)
    o1, o2 = h1.new_out(), h2.new_out()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        h1.hash(k1, o1); h2.hash(k2, o2)
    for mode in ("A_cold", "B_codehot", "warm"):
        pa.pa_profile_enable(h1.handle, True); pa.pa_profile_read(h1.handle)
        for it in range(30):
            flush.zero_()
            if mode == "B_codehot":
                h2.hash(k2, o2)
            if mode == "warm":
                pa.pa_profile_enable(h1.handle, False); h1.hash(k1, o1); pa.pa_profile_enable(h1.handle, True)
            h1.hash(k1, o1)
        kt = pa.pa_profile_read(h1.handle)
        pa.pa_profile_enable(h1.handle, False)
        print(name, mode, " ".join(f"{k}={v[1] / v[0] * 1e3:.1f}" for k, v in kt.items()))
