import ctypes, os, sys
import numpy as np, torch
os.environ.setdefault("PA_LIB", os.path.join(os.getcwd(), "paper_1805_02372_b200/libpa_T.so"))
sys.path.insert(0, os.getcwd())
import pa_synth as syn, paper_1805_02372_b200 as pa
from paper_1805_02372_b200 import _lib
f = _lib._lib.pa_debug_k2_clocks
names = {0: ("K1", "zero+tables", "rowbits", "zgen", "stages", "store"), 1: ("K2", "load", "tau+dif0", "dif", "fused", "dit", "last"), 2: ("K3", "load", "stages", "epilogue")}
for name in sys.argv[1:]:
    n, m, sw, kw = syn.config_inputs(name)
    dw = lambda w: torch.from_numpy(np.ascontiguousarray(w).view(np.int32).copy()).cuda()
    h = pa.Hasher(n, m, dw(sw)); key = dw(kw); out = h.new_out()
    for _ in range(3): h.hash(key, out)
    if os.environ.get("COLD"):  # flush L2 before the recorded hash (COLD=read: clean lines only)
        fb = torch.ones(256 << 20, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        if os.environ["COLD"] == "read":
            fb.sum(dtype=torch.int64).item()
        else:
            fb.zero_()
        h.hash(key, out)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (3 * 64 * 16))()
    f(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(3, 64, 16).astype(np.int64)
    print(name, h.info["n1"], h.info["n2"], h.info["cols_per_cta"])
    for k in range(3):
        nm = names[k]; np_ = len(nm) - 1
        d = np.diff(a[k, :, :np_ + 1], axis=1)
        print("  ", nm[0], " ".join(f"{nm[i+1]}={int(np.median(d[:, i]))}" for i in range(np_)), "total", int(np.median(a[k, :, np_] - a[k, :, 0])))
    h.close()
