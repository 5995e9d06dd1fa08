import ctypes, os, sys
import numpy as np, torch
os.environ["PA_LIB"] = os.path.join(os.getcwd(), "paper_1805_02372_b200/libpa_T.so")
sys.path.insert(0, os.getcwd())
import pa_synth as syn, paper_1805_02372_b200 as pa
from paper_1805_02372_b200 import _lib
f = _lib._lib.pa_debug_k2_clocks
for name in sys.argv[1:]:
    n, m, sw, kw = syn.config_inputs(name)
    dw = lambda w: torch.from_numpy(np.ascontiguousarray(w).view(np.int32).copy()).cuda()
    h = pa.Hasher(n, m, dw(sw)); key = dw(kw); out = h.new_out()
    for _ in range(3): h.hash(key, out)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (64 * 16))()
    f(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(64, 16).astype(np.int64)
    d = np.diff(a[:, :7], axis=1)
    print(name, h.info["n1"], h.info["n2"], "phase cycles (load, tau+dif0, dif, fused, dit, last):", np.median(d, axis=0).astype(int), "total", int(np.median(a[:,6]-a[:,0])))
    h.close()
