import ctypes, os, sys
import numpy as np, torch
os.environ.setdefault("PA_LIB", os.path.join(os.getcwd(), "paper_1805_02372_b200/libpa_T.so"))
sys.path.insert(0, os.getcwd())
import pa_synth as syn, paper_1805_02372_b200 as pa
from paper_1805_02372_b200 import _lib
f = _lib._lib.pa_debug_trace
for name in sys.argv[1:]:
    n, m, sw, kw = syn.config_inputs(name)
    dw = lambda w: torch.from_numpy(np.ascontiguousarray(w).view(np.int32).copy()).cuda()
    h = pa.Hasher(n, m, dw(sw)); key = dw(kw); out = h.new_out()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3): h.hash(key, out)
    flush.zero_(); torch.cuda.synchronize()
    if os.environ.get("QUEUED"):  # launches queued behind a 100 us spin: no CPU launch gaps
        torch.cuda._sleep(200000)
    h.hash(key, out); torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (4 * 8192 * 3))()
    f(buf)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(4, 8192, 3).astype(np.int64)
    info = h.info
    ctas = {0: None, 1: info["n1"] // info["cols_per_cta"], 2: info["n2"], 3: info["n1"] // info["cols_per_cta"]}
    t_ref = None
    print(name, info["n1"], info["n2"], info["cols_per_cta"])
    for k, nm in enumerate(["K0", "K1", "K2", "K3"]):
        rows = a[k][a[k, :, 2] > 0]
        if k == 0: t_ref = rows[:, 1].min()
        st, en = rows[:, 1] - t_ref, rows[:, 2] - t_ref
        dur = en - st
        per_sm = np.bincount(rows[:, 0], minlength=148)
        print(f"  {nm}: ctas={len(rows)} start={st.min()/1e3:.1f}us end={en.max()/1e3:.1f}us span={(en.max()-st.min())/1e3:.1f}us "
              f"cta dur med={np.median(dur)/1e3:.1f} max={dur.max()/1e3:.1f}us  ctas/SM max={per_sm.max()} "
              f"last-start={st.max()/1e3:.1f}us")
    h.close()
