"""Same-box sweep of forced plans (PA_FORCE_PLAN="N1,N2,C") for one config -- developer build.

    PA_LIB=$PWD/paper_1805_02372_b200/libpa_dev.so python tools/dev/plan_sweep.py C4 10240,6144,2 8192,7680,1 ...
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import pa_synth as syn  # noqa: E402
import paper_1805_02372_b200 as pa  # noqa: E402


def words(w):
    w = np.ascontiguousarray(w).view(np.int32)
    w = np.concatenate([w, np.zeros((-w.size) % 4, np.int32)])
    return torch.from_numpy(w.copy()).cuda()


batch = 1
if "--batch" in sys.argv:  # distinct keys per timed call (pa_hash_batch)
    i = sys.argv.index("--batch")
    batch = int(sys.argv[i + 1])
    del sys.argv[i:i + 2]
name = sys.argv[1]
if "," in name:  # "n,m": an arbitrary shape
    n, m = (int(v) for v in name.split(","))
    sw, kw = syn.random_bits(syn.seed_stream(70), n + m - 1), syn.random_bits(syn.key_stream(70, 1), n)
else:
    n, m, sw, kw = syn.config_inputs(name)
seed, key = words(sw), words(kw)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ref = None
for plan in ["default"] + sys.argv[2:]:
    if plan == "default":
        os.environ.pop("PA_FORCE_PLAN", None)
    else:
        os.environ["PA_FORCE_PLAN"] = plan
    h = pa.Hasher(n, m, seed, route="transform")
    out = h.new_out()
    if batch > 1:
        keys = syn.random_bits_torch([syn.key_stream(81, k) for k in range(batch)], n, "cuda")
        outs = h.new_out(batch)
        hash_once = lambda: h.hash_batch(keys, outs)  # noqa: E731
    else:
        hash_once = lambda: h.hash(key, out)  # noqa: E731
    for _ in range(3):
        hash_once()
    ts = []
    for _ in range(15):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hash_once()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    pa.pa_profile_enable(h.handle, True)
    pa.pa_profile_read(h.handle)
    for _ in range(5):
        flush.zero_()
        hash_once()
    kern = pa.pa_profile_read(h.handle)
    got = out.cpu().numpy()
    if ref is None:
        ref = got
    ok = np.array_equal(got[: (m + 31) // 32], ref[: (m + 31) // 32])
    ks = " ".join(f"{k.split('_')[0]}={v[1] / v[0] * 1e3:.1f}" for k, v in kern.items())
    i = h.info
    print(f"{plan:18s} -> {i['n1']}x{i['n2']} C={i['cols_per_cta']} C3={i['k3_cols_per_cta']}: "
          f"{np.median(ts) * 1e3 / batch:8.1f} us/key [{ks}] same={ok}", flush=True)
    h.close()
