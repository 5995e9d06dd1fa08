"""A few small hashes on both routes (for compute-sanitizer runs)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import pa_synth as syn, paper_1805_02372_b200 as pa
def dw(w):
    w = np.ascontiguousarray(w).view(np.int32)
    return torch.from_numpy(np.concatenate([w, np.zeros((-w.size) % 4, np.int32)])).cuda()
for n, m, route in ((100, 30, "transform"), (4097, 1000, "transform"), (65537, 6553, "transform"),
                    (1000003, 250000, "transform"), (4096, 1024, "bitpacked"), (70001, 17000, "bitpacked")):
    sw = syn.random_bits(1, n + m - 1); kw = syn.random_bits(2, n)
    h = pa.Hasher(n, m, dw(sw), route=route)
    out = h.hash(dw(kw))
    if route == "transform":
        keys = torch.stack([dw(syn.random_bits(3 + k, n)) for k in range(3)])
        h.hash_batch(keys)
        h.set_seed(dw(syn.random_bits(9, n + m - 1)))
        h.hash(dw(kw), out)
    torch.cuda.synchronize()
    print(n, m, route, "ok", h.residual(), flush=True)
    h.close()
