import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import pa_synth as syn, paper_1805_02372_b200 as pa
dev = torch.device("cuda", 0)
flush = torch.empty(bench.FLUSH_BYTES, dtype=torch.uint8, device=dev)
n, m, sw, kw = syn.config_inputs("C3")
h = pa.Hasher(n, m, bench.dev_words(torch, sw, dev))
key = bench.dev_words(torch, kw, dev)
out = h.new_out()
h.hash(key, out)
print("after 1 hash", h.residual())
for _ in range(3): h.hash(key, out)
print("after 3", h.residual())
ms = bench.time_steps(torch, lambda: h.hash(key, out), 10, flush)
print("after time_steps", h.residual())
