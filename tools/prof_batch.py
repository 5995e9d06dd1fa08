"""Run `reps` batched hashes of distinct keys (for ncu captures of the batched kernels).

    python tools/prof_batch.py C1 65536 [reps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pa_synth as syn  # noqa: E402
import paper_1805_02372_b200 as pa  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
count = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
n, m, sw, _ = syn.config_inputs(name)
seed = torch.from_numpy(np.ascontiguousarray(sw).view(np.int32).copy()).cuda()
keys = syn.random_bits_torch([syn.key_stream(syn.CONFIG_INDEX[name], k) for k in range(count)], n, "cuda")
h = pa.Hasher(n, m, seed)
outs = h.new_out(count)
for _ in range(reps):
    h.hash_batch(keys, outs)
torch.cuda.synchronize()
print(name, count, h.info)
h.close()
