"""Run pa_hash_fresh_batch on a configuration `reps` times (an ncu target for the fused
fresh-seed K2): python tools/prof_fresh.py C4 2 2"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pa_synth as syn  # noqa: E402
import paper_1805_02372_b200 as pa  # noqa: E402

name, count, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
n, m, _, _ = syn.config_inputs(name)
ci = syn.CONFIG_INDEX[name]
seeds = syn.random_bits_torch([syn.seed_stream(900 + k) for k in range(count)], n + m - 1, "cuda")
keys = syn.random_bits_torch([syn.key_stream(ci, k) for k in range(count)], n, "cuda")
with pa.Hasher(n, m, seeds[0]) as h:
    outs = h.new_out(count)
    for _ in range(reps):
        h.hash_fresh_batch(seeds, keys, outs)
    torch.cuda.synchronize()
print("ok", name, count, reps)
