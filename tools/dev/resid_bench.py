import os, sys
sys.path.insert(0, os.getcwd())
import torch
import bench
import paper_1805_02372_b200 as pa
r = bench.sweep(torch, pa, torch.device("cuda", 0), steps=3)
print({k: v.get("residual") for k, v in r.items()})
