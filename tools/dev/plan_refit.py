"""Grid-search the planner's cost-model factors on calibration sweeps (tools/dev/plan_calib.py
output): for each shape, the plan the model would pick among the measured candidates, and its
regret against the fastest measured candidate.

    python tools/dev/plan_refit.py gpurun_out/calib3.jsonl [...]
"""
import itertools
import json
import sys

import numpy as np

shapes = []
for path in sys.argv[1:]:
    for line in open(path):
        d = json.loads(line)
        c = [x for x in d["cands"] if "feat" in x]
        if len(c) >= 2:
            shapes.append(c)


def cost(x, p):
    f = x["feat"]
    a13, a2, l, b, s2, s13, k1p = p
    t13 = max(a13 * f["thr13"], l * f["lat13"]) + b
    t2 = max(a2 * f["thr2"], l * f["lat2"]) + b
    fs13 = s13 if f["spec13"] else 1.0
    return fs13 * t13 * (k1p if f["k1p"] else 1.0) + fs13 * t13 + (s2 if f["spec2"] else 1.0) * t2


def evaluate(p):
    reg = []
    for c in shapes:
        pick = min(c, key=lambda x: cost(x, p))
        best = min(x["meas_us"] for x in c)
        reg.append(pick["meas_us"] / best)
    r = np.array(reg)
    return r.mean(), r.max(), (r > 1.02).sum()


cur = (1.0, 1.0, 1.0, 2e-6, 0.9, 0.95, 0.91)
print("shapes", len(shapes), "current", evaluate(cur))
grid = itertools.product([0.8, 1.0, 1.2], [0.8, 1.0, 1.2, 1.4], [0.6, 1.0, 1.5, 2.0], [2e-6, 5e-6],
                         [0.7, 0.8, 0.9, 1.0], [0.85, 0.95, 1.0], [0.85, 0.91, 1.0])
res = sorted(((evaluate(p), p) for p in grid), key=lambda t: (t[0][0], t[0][1]))
for (mean, mx, n2), p in res[:12]:
    print(f"mean {mean:.4f} max {mx:.3f} >2%: {n2}  a13={p[0]} a2={p[1]} l={p[2]} b={p[3]} s2={p[4]} s13={p[5]} k1p={p[6]}")
