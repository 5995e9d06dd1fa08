"""Aggregate an ncu source-page SASS dump (ncu -i R --page source --csv --print-source sass
--kernel-name K) by opcode: stall samples, instructions executed, top stall reasons.

    python tools/ncu_sass_stalls.py dump.csv [top]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
ci = {k: i for i, k in enumerate(h)}
agg = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in rows[2:]:
    if len(r) < len(h):
        continue
    op = r[ci["Source"]].strip().split()[0] if r[ci["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[ci["Source"]].strip().split()[1]
    op = op.split(".")[0]
    a = agg[op]
    a["samples"] += int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    a["inst"] += int(r[ci["Instructions Executed"]] or 0)
    for k in h:
        if k.startswith("stall_") and "(Not Issued)" not in k:
            v = int(r[ci[k]] or 0)
            a[k] += v
            tot[k] += v
S = sum(a["samples"] for a in agg.values())
I = sum(a["inst"] for a in agg.values())
print(f"total samples {S}, warp instructions {I}")
for op, a in sorted(agg.items(), key=lambda kv: -kv[1]["samples"])[:top]:
    st = sorted(((k, v) for k, v in a.items() if k.startswith("stall_")), key=lambda kv: -kv[1])[:3]
    print(f"{op:10s} samples {a['samples'] / S:6.1%} inst {a['inst'] / I:6.1%}  " +
          " ".join(f"{k[6:]}={v / max(1, a['samples']):.0%}" for k, v in st))
print("all:", " ".join(f"{k[6:]}={v / S:.0%}" for k, v in tot.most_common(10)))
