"""Aggregate SASS-level warp-stall samples of one kernel by opcode and stall reason.
    python tools/ncu_sass.py report.ncu-rep kernel_regex
"""
import csv, io, subprocess, sys, collections
rep, k = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + k],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
S = h.index("Source"); W = h.index("Warp Stall Sampling (All Samples)"); X = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
by_op = collections.Counter(); by_reason = collections.Counter(); inst = collections.Counter()
tot = 0
for r in rows[hi + 1:]:
    if len(r) <= W: continue
    try: w = float(r[W])
    except ValueError: continue
    op = r[S].strip().split()[0] if r[S].strip() else "?"
    if op.startswith("@"): op = r[S].strip().split()[1]
    op = op.split(".")[0]
    by_op[op] += w; tot += w
    try: inst[op] += float(r[X])
    except ValueError: pass
    for c in reasons:
        try: by_reason[c] += float(r[h.index(c)])
        except ValueError: pass
print("stall samples by opcode:")
for op, w in by_op.most_common(18): print(f"  {op:10s} {100*w/tot:5.1f}%   warp-instr executed {inst[op]:.3g}")
print("by reason:")
t2 = sum(by_reason.values())
for c, w in by_reason.most_common(10): print(f"  {c:22s} {100*w/t2:5.1f}%")
print("total warp-instructions executed:", f"{sum(inst.values()):.4g}")
