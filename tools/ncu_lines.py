"""Top CUDA source lines by warp-stall samples for one kernel of an ncu report.

    python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv, io, subprocess, sys
rep, k = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda", "-k", "regex:" + k],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
# find header row containing "Source"
hi = next(i for i, r in enumerate(rows) if "Source" in r)
hdr = rows[hi]
si = hdr.index("Source"); wi = hdr.index("Warp Stall Sampling (All Samples)")
li = hdr.index("Line") if "Line" in hdr else None
items = []
tot = 0
for r in rows[hi + 1:]:
    if len(r) <= wi: continue
    try: s = float(r[wi])
    except ValueError: continue
    tot += s
    items.append((s, r[li] if li is not None else "", r[si].strip()[:110]))
items.sort(reverse=True)
for s, l, src in items[:top]:
    print(f"{100*s/tot:5.1f}%  {l:>5}  {src}")
