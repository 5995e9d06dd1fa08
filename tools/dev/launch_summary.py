"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): launches and mean
duration per kernel, and each kernel's share of the summed time.

python tools/dev/launch_summary.py gpurun_out/launches_C2.csv > profiles/launches_C2_r1_summary.json
"""
import csv
import json
import re
import sys


def short(name):
    """'void pa::k2_rows_t<16, 16>(...)' -> 'k2_rows_t<16, 16>'; other libraries' kernels keep
    their last identifier before the argument list."""
    head = name.split("(", 1)[0].strip()
    m = re.search(r"([A-Za-z_]\w*(?:<[^()]*>)?)$", head)
    return m.group(1) if m else head


def main(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr, body = rows[0], rows[1:]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    agg = {}
    for r in body:
        if r[mi] != "gpu__time_duration.sum":
            continue
        k = short(r[ki])
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    out = {k: {"launches": v[0], "mean_ns": v[1] / v[0], "share_of_total": v[1] / tot} for k, v in agg.items()}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
