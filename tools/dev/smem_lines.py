"""Per-SASS-line shared-memory wavefronts from an ncu report's source page (ncu --import-source on):
which instructions load the shared-memory pipe, and how much of it is bank-conflict excess.

    python tools/dev/smem_lines.py gpurun_out/prof_C4_now.ncu-rep k3_inv [top]
"""
import csv
import io
import subprocess
import sys


def main(rep, kern, top=15):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + kern],
                         capture_output=True, text=True, timeout=600).stdout
    rows = list(csv.reader(io.StringIO(out)))
    # one block per profiled launch: header row, then column names, then data
    i = 0
    while i < len(rows):
        if rows[i] and rows[i][0] == "Kernel Name":
            name = rows[i][1][:90]
            hdr = rows[i + 1]
            j = i + 2
            data = []
            while j < len(rows) and not (rows[j] and rows[j][0] == "Kernel Name"):
                if len(rows[j]) == len(hdr):
                    data.append(rows[j])
                j += 1
            iw, ix, isrc = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Excessive"), hdr.index("Source")
            f = lambda r, k: float(r[k] or 0)  # noqa: E731
            tot, exc = sum(f(r, iw) for r in data), sum(f(r, ix) for r in data)
            print(f"== {name}\n   shared wavefronts {tot:.4g}, excessive {exc:.4g} ({100 * exc / max(tot, 1):.1f}%)")
            by_op = {}
            for r in data:
                op = r[isrc].split()[0] if r[isrc].split() else "?"
                if op.startswith("@"):
                    op = r[isrc].split()[1]
                op = op.split(".")[0]
                a = by_op.setdefault(op, [0.0, 0.0])
                a[0] += f(r, iw)
                a[1] += f(r, ix)
            for op, (w, x) in sorted(by_op.items(), key=lambda kv: -kv[1][0])[:8]:
                if w:
                    print(f"   {op:8s} {w:.4g} wavefronts ({100 * w / tot:.1f}%), excessive {x:.4g}")
            for r in sorted(data, key=lambda r: -f(r, ix))[:top]:
                if f(r, ix):
                    print(f"   {r[isrc].strip()[:64]:64s} {f(r, iw):.4g} exc {f(r, ix):.4g}")
            i = j
        else:
            i += 1


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 8)
