"""Per-source-line stall breakdown from an ncu report (needs -lineinfo and --import-source on).
Usage: python tools/ncu_lines.py REPORT.ncu-rep [line_lo line_hi] [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (0, 1 << 30)
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi_row = [i for i, r in enumerate(rows) if len(r) > 3 and r[0] == "Line No"][0]
h = rows[hi_row]
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
idx = {k: h.index(k) for k in stalls}
isamp, iinst = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


per = collections.defaultdict(lambda: collections.Counter())
src = {}
line = None
for r in rows[hi_row + 1:]:
    if not r:
        continue
    if r[0]:
        try:
            line = int(r[0])
        except ValueError:
            continue
        src[line] = r[1]
    if len(r) <= isamp or not r[2]:
        continue
    c = per[line]
    c["samples"] += num(r[isamp])
    c["inst"] += num(r[iinst])
    for k in stalls:
        c[k] += num(r[idx[k]])
tot = sum(c["samples"] for c in per.values())
print(f"total samples {tot:.0f}")
sel = [(l, c) for l, c in per.items() if lo <= l <= hi]
print(f"lines {lo}..{hi}: {sum(c['samples'] for _, c in sel) / tot * 100:.1f}% of samples")
for l, c in sorted(sel, key=lambda x: -x[1]["samples"])[:top]:
    st = sorted(((c[k], k[6:]) for k in stalls), reverse=True)[:3]
    print(f"{c['samples'] / tot * 100:5.1f}% L{l:<4} inst {c['inst']:9.0f}  " + " ".join(f"{k}:{v / max(c['samples'], 1) * 100:.0f}%" for v, k in st)
          + f"  | {src.get(l, '').strip()[:80]}")
