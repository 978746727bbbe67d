"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X): per kernel the
number of launches and the summed duration, and the share of assemble_kv_kernel in the GPU time.
Usage: python tools/launch_summary.py launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
iK, iM, iV, iID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.OrderedDict()
seq = []
for r in rows[hi + 1:]:
    if len(r) <= iV or r[iM] != "gpu__time_duration.sum":
        continue
    name = r[iK].split("(")[0]
    us = float(r[iV].replace(",", "")) / 1e3   # ns -> us
    n, t = per.get(name, (0, 0.0))
    per[name] = (n + 1, t + us)
    seq.append((name, us))
tot = sum(t for _, t in per.values())
print(f"{'kernel':70s} {'launches':>9s} {'total_us':>12s} {'share':>7s}")
for k, (n, t) in per.items():
    print(f"{k[:70]:70s} {n:9d} {t:12.1f} {t / tot:7.3f}")
asm = [us for name, us in seq if "assemble_kv_kernel" in name]
if asm:
    print(f"assemble_kv_kernel launches: {len(asm)}; first 16 (us): " + ", ".join(f"{x:.0f}" for x in asm[:16]))
