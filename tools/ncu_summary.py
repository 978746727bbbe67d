"""One-screen summary of an ncu --set full report (the profiles/round*/ncu_full_*.txt format).
Usage: python tools/ncu_summary.py REPORT.ncu-rep > summary.txt"""
import csv
import io
import subprocess
import sys

WANT = ["Memory Throughput", "DRAM Throughput", "Duration", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "SM Busy", "Mem Busy", "Max Bandwidth", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Mem Pipes Busy", "No Eligible", "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Block Size", "Grid Size", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Theoretical Occupancy", "Achieved Occupancy"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
       "launch__registers_per_thread"]


def run(args):
    return subprocess.run(["ncu", "-i", sys.argv[1]] + args, capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
rows = rows[[i for i, r in enumerate(rows) if "Kernel Name" in r][0]:]
h = rows[0]
iK, iN, iU, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
kernels = {}
for r in rows[1:]:
    if len(r) > iV:
        kernels.setdefault(r[iK], {}).setdefault(r[iN], (r[iV], r[iU]))
raw_rows = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
raw_rows = raw_rows[[i for i, r in enumerate(raw_rows) if "Kernel Name" in r][0]:]
rh, runits = raw_rows[0], raw_rows[1]
for k, m in kernels.items():
    print("kernel:", k.split("(")[0] + "(" + k.split("(")[1] if "(" in k else k)
    for w in WANT:
        if w in m:
            v, u = m[w]
            print(f"  {w:<40s}{v:>16s} {u}")
    for r in raw_rows[2:]:
        if len(r) == len(rh) and r[rh.index("Kernel Name")] == k:
            for w in RAW:
                if w in rh:
                    print(f"  {w:<40s}{r[rh.index(w)]:>16s} {runits[rh.index(w)]}")
            break
