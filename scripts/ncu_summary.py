"""Summarise an ncu report (details + raw dram bytes) as text: python scripts/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Eligible Warps Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction", "Executed Instructions",
        "L2 Hit Rate", "L1/TEX Hit Rate", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
        "Mem Busy", "Max Bandwidth", "Mem Pipes Busy", "SM Busy"]


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    iN, iU, iV, iK = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value"), h.index("Kernel Name")
    print("kernel:", rows[1][iK])
    seen = set()
    for r in rows[1:]:
        if r[iN] in KEYS and r[iN] not in seen:
            seen.add(r[iN])
            print(f"  {r[iN]:40s} {r[iV]:>16s} {r[iU]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    names, units, vals = rr[0], rr[1], rr[2]
    for want in ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                 "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
                 "lts__t_bytes.sum", "launch__registers_per_thread"]:
        if want in names:
            i = names.index(want)
            print(f"  {want:40s} {vals[i]:>16s} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
