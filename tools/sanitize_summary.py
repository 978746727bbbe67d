"""Classify a compute-sanitizer log (tools/sanitize.sh): error blocks grouped by kind and by the first
frame in this repo's code (libharag, a kernel, or the driver script), leaks split into this repo's
allocations and everyone else's (torch's caching allocators keep blocks until exit)."""
import re
import sys
from collections import Counter

text = open(sys.argv[1]).read()
blocks = re.split(r"\n========= \n", text)
kinds, leaks_ours, leaks_other = Counter(), 0, 0
for b in blocks:
    lines = [l for l in b.splitlines() if l.startswith("=========")]
    if not lines:
        continue
    head = next((l for l in lines if not l.startswith("=========     ") and "COMPUTE-SANITIZER" not in l
                 and "SUMMARY" not in l), None)
    if head is None:
        continue
    ours = next((l.split("Frame:")[1].strip() for l in lines if "Frame:" in l and
                 ("libharag" in l or "harag::" in l)), "-")
    ours = re.sub(r" \[0x[0-9a-f]+\]", "", ours)[:110]
    if head.strip().startswith("========= Leaked"):
        if ours != "-":
            leaks_ours += 1
        else:
            leaks_other += 1
        continue
    detail = next((l.strip("= ").strip() for l in lines[1:3] if "access" in l or "Barrier" in l or "at " in l), "")
    detail = re.sub(r"0x[0-9a-f]+", "0x..", detail)
    kinds[(re.sub(r"0x[0-9a-f]+", "0x..", head.strip("= ").strip()), detail, ours)] += 1
summ = [l for l in text.splitlines() if "SUMMARY" in l]
print("summary lines:", *summ, sep="\n  ")
print(f"leaks: {leaks_ours} from this repo's allocations, {leaks_other} from other libraries (torch caching allocators)")
for (h, d, o), n in kinds.most_common(20):
    print(f"{n:7d}  {h} | {d} | first repo frame: {o}")
