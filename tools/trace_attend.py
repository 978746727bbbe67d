"""Summarise a -DHARAG_ATT_TRACE run of tools/prof_attend.py (per-tile clock64 events of CTA 0).
Usage: python tools/trace_attend.py gpurun_out/trace.txt [first_tile last_tile]"""
import sys

import numpy as np

rows = [l.split() for l in open(sys.argv[1]) if l[:1].isdigit() and "|" in l]
a = np.array([[float(x) for x in r if x != "|"] for r in rows])
a = a[np.nonzero(a[:, 0] == 0)[0][-1]:]  # the last launch's trace
lo, hi = (int(sys.argv[2]), int(sys.argv[3])) if len(sys.argv) > 3 else (len(a) // 4, 3 * len(a) // 4)
s = slice(lo, hi)
sf, pf, kve, kvf, si, pv, ds, li, tl, ex = (a[:, i] for i in (1, 2, 3, 4, 5, 6, 7, 8, 9, 12))
print(f"tiles {lo}..{hi - 1}")
print(f"tile period               {np.diff(sf)[s].mean():8.0f} cycles")
print(f"softmax busy (S seen->P)  {(pf - sf)[s].mean():8.0f}   max pass {(tl - sf)[s].mean():6.0f}  P pass {(ex - tl)[s].mean():6.0f}")
print(f"softmax waits for S       {(sf[1:] - pf[:-1])[s].mean():8.0f}")
print(f"S issue -> S seen         {(sf - si)[s].mean():8.0f}")
print(f"P ready -> PV issue       {(pv - pf)[s].mean():8.0f}")
print(f"operands ready -> S issue {(si - kvf)[s].mean():8.0f}")
print(f"decode (loads in -> kvf)  {(kvf - li)[s].mean():8.0f}   stage (start -> loads in) {(li - ds)[s].mean():6.0f}")
sid, pvd = a[:, 10], a[:, 11]
print(f"S issue call -> returned   {(sid - si)[s].mean():8.0f}   PV issue call -> returned {(pvd - pv)[s].mean():6.0f}")
print(f"PV_j issued -> S_j+2 issue {(si[2:] - pvd[:-2])[s].mean():8.0f}   S_j returned -> PV_j-1 issue {(pv[:-1] - sid[1:])[s].mean():6.0f}")
kw = a[:, 3]
print(f"decoder: start -> kve ok   {(kw - ds)[s].mean():8.0f}   kve ok -> stage landed {(li - kw)[s].mean():6.0f}")
