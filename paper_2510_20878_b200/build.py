"""In-tree build of the native libraries (nvcc, sm_100a only).

  paper_2510_20878_b200/libharag.so   product: C ABI (include/harag.h), store
                                      runtime (C++), sm_100a kernels
  synth/libharag_synth.so             device copy of the synthetic input generator

Run ``python paper_2510_20878_b200/build.py`` or ``__graft_entry__.build()`` (both
work before the library exists; ``python -m paper_2510_20878_b200.build`` imports
the package and so needs a loadable library).
Rebuilds when any source or header is newer than the library.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2510_20878_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-O3,-Wall", f"-I{ROOT}/include"]
COMMON += os.environ.get("HARAG_NVCC_EXTRA", "").split()  # experiments only (e.g. -DHARAG_ST_CS)

LIBHARAG = os.path.join(PKG, "libharag.so")
LIBSYNTH = os.path.join(ROOT, "synth", "libharag_synth.so")


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.stderr.strip() and os.environ.get("HARAG_BUILD_VERBOSE"):
        sys.stderr.write(r.stderr)


def _lib(target: str, sources: list[str], headers: list[str], objdir: str, extra: list[str] | None = None) -> bool:
    if not _newer(target, sources + headers) and not os.environ.get("HARAG_FORCE_BUILD"):
        return False
    os.makedirs(objdir, exist_ok=True)
    extra = extra or []
    objs, jobs = [], []
    for src in sources:
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", src, "-o", obj]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-v"] if os.environ.get("HARAG_PTXAS_VERBOSE") else []
        jobs.append(cmd)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
        list(ex.map(_run, jobs))
    tmp = target + ".tmp"
    _run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lpthread", "-ldl"])
    os.replace(tmp, target)
    return True


def build(verbose: bool = False) -> list[str]:
    """Compile every CUDA/C++ library in-tree; returns the libraries rebuilt."""
    csrc = os.path.join(PKG, "csrc")
    srcs = sorted(glob.glob(os.path.join(csrc, "*.cpp")) + glob.glob(os.path.join(csrc, "kernels", "*.cu")))
    hdrs = sorted(glob.glob(os.path.join(csrc, "*.h")) + glob.glob(os.path.join(csrc, "kernels", "*.h")) + [os.path.join(ROOT, "include", "harag.h")])
    built = []
    if _lib(LIBHARAG, srcs, hdrs, os.path.join(ROOT, "build", "harag")):
        built.append(LIBHARAG)
    ssrc = [os.path.join(ROOT, "synth", "csrc", "synth.cu")]
    if _lib(LIBSYNTH, ssrc, [], os.path.join(ROOT, "build", "synth")):
        built.append(LIBSYNTH)
    # test infrastructure: exhaustive check of the quantizer's division-free arithmetic
    chk_src = os.path.join(ROOT, "tests", "csrc", "markstein_check.cu")
    chk = os.path.join(ROOT, "tests", "csrc", "markstein_check")
    if os.path.exists(chk_src) and (_newer(chk, [chk_src]) or os.environ.get("HARAG_FORCE_BUILD")):
        _run([NVCC, *ARCH, "-O3", "-o", chk, chk_src])
        built.append(chk)
    if verbose:
        print("built:", built or "up to date")
    return built


if __name__ == "__main__":
    build(verbose=True)
