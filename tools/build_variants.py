"""Build tuning variants of libharag.so (compile-time knobs) under build/variants/<name>/.
Usage: python tools/build_variants.py NAME="-DKNOB=V ..." ...   then run with HARAG_LIB=build/variants/NAME/libharag.so"""
import glob
import importlib.util
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location("harag_build", os.path.join(ROOT, "paper_2510_20878_b200", "build.py"))
b = importlib.util.module_from_spec(spec)
spec.loader.exec_module(b)
csrc = os.path.join(b.PKG, "csrc")
srcs = sorted(glob.glob(os.path.join(csrc, "*.cpp")) + glob.glob(os.path.join(csrc, "kernels", "*.cu")))
hdrs = sorted(glob.glob(os.path.join(csrc, "*.h")) + glob.glob(os.path.join(csrc, "kernels", "*.h")))
for arg in sys.argv[1:]:
    name, flags = arg.split("=", 1)
    out = os.path.join(ROOT, "build", "variants", name)
    os.makedirs(out, exist_ok=True)
    b._lib(os.path.join(out, "libharag.so"), srcs, hdrs, os.path.join(out, "obj"), flags.split())
    print("built", name, flags)
