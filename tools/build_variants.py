"""Builds compile-time variants of libsphg.so for on-GPU sweeps (SPHG_LIB selects one at run time).
usage: python tools/build_variants.py NAME:-DFLAG=V,-DFLAG2=V ..."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2103_07925_b200 import build as B
for spec in sys.argv[1:]:
    name, flags = spec.split(":", 1)
    extra = [f for f in flags.split(",") if f]
    out = os.path.join(os.path.dirname(B.OUT), f"libsphg_{name}.so")
    bd = os.path.join(os.path.dirname(B.OUT), f"_build_{name}")
    print(name, B.build(out=out, extra=extra, build_dir=bd, force=True))
