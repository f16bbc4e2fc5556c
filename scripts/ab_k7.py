"""A/B experiment builds of libtcgs.so: python scripts/ab_k7.py name:-DFOO=1,-DBAR=2 ...  (builds only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_24796_b200 import build  # noqa: E402

for spec in sys.argv[1:]:
    name, _, defs = spec.partition(":")
    out = os.path.join(build.LIB_DIR, f"exp_{name}.so")
    print(build.build(out=out, defines=[d for d in defs.split(",") if d]))
