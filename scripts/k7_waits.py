"""Where K7's warps wait (experiment build with -DTCGS_K7_TIMING): python scripts/k7_waits.py [config]
Run with TCGS_LIB pointing at the timing build (scripts/ab_k7.py timing:-DTCGS_K7_TIMING=1)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_24796_b200 as tcgs  # noqa: E402
from paper_2505_24796_b200 import synthetic  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
spec = sys.argv[2] if len(sys.argv) > 2 else "tcgs"
scene, cams = synthetic.config_scene(cfg, 1.0)
cloud = tcgs.GaussianCloud.from_arrays(scene, "cuda")
r = tcgs.Renderer("cuda", spec)
r.render_frame(cloud, cams[0], timed=False)
fn = r.lib.tcgs_k7_timing
fn.argtypes = [ctypes.c_void_p]
buf = (ctypes.c_ulonglong * 8)()
fn(buf)  # clear
n = 5
for _ in range(n):
    f = r.render_frame(cloud, cams[0], timed=True)
fn(buf)
names = ["prod token", "prod empty stage", "prod tmem buffer", "cons full stage", "cons mma done", "prod total",
         "cons total"]
v = list(buf)
print(cfg, spec, "K7 ms", f.stats.stage_ms["blending"])
for i in range(5):
    tot = v[5] if i < 3 else v[6]
    print(f"{names[i]:18s} {v[i] / n:14.4g} cycles  {100 * v[i] / max(tot, 1):5.1f}% of the role's warp-time")
print(f"{'prod total':18s} {v[5] / n:14.4g}   {'cons total':12s} {v[6] / n:14.4g}")
print(f"token held (serial compaction) {v[7] / n:14.4g} cycles summed over CTAs = "
      f"{100 * v[7] / max(v[5] / 4, 1):5.1f}% of one producer's time")
