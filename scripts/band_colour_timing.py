"""Replicated per-rank K1 cost of tile bands at C3 (3M Gaussians, SH3, 4K): K1 with colour for every Gaussian
versus geometry-only K1 + the deferred colour of one band of 1/N of the tile rows (N = 2, 4, 8).  One GPU."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_24796_b200 as tcgs  # noqa: E402
from paper_2505_24796_b200 import synthetic  # noqa: E402

scene, cams = synthetic.config_scene("c3", 1.0)
cam = cams[0]
cloud = tcgs.GaussianCloud.from_arrays(scene, "cuda")
r = tcgs.Renderer("cuda", "tcgs")
r.render_frame(cloud, cam, timed=False)
ty = (cam.height + 15) // 16


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


full = timed(lambda: r.preprocess(cloud, cam))
geo = timed(lambda: r.preprocess(cloud, cam, defer_colour=True))
print(f"K1 with colour: {full:.1f} us; geometry only: {geo:.1f} us")
for n in (2, 4, 8):
    band = (ty // 2 - ty // (2 * n), ty // 2 - ty // (2 * n) + ty // n)  # a middle band of 1/n of the rows
    col = timed(lambda: r.colour(cloud, cam, band))
    print(f"N={n}: band rows {band}: colour {col:.1f} us -> replicated K1 {geo + col:.1f} us (was {full:.1f})")
