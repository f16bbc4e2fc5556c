"""Per-warp K7 work balance at C2 (experiment: needs a TCGS_K7_PROFILE build via TCGS_LIB).

The profile build writes, per pixel, the stages its warp entered (T) and the columns relevant to its warp
(n_contrib).  Work per warp ~ A * stages + B * relevant columns; a tile takes as long as its slowest warp."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_24796_b200 as tcgs  # noqa: E402
from paper_2505_24796_b200 import synthetic  # noqa: E402

scene, cams = synthetic.config_scene("c2", 1.0)
cloud = tcgs.GaussianCloud.from_arrays(scene, "cuda")
fr = tcgs.Renderer("cuda").render_frame(cloud, cams[0], timed=False)
st = fr.T.cpu().numpy()
rel = fr.n_contrib.cpu().numpy().astype(np.float64)
H, W = st.shape
th, tw = (H + 15) // 16, (W + 15) // 16
pad = lambda a: np.pad(a, ((0, th * 16 - H), (0, tw * 16 - W)))
st, rel = pad(st), pad(rel)
# warp w of a tile: lx // 8 + 2 * (ly // 4); take one lane per warp block (8 x 4)
stw = st.reshape(th, 4, 4, tw, 2, 8)[:, :, 0, :, :, 0]      # [ty, wy, tx, wx]
relw = rel.reshape(th, 4, 4, tw, 2, 8)[:, :, 0, :, :, 0]
stw = stw.transpose(0, 2, 1, 3).reshape(th * tw, 8)
relw = relw.transpose(0, 2, 1, 3).reshape(th * tw, 8)
for A, B in ((136.0, 14.0), (100.0, 14.0), (0.0, 1.0)):
    work = A * stw + B * relw
    mx, mean = work.max(1), work.mean(1)
    print(f"A={A} B={B}: sum(max)/sum(mean) = {mx.sum() / max(mean.sum(), 1):.3f}")
print("stages/warp mean %.1f, relevant/warp mean %.1f, tiles %d" % (stw.mean(), relw.mean(), th * tw))
tile_stages = stw.max(1)
print("relevant fraction of stage columns: %.3f" % (relw.sum() / max((stw * 32).sum(), 1)))
