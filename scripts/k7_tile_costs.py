"""Per-tile K7 work at C2 (needs a TCGS_K7_PROFILE build via TCGS_LIB): writes gpurun_out/k7_tile_costs.npy with,
per tile, the slowest warp's work (136 x stages + 14 x relevant columns, in warp instructions)."""
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
st, rel = fr.T.cpu().numpy(), fr.n_contrib.cpu().numpy().astype(np.float64)
H, W = st.shape
th, tw = (H + 15) // 16, (W + 15) // 16
pad = lambda a: np.pad(a, ((0, th * 16 - H), (0, tw * 16 - W)))
st, rel = pad(st), pad(rel)
stw = st.reshape(th, 4, 4, tw, 2, 8)[:, :, 0, :, :, 0].transpose(0, 2, 1, 3).reshape(th * tw, 8)
relw = rel.reshape(th, 4, 4, tw, 2, 8)[:, :, 0, :, :, 0].transpose(0, 2, 1, 3).reshape(th * tw, 8)
cost = (136.0 * stw + 14.0 * relw).max(1)
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/k7_tile_costs.npy", cost)
print("tiles", cost.size, "mean", cost.mean(), "max", cost.max())
