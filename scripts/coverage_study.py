"""How many splats a precise tile-ellipse coverage would drop, measured offline on a
config scene with the oracle's projection: N for the reference's 3-sigma square, for the alpha = 1/255 ellipse's
bounding box, and for exact ellipse-tile intersection (box minimum of the quadratic form)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_2505_24796_b200 import synthetic  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
scene, cams = synthetic.config_scene(cfg, scale)
cam = cams[0]
pr = oracle.project(scene["means"], scene["scales"], scene["rotations"], cam)
vis = np.nonzero(pr.visible)[0]
m = pr.mean2d[vis]
s11, s12, s22 = pr.inv_cov[vis].T
o = np.asarray(scene["opacities"], np.float64).reshape(-1)[vis]
r = pr.radius[vis]
tx_n, ty_n = (cam.width + 15) // 16, (cam.height + 15) // 16
x0 = np.clip(np.floor((m[:, 0] - r) / 16), 0, tx_n - 1).astype(int)
x1 = np.clip(np.floor((m[:, 0] + r) / 16), 0, tx_n - 1).astype(int)
y0 = np.clip(np.floor((m[:, 1] - r) / 16), 0, ty_n - 1).astype(int)
y1 = np.clip(np.floor((m[:, 1] + r) / 16), 0, ty_n - 1).astype(int)
inside = (np.floor((m[:, 0] + r) / 16) >= 0) & (np.floor((m[:, 0] - r) / 16) <= tx_n - 1) & \
         (np.floor((m[:, 1] + r) / 16) >= 0) & (np.floor((m[:, 1] - r) / 16) <= ty_n - 1)
area = np.where(inside, (x1 - x0 + 1) * (y1 - y0 + 1), 0)
N_ref = int(area.sum())
Q = 2.0 * (np.log(o) + np.log(255.0))  # live iff q <= Q
det = s11 * s22 - s12 * s12
cxx, cyy = s22 / det, s11 / det        # covariance diagonal
ex = np.sqrt(np.maximum(Q, 0) * cxx) + 0.5
ey = np.sqrt(np.maximum(Q, 0) * cyy) + 0.5
ax0 = np.maximum(x0, np.floor((m[:, 0] - ex) / 16).astype(int))
ax1 = np.minimum(x1, np.floor((m[:, 0] + ex) / 16).astype(int))
ay0 = np.maximum(y0, np.floor((m[:, 1] - ey) / 16).astype(int))
ay1 = np.minimum(y1, np.floor((m[:, 1] + ey) / 16).astype(int))
aabb = np.where(inside & (Q > 0) & (ax1 >= ax0) & (ay1 >= ay0), (ax1 - ax0 + 1) * (ay1 - ay0 + 1), 0)
N_aabb = int(aabb.sum())
# exact: per (Gaussian, tile) of the reference rect, min of q over the tile's pixel box
idx = np.repeat(np.arange(len(vis)), area)
off = np.arange(area.sum()) - np.repeat(np.cumsum(area) - area, area)
w = (x1 - x0 + 1)[idx]
tx = x0[idx] + off % w
ty = y0[idx] + off // w
mx, my = m[idx, 0], m[idx, 1]
a, b, c = s11[idx], s12[idx], s22[idx]
# box of pixel offsets d = p - mean, p in [16t, 16t+15]
lx, hx = 16 * tx - mx, 16 * tx + 15 - mx
ly, hy = 16 * ty - my, 16 * ty + 15 - my


def q(dx, dy):
    return a * dx * dx + 2 * b * dx * dy + c * dy * dy


inbox = (lx <= 0) & (hx >= 0) & (ly <= 0) & (hy >= 0)
best = np.where(inbox, 0.0, np.inf)
for fixed, lo_, hi_, is_x in ((lx, ly, hy, True), (hx, ly, hy, True), (ly, lx, hx, False), (hy, lx, hx, False)):
    if is_x:  # dx fixed: minimise over dy
        t = np.clip(-b * fixed / c, lo_, hi_)
        best = np.minimum(best, q(fixed, t))
    else:
        t = np.clip(-b * fixed / a, lo_, hi_)
        best = np.minimum(best, q(t, fixed))
live = best <= Q[idx]
N_exact = int(live.sum())
print(f"{cfg} x{scale}: visible {len(vis)}, N_ref {N_ref}, N_aabb {N_aabb} ({N_aabb / N_ref:.3f}), "
      f"N_exact {N_exact} ({N_exact / N_ref:.3f})")
