# compute-sanitizer (memcheck, racecheck, synccheck) over one small frame of every alpha mode
mkdir -p gpurun_out
cat > /tmp/sani.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_2505_24796_b200 as tcgs
from paper_2505_24796_b200 import synthetic
s = synthetic.make_scene(0, 2000); cam = synthetic.make_camera(96, 80)
c = tcgs.GaussianCloud.from_arrays(s, "cuda")
for spec in ("tcgs", "tcgs-fp16", "tcgs-ffma"):
    f = tcgs.Renderer("cuda", spec).render_frame(c, cam)
    print(spec, f.stats.f_blend, float(f.rgb.sum()))
f = tcgs.Renderer("cuda", "tcgs", coverage="ellipse").render_frame(c, cam)
print("ellipse coverage", f.stats.f_blend, f.stats.n_splats)
# fused multi-view K1 (a ragged tail CTA: P = 2000 is not a multiple of 256) and per-view K2-K7 on 3 streams
views = [synthetic.make_camera(96, 80)]
for yaw in (0.01, -0.02):
    v = synthetic.make_camera(96, 80)
    R = np.array([[np.cos(yaw), 0, np.sin(yaw)], [0, 1, 0], [-np.sin(yaw), 0, np.cos(yaw)]])
    m = np.asarray(v.view, np.float64).reshape(4, 4).copy()
    m[:3, :3] = R @ m[:3, :3]
    views.append(synthetic.CameraSpec(m, v.fx, v.fy, v.cx, v.cy, v.width, v.height, v.near))
vr = tcgs.ViewRenderer("cuda", "tcgs", n_streams=3)
vr.warm(c, views[0])
outs = vr.launch_group(c, views)
vr.join(); torch.cuda.synchronize()
print("view group", [float(o[0].sum()) for o in outs])
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/sani.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
