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
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python /tmp/sani.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "== $tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
