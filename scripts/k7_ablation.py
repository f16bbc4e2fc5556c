"""K7 alone for every alpha mode x EarlyCull on/off on one frame of a config (the paper's ablation,
PAPER.md:598-614, 640-647).  Run under ncu to capture the six K7 variants:
    ncu --set full -k regex:render_kernel -o gpurun_out/x python scripts/k7_ablation.py c2
Each variant renders one frame (its K1-K7) and then launches K7 once more on the same binned frame."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_24796_b200 as tcgs  # noqa: E402
from paper_2505_24796_b200 import synthetic  # noqa: E402
from paper_2505_24796_b200.raster import camera_struct  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
scene, cams = synthetic.config_scene(cfg, 1.0)
cloud = tcgs.GaussianCloud.from_arrays(scene, "cuda")
cam = cams[0]
for spec in ("tcgs", "tcgs-fp16", "tcgs-ffma"):
    for ec in (True, False):
        r = tcgs.Renderer("cuda", tcgs.make_backend(spec, use_early_cull=ec))
        f = r.render_frame(cloud, cam, timed=True)
        c = camera_struct(cam)
        rgb, T, cnt = r.outputs(c.width, c.height)
        rc = r.lib.tcgs_blend(cloud.P, c, r._opts(), r.ws.data_ptr(), r.ws.numel(), r.max_splats, rgb.data_ptr(),
                              T.data_ptr(), cnt.data_ptr(), torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        print(f"{cfg} {spec} earlycull={'on' if ec else 'off'} rc={rc} K7 {f.stats.stage_ms['blending']:.3f} ms "
              f"exp_calls={f.stats.exp_calls} f_blend={f.stats.f_blend} f_cull={f.stats.f_cull}", flush=True)
