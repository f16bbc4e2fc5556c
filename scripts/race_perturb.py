"""Timing-perturbation check of K7's mbarrier protocol (racecheck cannot model inline-PTX mbarrier waits, so its
reported producer-write / consumer-read pairs are checked this way): render frames of three configs with the library
named by TCGS_LIB and print one digest of every output byte and FragmentStats counter.  Builds that perturb the
producer/consumer timing (producer back-off, extra consumer or producer work, 2 stages) must print the same digests
as the default build -- a missing happens-before edge would let a consumer read a stage mid-write under one of them.
    TCGS_LIB=paper_2505_24796_b200/_lib/exp_X.so python scripts/race_perturb.py"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_24796_b200 as tcgs  # noqa: E402
from paper_2505_24796_b200 import synthetic  # noqa: E402

out = []
for cfg, scale in (("c2", 0.1), ("c5", 0.03), ("c1", 1.0)):
    scene, cams = synthetic.config_scene(cfg, scale)
    cloud = tcgs.GaussianCloud.from_arrays(scene, "cuda")
    for spec in ("tcgs", "tcgs-ffma"):
        for sched in ("dynamic", "static"):
            r = tcgs.Renderer("cuda", spec, schedule=sched)
            for rep in range(3):
                f = r.render_frame(cloud, cams[0], timed=False)
                torch.cuda.synchronize()
                h = hashlib.sha256()
                for t in (f.rgb, f.T, f.n_contrib):
                    h.update(t.contiguous().cpu().numpy().tobytes())
                st = f.stats
                h.update(repr((st.f_blend, st.f_cull, st.f_skip, st.exp_calls, st.n_splats,
                               st.pixels_terminated)).encode())
                out.append(f"{cfg} {spec} {sched} {rep} {h.hexdigest()[:16]}")
print("\n".join(out))
print("DIGEST", hashlib.sha256("\n".join(l.rsplit(" ", 2)[0] + " " + l.rsplit(" ", 1)[1] for l in out).encode()).hexdigest()[:16])
