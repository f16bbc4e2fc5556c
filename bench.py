"""Benchmark: TC-GS forward render on B200 (BASELINE.json metric, config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

One step = one full frame of the hot path (K1 preprocess -> K2-K6 binning ->
K7 tensor-core alpha + blend) of a new camera view of the config-2 workload:
1M synthetic Gaussians with SH degree 3 at 1920x1080, inputs resident in HBM
(the 236 MB scene exceeds the 126 MB L2, so no flush is needed between frames).

* ``value`` is the single-camera frame rate: lone frames back to back on one
  CUDA stream (the K7 dynamic tile queue), each frame fully re-projected,
  re-binned and re-blended.  ``views_in_flight`` reports the multi-view
  throughput (16 frames on 16 streams, one fused K1 per 8 views) separately.
* N > 1 shards camera views across ranks (one process per GPU, no collective on
  the data path; weak scaling: every rank renders K frames).  ``--gpus N``
  without torchrun re-launches itself under ``torch.distributed.run``.
  ``--config c3`` renders 4K frames split into tile-row bands across the ranks
  (strong scaling; K7 writes into rank 0's frame over NVLink peer memory).

The JSON line carries the device-timed throughput (`value`), the end-to-end
throughput through the public API with host buffers (`e2e`), the roofline of
the dominant kernel (K7: issue-bound; tensor, MUFU and issue fractions side
by side), the alpha-blend ablation (Frag2Mat x EarlyCull, the paper's table),
the CPU baseline (the oracle's C port of the reference renderer on this
host's cores, whole frames), clocks and the kernel-launch count.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec at 1080p (1M Gaussians) and alpha-blend ms/frame; TC/MUFU % of peak"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--scale", type=float, default=1.0, help="scene-size multiplier (testing only)")
    ap.add_argument("--impl", default="tcgs", choices=["tcgs", "reference"])
    ap.add_argument("--backend", default="tcgs")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--streams", type=int, default=16, help="views in flight (one workspace + CUDA stream each)")
    ap.add_argument("--coverage", choices=["square", "box", "ellipse"], default="square",
                    help="tiles per Gaussian: the reference's 3-sigma square (parity), or opt-in (same image, fewer "
                         "splats; SURVEY.md 8(f) 4): the alpha-ellipse's bounding box, or every tile it touches")
    ap.add_argument("--view-group", type=int, default=8,
                    help="views per fused K1 pass (tcgs_preprocess_views; <= --streams, <= 8); 0 = one K1 per "
                         "view.  Two groups in flight: the next group's K1 overlaps this group's K2-K7")
    ap.add_argument("--band-output", default="peer", choices=["peer", "gather"],
                    help="c3 tile bands: K7 writes into rank 0's frame over peer memory, or one NCCL gather")
    ap.add_argument("--no-ablation", action="store_true",
                    help="skip the alpha-blend ablation (K7 per alpha mode x EarlyCull on/off)")
    ap.add_argument("--no-in-flight", action="store_true", help="skip the views-in-flight throughput")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="CPU baseline leg: whole oracle frames until this much CPU time has been spent")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def view_cameras(base, n):
    """Views of the config scene: yaw steps of 0.5 mrad about the camera centre (view sharding)."""
    from paper_2505_24796_b200.synthetic import CameraSpec

    cams = []
    for k in range(n):
        th = 0.0005 * k
        c, s = math.cos(th), math.sin(th)
        v = np.array(base.view, dtype=np.float64).copy()
        R = np.array([[c, 0.0, s], [0.0, 1.0, 0.0], [-s, 0.0, c]])
        v[:3, :3] = R @ v[:3, :3]
        v[:3, 3] = R @ v[:3, 3]
        cams.append(CameraSpec(v, base.fx, base.fy, base.cx, base.cy, base.width, base.height, base.near))
    return cams


class ClockSampler:
    """Samples SM clocks and throttle reasons (NVML) while the timed region runs."""

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.pynvml = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:  # noqa: BLE001 - clocks are best effort
            self.pynvml = None
        return self

    def _sample(self):
        p = self.pynvml
        self.samples.append(p.nvmlDeviceGetClockInfo(self.h, p.NVML_CLOCK_SM))
        r = p.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
        }
        for k, bit in names.items():
            if r & bit:
                self.reasons.add(k)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                break
            time.sleep(0.001)  # (the driver times 20 steps: ~16 ms at C2)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()
        if self.pynvml and not self.samples:
            try:
                self._sample()
            except Exception:  # noqa: BLE001
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        busy = [s for s in self.samples]
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons - {"gpu_idle"}), "samples": len(busy)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def rank_views(cams, base, per_rank, rank, world, bands_mode):
    """The cameras this rank renders: in tile-band mode every rank renders its band of the same frames; otherwise
    the config's camera pool (C4's orbit, or new yaw views of the base camera) is split into contiguous blocks,
    one per rank (shard.view_blocks: no view twice, no collective on the data path)."""
    from paper_2505_24796_b200 import shard

    if bands_mode:
        return view_cameras(base, per_rank)
    pool = cams if len(cams) > 1 else view_cameras(base, world * per_rank)
    b0, b1 = shard.view_blocks(len(pool), world)[rank]
    mine = pool[b0:b1] or pool[:1]
    return [mine[k % len(mine)] for k in range(per_rank)]


def max_over_ranks(values, device, world):
    """Device times of the timed region, max over ranks (the contract's whole-job time)."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(values), dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def pinned_h2d_GBps(host, dev, reps=3):
    """Measured pinned host -> device copy bandwidth of this GPU's link (the scene's own buffers, CUDA events)."""
    import torch

    bufs = [(v, torch.empty_like(v, device=dev)) for v in host.values()]
    nbytes = sum(v.numel() * v.element_size() for v in host.values())
    for h, d in bufs:  # warm
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize(dev)
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(reps):
        for h, d in bufs:
            d.copy_(h, non_blocking=True)
    t1.record()
    torch.cuda.synchronize(dev)
    return reps * nbytes / (t0.elapsed_time(t1) * 1e-3) / 1e9


def e2e_resident(vr, cloud, views, base, dev, world, dist):
    """Context for `e2e`: the same host-facing loop with the scene kept resident in HBM (a renderer's usual
    case): per frame only the camera goes host -> device (as kernel parameters) and the RGB image plus the
    FragmentStats snapshot come back to pinned host memory, with views in flight on the ViewRenderer."""
    import ctypes

    import torch

    n = len(vr.streams)
    outs = [torch.empty((base.height, base.width, 3), dtype=torch.float32).pin_memory() for _ in range(n)]
    nb = int(vr.lib.tcgs_counters_bytes())
    snaps = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(n)]
    steps = max(8, min(len(views), 40))

    def run(k):
        i = vr.k % n
        rgb, _, _ = vr.launch(cloud, views[k % len(views)])
        with torch.cuda.stream(vr.streams[i]):
            outs[i].copy_(rgb, non_blocking=True)
            vr.lib.tcgs_snapshot_stats(ctypes.c_void_p(vr.renderers[i].ws.data_ptr()),
                                       ctypes.c_void_p(snaps[i].data_ptr()), ctypes.c_void_p(vr.streams[i].cuda_stream))

    for k in range(n):
        run(k)
    vr.join()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(steps):
        run(k)
    vr.join()
    torch.cuda.synchronize(dev)
    t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    cam_bytes = 16 * 8 + 5 * 8 + 2 * 4
    return {"value": world * steps / float(t.item()), "unit": "frames/s", "h2d_bytes_per_step": cam_bytes,
            "d2h_bytes_per_step": base.width * base.height * 12 + nb, "steps": steps}


def stage_rooflines(scene, P, st, stage_ms, peaks, cam):
    """Algorithmic bytes per stage / isolated stage time, against the measured HBM copy peak.
    K1: P x (inputs + 76 B of outputs); binning: P (8 B depth + 4 B index) read + write, N (2 B tile key +
    4 B id) written and sorted once, N x 2 B of ranges; K7: N x 52 B (id + 48 B record) + 20 B per pixel.
    """
    feats = 3 * 4 * ((scene.get("sh_degree", 0) + 1) ** 2 if scene.get("sh_degree", 0) > 0 else 1)
    N = st.n_splats
    work = {"preprocess": P * (44 + feats + 76), "binning": P * 12 * 2 + N * 6 * 2 + N * 2,
            "blend": N * 52 + cam.width * cam.height * 20}
    out = {}
    for k, b in work.items():
        ms = stage_ms.get(k) if isinstance(stage_ms, dict) else None
        if not ms:
            continue
        gbs = b / (ms * 1e-3) / 1e9
        out[k] = {"bytes_alg": int(b), "ms": ms, "achieved_GBps": gbs, "peak_GBps": peaks["hbm_gbs"],
                  "frac": gbs / peaks["hbm_gbs"]}
    return out


def issue_roofline(traffic, blend_ms, clocks):
    """K7's binding resource: warp-instruction issue (4 per clock per SM).  Instructions per launch come from
    the committed ncu capture of the same build and workload (smsp__inst_executed.sum), the duration from this
    run's CUDA events, the clock from the NVML samples of this run's timed region."""
    inst = (traffic or {}).get("warp_inst_per_launch")
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    if not inst:
        return None
    peak = 4 * 148 * mhz * 1e6
    ach = inst / (blend_ms * 1e-3)
    return {"achieved": ach, "peak": peak, "unit": "warp-instructions/s", "frac": ach / peak,
            "warp_inst_per_launch": inst, "source": traffic.get("source"),
            "note": "instructions from the committed ncu profile; clock = median SM clock sampled during the timed "
                    "region"}


def profile_traffic(config="c2"):
    """K7 DRAM bytes and warp instructions per launch (dram__bytes_read.sum + dram__bytes_write.sum,
    smsp__inst_executed.sum) from the committed ncu --set full summaries under profiles/ (scripts/ncu_summary.py):
    C2 (the frame capture) and C5 (the ablation capture); other configs get None."""
    import glob

    if config == "c5":  # the ablation capture's default variant (hi/lo, EarlyCull on, dynamic schedule)
        p = os.path.join(ROOT, "profiles", "r2j2_ablation_c5_ncu.json")
        if not os.path.exists(p):
            return None
        with open(p) as f:
            rows = [e for e in json.load(f) if "render_kernel<0, 1, 0>" in e.get("kernel", "")]
        if not rows:
            return None
        mb = [e["dram_read_MB"] + e["dram_write_MB"] for e in rows]
        inst = [e["inst_executed"] for e in rows]
        return {"bytes_per_launch": 1e6 * sum(mb) / len(mb), "source": os.path.relpath(p, ROOT),
                "warp_inst_per_launch": sum(inst) / len(inst)}
    if config != "c2":
        return None
    # the capture of the current build first (K7 rows of profiles/r2j2_frame_ncu.json), then older ones
    current = os.path.join(ROOT, "profiles", "r2j2_k7_ncu.json")
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_k7_ncu.json")))  # r1_ < ... < r2a_ < r2b_
    files = [f for f in files if f != current] + ([current] if os.path.exists(current) else [])
    for p in reversed(files):
        with open(p) as f:
            rows = [e for e in json.load(f) if "render_kernel" in e.get("kernel", "")]
        if rows:
            mb = [e["dram_read_MB"] + e["dram_write_MB"] for e in rows]
            inst = [e.get("inst_executed") for e in rows if isinstance(e.get("inst_executed"), float)]
            return {"bytes_per_launch": 1e6 * sum(mb) / len(mb), "source": os.path.relpath(p, ROOT),
                    "warp_inst_per_launch": sum(inst) / len(inst) if inst else None}
    return None


# ------------------------------------------------------------------------------------------ CPU side

def cpu_reference_frame(scene, cam):
    """One WHOLE frame of the oracle's C port of the reference renderer (tilesplat.render 'reference',
    src/tilesplat/raster.py:161-201: project, build_tiles, blend every tile) on the host cores (OpenMP)."""
    import oracle

    t0 = time.perf_counter()
    colors = scene["colors"]
    if scene.get("sh_degree", 0) > 0:
        colors = oracle.sh_color(scene["means"], scene["features"], scene["sh_degree"], cam.view)
    proj = oracle.project(scene["means"], scene["scales"], scene["rotations"], cam)
    t1 = time.perf_counter()
    off, ids = oracle.build_tiles(proj, cam)
    t2 = time.perf_counter()
    oracle.blend(proj, off, ids, scene["opacities"], colors, cam)
    t3 = time.perf_counter()
    return t3 - t0, {"preprocess_s": t1 - t0, "sort_s": t2 - t1, "blend_s": t3 - t2}


def cpu_frames(scene, cam, budget_s, max_frames=20):
    """Whole oracle frames until ``budget_s`` seconds have been spent (at least one)."""
    times, det = [], None
    spent = 0.0
    while not times or (spent < budget_s and len(times) < max_frames):
        s_, det = cpu_reference_frame(scene, cam)
        times.append(s_)
        spent += s_
    return times, det


def bench_config(args, scene, cam, world):
    """The workload description both arms print (the driver compares them)."""
    from paper_2505_24796_b200 import synthetic

    bands = args.config == "c3"
    feats = "features" if scene.get("sh_degree", 0) > 0 else "colors"
    mb = sum(np.asarray(scene[k]).nbytes for k in ("means", "scales", "rotations", "opacities", feats)) / 1e6
    return {"workload": f"{args.config}: " + synthetic.CONFIGS[args.config],
            "P": int(np.asarray(scene["means"]).shape[0]), "sh_degree": int(scene.get("sh_degree", 0)),
            "width": int(cam.width), "height": int(cam.height),
            "parallelism": (f"tile bands x{world}" if bands else (f"views x{world}" if world > 1 else "single view")),
            "l2": "no flush: per-frame inputs (%.0f MB) exceed the 126 MB L2" % mb}


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        return os.cpu_count() or 1


def run_reference(args):
    """The reference arm: the oracle's C port of tilesplat.render 'reference' (float64), WHOLE frames on all of
    this host's cores; rank 0 only (the other ranks of a torchrun launch exit without work)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2505_24796_b200 import synthetic

    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_threads()))
    scene, cams = synthetic.config_scene(args.config, args.scale)
    cam = cams[0]
    for _ in range(max(args.warmup, 0)):
        cpu_reference_frame(scene, cam)
    times = []
    detail = None
    for _ in range(args.steps):
        s_, detail = cpu_reference_frame(scene, cam)
        times.append(s_)
    mean_s = sum(times) / len(times)
    fps = 1.0 / mean_s
    n = max(world, args.gpus)
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": n,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.config == "c3" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(args, scene, cam, n),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": int(os.environ["OMP_NUM_THREADS"]),
                         "kind": "port",
                         "sample": "oracle C port (float64 restatement of tilesplat.render 'reference'): whole "
                                   "frames (project + build_tiles + blend of every tile), one camera"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "detail": detail,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------ GPU side

def blend_ablation(tcgs, cloud, cam, dev, reps=10):
    """The paper's alpha-blend ablation on B200: K7 alone, re-run on one binned
    frame, for every alpha mode (Frag2Mat on tcgen05: hi/lo and the paper's K8 vector; off: the FFMA quadratic
    form) x EarlyCull on/off.  Device ms per launch (CUDA events on the launching stream) + fragment counts."""
    import torch

    from paper_2505_24796_b200.raster import camera_struct

    out = {}
    for spec in ("tcgs", "tcgs-fp16", "tcgs-ffma"):
        for ec in (True, False):
            r = tcgs.Renderer(dev, tcgs.make_backend(spec, use_early_cull=ec), schedule="dynamic")
            f = r.render_frame(cloud, cam, timed=False)
            c = camera_struct(cam)
            o = r._opts()
            rgb, T, cnt = r.outputs(c.width, c.height)
            st = torch.cuda.current_stream(dev).cuda_stream

            def k7():
                rc = r.lib.tcgs_blend(cloud.P, c, o, r.ws.data_ptr(), r.ws.numel(), r.max_splats, rgb.data_ptr(),
                                      T.data_ptr(), cnt.data_ptr(), st)
                if rc:
                    raise RuntimeError(f"tcgs_blend rc={rc}")

            for _ in range(2):
                k7()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(dev)
            e0.record()
            for _ in range(reps):
                k7()
            e1.record()
            torch.cuda.synchronize(dev)
            s_ = f.stats
            out[f"{spec}/earlycull_{'on' if ec else 'off'}"] = {
                "blend_ms": e0.elapsed_time(e1) / reps, "f_blend": s_.f_blend, "f_cull": s_.f_cull,
                "exp_calls": s_.exp_calls, "pixels_terminated": s_.pixels_terminated}
            del r
    base = out["tcgs-ffma/earlycull_off"]["blend_ms"]
    for v in out.values():
        v["speedup_vs_ffma_no_earlycull"] = base / v["blend_ms"]
    return out


def run_tcgs(args):
    import torch
    import torch.distributed as dist

    import paper_2505_24796_b200 as tcgs
    from paper_2505_24796_b200 import shard, synthetic

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    bands_mode = args.config == "c3"

    scene, cams = synthetic.config_scene(args.config, args.scale)
    base = cams[0]
    per_rank = args.steps + args.warmup
    my_views = rank_views(cams, base, per_rank, rank, world, bands_mode)

    cloud = tcgs.GaussianCloud.from_arrays(scene, dev)
    stream = torch.cuda.current_stream(dev)
    if bands_mode:
        if world == 1 and not dist.is_initialized():
            dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % (29500 + os.getpid() % 1000),
                                    rank=0, world_size=1)
        br = shard.BandRenderer(dev, args.backend, output=args.band_output if world > 1 else "gather")
        r = br.r
        st0 = br.render(cloud, base, with_stats=True).stats  # sizes the workspace

        def frame(cam, ev=None):
            return br.render(cloud, cam, with_stats=False, timers=ev)
    else:
        # the single-camera path: one renderer, one stream, frames back to back (K7's dynamic tile queue)
        r = tcgs.Renderer(dev, args.backend, coverage=args.coverage, schedule="dynamic")
        st0 = r.render_frame(cloud, base, timed=False).stats  # sizes the workspace

        def frame(cam, ev=None):
            return r.launch(cloud, cam, timers=ev)

    for k in range(args.warmup):
        frame(my_views[k])
    torch.cuda.synchronize(dev)

    # ---- timed region: K lone frames, inputs resident in HBM
    nev = 5 if bands_mode else 4
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(nev)] for _ in range(args.steps)]
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    launches0 = r.lib.tcgs_launch_count()
    with ClockSampler(local) as clk:
        start.record(stream)
        for k in range(args.steps):
            frame(my_views[args.warmup + k], evs[k])
        stop.record(stream)
        torch.cuda.synchronize(dev)
    launches = r.lib.tcgs_launch_count() - launches0
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(stop)
    pre_ms = [e[0].elapsed_time(e[1]) for e in evs]
    bin_ms = [e[1].elapsed_time(e[2]) for e in evs]
    blend_ms = [e[2].elapsed_time(e[3]) for e in evs]
    gather_ms = [e[3].elapsed_time(e[4]) for e in evs] if bands_mode else None
    ms_max, blend_max = max_over_ranks([ms, sum(blend_ms) / len(blend_ms)], dev, world)
    if bands_mode:
        st_last = br.render(cloud, my_views[-1], with_stats=True).local.stats
    else:
        rc, st_last = r.read_stats(cloud.P)

    # ---- views in flight: many cameras at once (16 streams, one fused K1 per group of 8 views)
    inflight = None
    vr = None
    if not bands_mode and not args.no_in_flight:
        vr = tcgs.ViewRenderer(dev, args.backend, max(1, args.streams), coverage=args.coverage)
        vr.warm(cloud, base)
        group = max(0, min(args.view_group, max(1, args.streams), 8))
        n_if = max(args.steps, 2 * max(1, args.streams))
        views_if = [my_views[k % len(my_views)] for k in range(n_if)]

        def frames_if(lst):
            if not group:
                for cam in lst:
                    vr.launch(cloud, cam)
                return
            for g0 in range(0, len(lst), group):
                vr.launch_group(cloud, lst[g0:g0 + group])

        frames_if(views_if[:2 * group or 2])
        vr.join()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        frames_if(views_if)
        vr.join()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ti = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(ti, op=dist.ReduceOp.MAX)
        inflight = {"value": world * n_if / (float(ti.item()) / 1e3), "unit": "frames/s", "frames_per_rank": n_if,
                    "streams": max(1, args.streams), "view_group": group,
                    "what": "independent cameras rendered concurrently: one workspace + CUDA stream per view in "
                            "flight, one fused K1 pass per group of views (tcgs_preprocess_views), static K7 "
                            "schedule; every frame fully re-projected, re-binned and re-blended"}

    # ---- end to end through the public API: host scene -> device, render, image -> host
    e2e = None
    if not args.no_e2e:
        feats_key = "features" if scene["sh_degree"] > 0 else "colors"
        host = {k: torch.as_tensor(np.ascontiguousarray(scene[k])).pin_memory()
                for k in ("means", "scales", "rotations", "opacities", feats_key)}
        dev_bufs = {k: torch.empty_like(v, device=dev) for k, v in host.items()}
        out_host = torch.empty((base.height, base.width, 3), dtype=torch.float32).pin_memory()
        stats_bytes = int(r.lib.tcgs_counters_bytes())
        h2d = sum(v.numel() * v.element_size() for v in host.values())
        d2h = (out_host.numel() * 4 if (rank == 0 or not bands_mode) else 0) + stats_bytes
        e2e_steps = max(3, min(args.steps, 20))

        def e2e_frame(cam):  # bands mode: every rank uploads the scene, renders its band, rank 0 reads back
            for k, v in host.items():
                dev_bufs[k].copy_(v, non_blocking=True)
            c = tcgs.GaussianCloud(dev_bufs["means"], dev_bufs["scales"], dev_bufs["rotations"],
                                   dev_bufs["opacities"], dev_bufs[feats_key],
                                   scene["sh_degree"] if scene["sh_degree"] > 0 else -1)
            bf = br.render(c, cam, with_stats=True)  # stats: one all-reduce of 6 counters
            if rank == 0:
                out_host.copy_(bf.rgb, non_blocking=True)
            torch.cuda.synchronize(dev)

        if bands_mode:
            for k in range(2):
                e2e_frame(my_views[k])
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            for k in range(e2e_steps):
                e2e_frame(my_views[k % len(my_views)])
            torch.cuda.synchronize(dev)
            e2e_s = time.perf_counter() - t0
        else:
            # the public host-frame API: upload / render / read back overlapped on three streams
            from paper_2505_24796_b200.pipeline import FramePipeline

            pipe = FramePipeline(r)
            hs = dict(host)
            hs["features"] = hs.pop(feats_key)
            sh = scene["sh_degree"] if scene["sh_degree"] > 0 else -1
            outs = [torch.empty((base.height, base.width, 3), dtype=torch.float32).pin_memory() for _ in range(2)]
            for k in range(2):
                pipe.result(pipe.submit(hs, sh, my_views[k], outs[k % 2]))
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            t0 = time.perf_counter()
            tickets = []
            for k in range(e2e_steps):
                tickets.append(pipe.submit(hs, sh, my_views[k % len(my_views)], outs[k % 2]))
                if len(tickets) >= 2:
                    pipe.result(tickets.pop(0))  # the image and FragmentStats are on the host
            for tk in tickets:
                pipe.result(tk)
            e2e_s = time.perf_counter() - t0
        te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        frames_e2e = e2e_steps if bands_mode else world * e2e_steps
        e2e = {"value": frames_e2e / float(te.item()), "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": e2e_steps,
               "path": ("pinned host scene -> H2D -> tcgs render -> D2H RGB + FragmentStats, every step"
                        + ("" if bands_mode else "; FramePipeline overlaps H2D(k+1) / render(k) / D2H(k-1)"))}
        # what bounds it: the step's H2D bytes against this link's measured pinned-copy bandwidth
        per_rank_fps = e2e["value"] / (1 if bands_mode else world)
        e2e["h2d_achieved_GBps"] = h2d * per_rank_fps / 1e9
        e2e["h2d_link_GBps"] = pinned_h2d_GBps(host, dev)
        if vr is not None:
            e2e["resident_scene"] = e2e_resident(vr, cloud, my_views, base, dev, world, dist)

    ablation = None
    if world == 1 and not bands_mode and not args.no_ablation:
        ablation = blend_ablation(tcgs, cloud, base, dev)

    if bands_mode:
        br.close()  # unmaps / frees the peer frame (collective)
    if rank != 0:
        if dist.is_initialized():
            dist.destroy_process_group()
        return

    frames = args.steps if bands_mode else world * args.steps
    value = frames / (ms_max / 1e3)
    blend_avg = sum(blend_ms) / len(blend_ms)
    peaks, peak_kind = measured_peaks()
    traffic = profile_traffic(args.config)
    clocks = clk.summary()
    # K7 algorithmic work: F_alpha = f_blend + f_cull + pixels_terminated fragments, 16 flops each
    # (length-8 dot = 2*8 flops, src/tilesplat/tensor_path.py:40,53); ex2 = f_blend + terminated.
    F_alpha = st_last.f_blend + st_last.f_cull + st_last.pixels_terminated
    tc_tflops = 16.0 * F_alpha / (blend_avg * 1e-3) / 1e12
    ex2_rate = (st_last.f_blend + st_last.pixels_terminated) / (blend_avg * 1e-3)
    sm_mhz = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    ex2_peak = 148 * 16 * sm_mhz * 1e6  # MUFU: 16 ex2/clk/SM (nominal)
    issue = issue_roofline(traffic, blend_avg, clocks)
    tensor = {"achieved": tc_tflops, "peak": peaks["bf16_tflops"], "unit": "TFLOP/s",
              "frac": tc_tflops / peaks["bf16_tflops"], "peak_kind": peak_kind,
              "work": "16 flops x F_alpha (F_alpha = f_blend + f_cull + pixels_terminated)"}
    mufu = {"achieved": ex2_rate, "peak": ex2_peak, "unit": "ex2/s", "frac": ex2_rate / ex2_peak,
            "peak_kind": "nominal 16/clk/SM at the sampled SM clock", "work": "f_blend + pixels_terminated ex2"}
    if issue:
        roof = {"kernel": "K7 render_kernel (alpha + blend)", "bound": "issue", "achieved": issue["achieved"],
                "peak": issue["peak"], "unit": "warp-instructions/s", "frac": issue["frac"],
                "traffic": (traffic or {}).get("bytes_per_launch"), "traffic_source": (traffic or {}).get("source"),
                "issue": issue, "tensor": tensor, "mufu": mufu}
    else:  # no committed instruction count for this workload: the tensor-pipe fraction, labelled as such
        roof = {"kernel": "K7 render_kernel (alpha + blend)", "bound": "tensor", "achieved": tc_tflops,
                "peak": peaks["bf16_tflops"], "unit": "TFLOP/s", "frac": tc_tflops / peaks["bf16_tflops"],
                "traffic": None, "note": "K7 is issue-bound; no committed ncu instruction count for this config",
                "tensor": tensor, "mufu": mufu}
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = cpu_threads()
        os.environ["OMP_NUM_THREADS"] = str(threads)
        times, det = cpu_frames(scene, base, args.cpu_seconds)
        mean_s = sum(times) / len(times)
        cpu = {"value": 1.0 / mean_s, "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": f"oracle C port of tilesplat.render 'reference' (float64, OpenMP over tiles): "
                         f"{len(times)} whole frame(s) of view 0 (project + build_tiles + blend of every tile)",
               "detail": {**det, "frames": len(times)}}
    stage = {"preprocess": sum(pre_ms) / len(pre_ms), "binning": sum(bin_ms) / len(bin_ms), "blend": blend_avg}
    if gather_ms:
        stage["gather"] = sum(gather_ms) / len(gather_ms)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "frames/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_max / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if bands_mode else "weak",
        "vs_baseline": None,
        "dtype": "f64 preprocess / fp16-hi-lo tcgen05 alpha, fp32 blend",
        "data": "synthetic (SURVEY.md Appendix B generators; random scene, no dataset)",
        "config": bench_config(args, scene, base, world),
        "backend": args.backend,
        "what": ("one 4K frame at a time, tile-row bands across the ranks" if bands_mode else
                 "single-camera frames back to back on one stream (a new view each frame)"),
        "coverage": args.coverage,
        "band_output": (args.band_output if world > 1 else "local") if bands_mode else None,
        "alpha_blend_ms": blend_avg,
        "alpha_blend_ms_max_over_ranks": blend_max,
        "stage_ms": stage,
        "stage_rooflines": stage_rooflines(scene, cloud.P, st_last, stage, peaks, base),
        "frame_stats": {**st_last.to_dict(), "n_visible": st_last.n_visible},
        "roofline": roof,
        "views_in_flight": inflight,
        "alpha_blend_ablation": ablation,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def relaunch_under_torchrun(args) -> int:
    """``--gpus N`` (N > 1) outside torchrun: start N ranks of this script, one per GPU."""
    import socket
    import subprocess

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    _, world, _ = dist_env()
    launched = "WORLD_SIZE" in os.environ
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and not launched:
        sys.exit(relaunch_under_torchrun(args))
    if launched and world != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(2)
    run_tcgs(args)


if __name__ == "__main__":
    main()
