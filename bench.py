"""Benchmark: TC-GS forward render on B200 (BASELINE.json metric, config 2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

One step = one full frame of the hot path (K1 preprocess -> K2-K6 binning ->
K7 tensor-core alpha + blend) for the config-2 workload: 1M synthetic
Gaussians with SH degree 3 at 1920x1080, inputs resident in HBM (the 236 MB
scene exceeds the 126 MB L2, so no flush is needed between frames).  N > 1
shards camera views across ranks (one process per GPU, no collective on the
data path; weak scaling: every rank renders K frames).  ``--config c3``
renders 4K frames split into tile-row bands across the ranks with one NCCL
gather to rank 0 per frame (strong scaling).

The JSON line carries the device-timed throughput (`value`), the end-to-end
throughput through the public API with host buffers (`e2e`), the roofline of
the dominant kernel (K7), the CPU baseline (the oracle's C port of the
reference renderer on this host's cores), clocks and the kernel-launch count.
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
            time.sleep(0.004)

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


def stage_rooflines(scene, P, st, stage_ms, peaks, cam, group=0):
    """Algorithmic bytes per stage / isolated stage time, against the measured HBM copy peak.
    K1: P x (inputs + 76 B of outputs); binning: P (8 B depth + 4 B index) read + write, N (2 B tile key +
    4 B id) written and sorted once, N x 2 B of ranges; K7: N x 52 B (id + 48 B record) + 20 B per pixel.
    The fused multi-view K1 reads the inputs once per group of views: P x (inputs / group + 76 B) per view."""
    feats = 3 * 4 * ((scene.get("sh_degree", 0) + 1) ** 2 if scene.get("sh_degree", 0) > 0 else 1)
    N = st.n_splats
    work = {"preprocess": P * (44 + feats + 76), "binning": P * 12 * 2 + N * 6 * 2 + N * 2,
            "blend": N * 52 + cam.width * cam.height * 20}
    if group > 1:
        work["preprocess_fused_per_view"] = P * ((44 + feats) / group + 76)
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
    the committed ncu capture (smsp__inst_executed.sum), the duration from this run's CUDA events."""
    inst = (traffic or {}).get("warp_inst_per_launch")
    mhz = (clocks or {}).get("sm_mhz") or 1965.0
    if not inst:
        return None
    peak = 4 * 148 * mhz * 1e6
    ach = inst / (blend_ms * 1e-3)
    return {"achieved_warp_inst_per_s": ach, "peak_warp_inst_per_s": peak, "frac": ach / peak,
            "warp_inst_per_launch": inst, "note": "instructions from the committed ncu profile; clock = median "
                                                  "SM clock sampled during the timed region"}


def profile_traffic():
    """K7 DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) from the newest committed
    ncu --set full summary under profiles/ (scripts/ncu_summary.py), if present."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_k7_ncu.json")))  # r1_ < r1e_ < r1j_ < ...
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

def cpu_reference_frame(scene, cam, rows):
    """The oracle's C port of the reference renderer (project, build_tiles, blend) on host cores.
    Blend runs on a band of `rows` tile rows and is extrapolated to the frame."""
    import oracle

    t0 = time.perf_counter()
    colors = scene["colors"]
    if scene.get("sh_degree", 0) > 0:
        colors = oracle.sh_color(scene["means"], scene["features"], scene["sh_degree"], cam.view)
    proj = oracle.project(scene["means"], scene["scales"], scene["rotations"], cam)
    t1 = time.perf_counter()
    off, ids = oracle.build_tiles(proj, cam)
    t2 = time.perf_counter()
    tiles_y = (cam.height + 15) // 16
    r0 = max(0, tiles_y // 2 - rows // 2)
    r1 = min(tiles_y, r0 + rows)
    oracle.blend(proj, off, ids, scene["opacities"], colors, cam, band=(r0, r1))
    t3 = time.perf_counter()
    frame_s = (t1 - t0) + (t2 - t1) + (t3 - t2) * tiles_y / (r1 - r0)
    return frame_s, {"preprocess_s": t1 - t0, "sort_s": t2 - t1, "blend_band_s": t3 - t2,
                     "band_rows": r1 - r0, "tile_rows": tiles_y}


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
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2505_24796_b200 import synthetic

    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_threads()))
    scene, cams = synthetic.config_scene(args.config, args.scale)
    cam = cams[0]
    rows = 2
    for _ in range(max(args.warmup, 0)):
        cpu_reference_frame(scene, cam, rows)
    times = []
    detail = None
    for _ in range(args.steps):
        s, detail = cpu_reference_frame(scene, cam, rows)
        times.append(s)
    mean_s = sum(times) / len(times)
    fps = 1.0 / mean_s
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
        "scaling": "strong" if args.config == "c3" else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(args, scene, cam, world),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": int(os.environ["OMP_NUM_THREADS"]),
                         "kind": "port",
                         "sample": f"oracle C port (float64 restatement of tilesplat.render 'reference'): full "
                                   f"project + build_tiles, blend on {detail['band_rows']} of {detail['tile_rows']} "
                                   f"tile rows extrapolated to the frame"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "detail": detail,
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------ GPU side

def run_tcgs(args):
    import torch
    import torch.distributed as dist

    import paper_2505_24796_b200 as tcgs
    from paper_2505_24796_b200 import _abi, shard, synthetic

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    bands_mode = args.config == "c3"

    scene, cams = synthetic.config_scene(args.config, args.scale)
    base = cams[0]
    per_rank = args.steps + args.warmup
    if bands_mode:
        my_views = view_cameras(base, per_rank)  # every rank renders its band of the same frames
    else:
        pool = cams if len(cams) > 1 else view_cameras(base, world * per_rank)
        b0, b1 = shard.view_blocks(len(pool), world)[rank]
        mine = pool[b0:b1] or pool[:1]
        my_views = [mine[k % len(mine)] for k in range(per_rank)]

    cloud = tcgs.GaussianCloud.from_arrays(scene, dev)
    if bands_mode:
        if world == 1 and not dist.is_initialized():
            dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % (29500 + os.getpid() % 1000),
                                    rank=0, world_size=1)
        br = shard.BandRenderer(dev, args.backend, output=args.band_output if world > 1 else "gather")
        r = br.r
        first = br.render(cloud, base, with_stats=True)  # sizes the workspace
        st0 = first.stats
    else:
        vr = tcgs.ViewRenderer(dev, args.backend, max(1, args.streams), coverage=args.coverage)
        r = vr.renderers[0]
        st0 = vr.warm(cloud, base)  # sizes the workspaces; stats of the base view
    stream = torch.cuda.current_stream(dev)

    group = 0 if bands_mode else max(0, min(args.view_group, max(1, args.streams), 8))

    def frame(cam, ev=None):
        if bands_mode:
            return br.render(cloud, cam, with_stats=False, timers=ev)
        return vr.launch(cloud, cam, timers=ev)

    def frames(k0, n, ev=None):  # frames k0 .. k0+n-1 of my_views: one at a time, or in fused-K1 groups
        if not group:
            for k in range(k0, k0 + n):
                frame(my_views[k], ev[k - k0] if ev else None)
            return
        for g0 in range(k0, k0 + n, group):
            g1 = min(g0 + group, k0 + n)
            vr.launch_group(cloud, my_views[g0:g1], timers=ev[g0 - k0] if ev else None)

    frames(0, args.warmup)
    if not bands_mode:
        vr.join()
    torch.cuda.synchronize(dev)

    # ---- timed region: K frames, inputs resident in HBM
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
        frames(args.warmup, args.steps, evs)
        if not bands_mode:
            vr.join()
        stop.record(stream)
        torch.cuda.synchronize(dev)
    launches = r.lib.tcgs_launch_count() - launches0
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(stop)
    if group:  # one event set per group (recorded on its first frame): fused K1 per view, last view's K2-K7
        evs = [evs[k] for k in range(0, args.steps, group)]
        sizes = [min(group, args.steps - k) for k in range(0, args.steps, group)]
        pre_ms = [e[0].elapsed_time(e[1]) / n for e, n in zip(evs, sizes)]
    else:
        pre_ms = [e[0].elapsed_time(e[1]) for e in evs]
    bin_ms = [e[1].elapsed_time(e[2]) for e in evs]
    blend_ms = [e[2].elapsed_time(e[3]) for e in evs]
    gather_ms = [e[3].elapsed_time(e[4]) for e in evs] if bands_mode else None
    t = torch.tensor([ms, sum(blend_ms) / len(blend_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, blend_max = float(t[0].item()), float(t[1].item())

    # per-frame stats of this rank's last timed view (device counters; the band's in bands mode)
    # isolated per-stage device times (one view at a time on one stream): with several views in flight the
    # timed region overlaps stages of different views, so its per-stage events include interference
    iso = None
    if not bands_mode and len(vr.renderers) > 1:
        r0 = vr.renderers[0]
        iso_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(min(10, args.steps))]
        for k, ev in enumerate(iso_ev):
            r0.launch(cloud, my_views[args.warmup + k], timers=ev)
        torch.cuda.synchronize(dev)
        iso = {"preprocess": sum(e[0].elapsed_time(e[1]) for e in iso_ev) / len(iso_ev),
               "binning": sum(e[1].elapsed_time(e[2]) for e in iso_ev) / len(iso_ev),
               "blend": sum(e[2].elapsed_time(e[3]) for e in iso_ev) / len(iso_ev)}
        if group > 1:  # the fused K1 alone: one pass over the scene for `group` views, per view
            gev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            vr.launch_group(cloud, my_views[args.warmup:args.warmup + group], timers=gev)
            vr.join()
            torch.cuda.synchronize(dev)
            iso["preprocess_fused_per_view"] = gev[0].elapsed_time(gev[1]) / group
    if bands_mode:
        st_last = br.render(cloud, my_views[-1], with_stats=True).local.stats
    else:
        last = vr.renderers[(args.warmup + args.steps - 1 + len(vr.renderers)) % len(vr.renderers)]
        rc, st_last = last.read_stats(cloud.P)

    # ---- end to end through the public API: host scene -> device, render, image -> host
    e2e = None
    if not args.no_e2e:
        feats_key = "features" if scene["sh_degree"] > 0 else "colors"
        host = {k: torch.as_tensor(np.ascontiguousarray(scene[k])).pin_memory()
                for k in ("means", "scales", "rotations", "opacities", feats_key)}
        dev_bufs = {k: torch.empty_like(v, device=dev) for k, v in host.items()}
        out_host = torch.empty((base.height, base.width, 3), dtype=torch.float32).pin_memory()
        stats_bytes = 9 * 8
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
        if not bands_mode:
            e2e["resident_scene"] = e2e_resident(vr, cloud, my_views, base, dev, world, dist)

    if bands_mode:
        br.close()  # unmaps / frees the peer frame (collective)
    if rank != 0:
        if dist.is_initialized():
            dist.destroy_process_group()
        return

    frames = args.steps if bands_mode else world * args.steps
    value = frames / (ms_max / 1e3)
    blend_avg = iso["blend"] if iso else sum(blend_ms) / len(blend_ms)
    peaks, peak_kind = measured_peaks()
    traffic = profile_traffic()
    # K7 algorithmic work: F_alpha = f_blend + f_cull + pixels_terminated fragments, 16 flops each
    # (length-8 dot = 2*8 flops, src/tilesplat/tensor_path.py:40,53); ex2 = f_blend + terminated.
    F_alpha = st_last.f_blend + st_last.f_cull + st_last.pixels_terminated
    tc_tflops = 16.0 * F_alpha / (blend_avg * 1e-3) / 1e12
    ex2_rate = (st_last.f_blend + st_last.pixels_terminated) / (blend_avg * 1e-3)
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    ex2_peak = 148 * 16 * sm_mhz * 1e6  # MUFU: 16 ex2/clk/SM (nominal)
    clocks = clk.summary()
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        threads = cpu_threads()
        os.environ["OMP_NUM_THREADS"] = str(threads)
        s, det = cpu_reference_frame(scene, base, rows=2)
        cpu = {"value": 1.0 / s, "unit": "frames/s", "cores": threads, "kind": "port",
               "sample": f"oracle C port of tilesplat.render 'reference' (float64, OpenMP over tiles), view 0: full "
                         f"project + build_tiles, blend on {det['band_rows']}/{det['tile_rows']} tile rows "
                         f"extrapolated to the frame",
               "detail": det}
    stage = {"preprocess": sum(pre_ms) / len(pre_ms), "binning": sum(bin_ms) / len(bin_ms),
             "blend": sum(blend_ms) / len(blend_ms)}
    if gather_ms:
        stage["gather"] = sum(gather_ms) / len(gather_ms)
    if iso:
        stage = {"isolated": iso, "in_flight": stage}
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
        "views_in_flight": 1 if bands_mode else max(1, args.streams),
        "view_group": group,
        "coverage": args.coverage,
        "band_output": (args.band_output if world > 1 else "local") if bands_mode else None,
        "alpha_blend_ms": blend_avg,
        "stage_rooflines": stage_rooflines(scene, cloud.P, st_last, iso or stage, peaks, base, group),
        "alpha_blend_ms_max_over_ranks": blend_max,
        "stage_ms": stage,
        "frame_stats": {**st_last.to_dict(), "n_visible": st_last.n_visible},
        "roofline": {"kernel": "K7 render_kernel (alpha + blend)", "bound": "tensor", "achieved": tc_tflops,
                     "peak": peaks["bf16_tflops"], "unit": "TFLOP/s", "frac": tc_tflops / peaks["bf16_tflops"],
                     "traffic": (traffic or {}).get("bytes_per_launch") if args.config == "c2" else None,
                     "traffic_source": (traffic or {}).get("source"), "peak_kind": peak_kind,
                     "work": "16 flops x F_alpha (F_alpha = f_blend + f_cull + pixels_terminated)",
                     "mufu": {"achieved_ex2_per_s": ex2_rate, "peak_ex2_per_s": ex2_peak,
                              "frac": ex2_rate / ex2_peak, "peak_kind": "nominal 16/clk/SM"},
                     # the committed K7 profile is of the C2 workload: its instruction count only applies there
                     "issue": issue_roofline(traffic, blend_avg, clocks) if args.config == "c2" else None},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_tcgs(args)


if __name__ == "__main__":
    main()
