"""Host-resident frames at copy-engine speed: upload, render and read back overlapped.

The reference's ``render(scene, cam)`` (src/tilesplat/raster.py:161) takes the
scene from host memory on every call.  Done naively on the GPU, each frame is
three serial steps: H2D of the scene (236 MB at SH3 for 1M Gaussians,
PCIe-bound), the render on the SMs, and D2H of the image.  ``FramePipeline``
runs them on three CUDA streams with double-buffered device inputs and
outputs.  Frame k+1 uploads while frame k renders and frame k-1's image
comes back, so a stream of host frames runs at the rate of its slowest engine
instead of the sum of all three.

    pipe = FramePipeline(Renderer("cuda"))
    t = [pipe.submit(host_scene, sh_degree, cam, out=pinned_rgb) for cam in cams]
    rgb, stats = pipe.result(t[0])

``host_scene`` holds pinned CPU tensors ``means, scales, rotations,
opacities, features``.  Ordering is enforced with events only; there is no
host synchronisation until ``result``.  At most ``depth`` frames are in
flight: ``submit`` collects frame k-depth first.
"""

from __future__ import annotations

import ctypes

import torch

from . import _abi
from .raster import FragmentStats, GaussianCloud, Renderer

_KEYS = ("means", "scales", "rotations", "opacities", "features")


class FramePipeline:
    def __init__(self, renderer: Renderer, depth: int = 2):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        self.r = renderer
        self.dev = renderer.device
        self.depth = depth
        self.h2d = torch.cuda.Stream(self.dev)
        self.comp = torch.cuda.Stream(self.dev)
        self.d2h = torch.cuda.Stream(self.dev)
        nb = int(self.r.lib.tcgs_counters_bytes())
        self.snap = [torch.empty(nb, dtype=torch.uint8).pin_memory() for _ in range(depth)]
        self.inputs = [None] * depth
        self.outputs = [None] * depth
        self.ev_in_free = [None] * depth   # K1 of the slot's last frame has read its inputs
        self.ev_out_free = [None] * depth  # the slot's last image has reached the host
        self.pending = {}
        self.n = 0

    def _slot_inputs(self, s: int, host: dict):
        cur = self.inputs[s]
        if cur is None or any(cur[k].shape != host[k].shape or cur[k].dtype != host[k].dtype for k in _KEYS):
            cur = {k: torch.empty(host[k].shape, dtype=host[k].dtype, device=self.dev) for k in _KEYS}
            self.inputs[s] = cur
        return cur

    def _slot_outputs(self, s: int, W: int, H: int):
        cur = self.outputs[s]
        if cur is None or cur[0].shape != (H, W, 3):
            cur = (torch.zeros((H, W, 3), dtype=torch.float32, device=self.dev),
                   torch.ones((H, W), dtype=torch.float32, device=self.dev),
                   torch.zeros((H, W), dtype=torch.int32, device=self.dev))
            self.outputs[s] = cur
        return cur

    def _collect(self, k: int):
        rec = self.pending[k]
        if "stats" in rec:
            return
        rec["ev"].synchronize()
        st = _abi.Stats()
        rc = self.r.lib.tcgs_decode_stats(ctypes.c_void_p(self.snap[rec["slot"]].data_ptr()), self.r._opts(), st)
        rec["rc"] = rc
        rec["stats"] = FragmentStats(f_blend=st.f_blend, f_cull=st.f_cull, f_skip=st.f_skip, exp_calls=st.exp_calls,
                                     n_splats=st.n_splats, dropped=st.dropped,
                                     pixels_terminated=st.pixels_terminated, n_visible=st.n_visible)

    def submit(self, host: dict, sh_degree: int, cam, out: torch.Tensor | None = None) -> int:
        """Enqueue one frame; returns a ticket for ``result``.  ``out``: pinned [H,W,3] f32 host image."""
        k = self.n
        s = k % self.depth
        if k - self.depth in self.pending:
            self._collect(k - self.depth)  # its snapshot / image slot is about to be reused
        self.n += 1
        H, W = int(cam.height), int(cam.width)
        if out is None:
            out = torch.empty((H, W, 3), dtype=torch.float32).pin_memory()
        dev_in = self._slot_inputs(s, host)
        with torch.cuda.stream(self.h2d):
            if self.ev_in_free[s] is not None:
                self.h2d.wait_event(self.ev_in_free[s])
            for name in _KEYS:
                dev_in[name].copy_(host[name], non_blocking=True)
            in_ready = torch.cuda.Event()
            in_ready.record(self.h2d)
        cloud = GaussianCloud(dev_in["means"], dev_in["scales"], dev_in["rotations"], dev_in["opacities"].reshape(-1),
                              dev_in["features"], int(sh_degree))
        outs = self._slot_outputs(s, W, H)
        with torch.cuda.stream(self.comp):
            self.comp.wait_event(in_ready)
            if self.ev_out_free[s] is not None:
                self.comp.wait_event(self.ev_out_free[s])
            self.r.preprocess(cloud, cam)
            in_free = torch.cuda.Event()
            in_free.record(self.comp)
            self.ev_in_free[s] = in_free
            rgb, _, _ = self.r.bin_blend(cloud, cam, outputs=outs)
            _abi.check(self.r.lib.tcgs_snapshot_stats(ctypes.c_void_p(self.r.ws.data_ptr()),
                                                      ctypes.c_void_p(self.snap[s].data_ptr()),
                                                      ctypes.c_void_p(self.comp.cuda_stream)), "tcgs_snapshot_stats")
            done = torch.cuda.Event()
            done.record(self.comp)
        with torch.cuda.stream(self.d2h):
            self.d2h.wait_event(done)
            out.copy_(rgb, non_blocking=True)
            back = torch.cuda.Event()
            back.record(self.d2h)
            self.ev_out_free[s] = back
        ev = torch.cuda.Event()
        ev.record(self.d2h)
        self.pending[k] = {"slot": s, "out": out, "ev": ev, "host": host, "sh": int(sh_degree), "cam": cam}
        return k

    def result(self, k: int):
        """(host RGB [H,W,3] f32, FragmentStats) of ticket ``k`` (blocks until it is done)."""
        self._collect(k)
        rec = self.pending.pop(k)
        if rec["rc"] == _abi.TCGS_ERR_CAPACITY:
            # the frame needed more splats than the workspace holds: re-render it synchronously
            self.sync()
            self.r.max_splats = int(rec["stats"].n_splats * 1.25) + 1024
            dev = {name: rec["host"][name].to(self.dev) for name in _KEYS}
            cloud = GaussianCloud(dev["means"], dev["scales"], dev["rotations"], dev["opacities"].reshape(-1),
                                  dev["features"], rec["sh"])
            f = self.r.render_frame(cloud, rec["cam"], timed=False)
            rec["out"].copy_(f.rgb)
            return rec["out"], f.stats
        _abi.check(rec["rc"], "tcgs_decode_stats")
        return rec["out"], rec["stats"]

    def sync(self):
        for st in (self.h2d, self.comp, self.d2h):
            st.synchronize()
