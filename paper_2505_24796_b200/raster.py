"""Host side of the B200 TC-GS renderer: the reference's render entry point,
re-implemented over libtcgs.so.

Mirrors tilesplat.raster (/root/reference/pkg/src/tilesplat/raster.py):
``render(scene, cam, backend) -> (ImageBuffer, FragmentStats)`` (:161-201),
``make_backend`` (:149-158), ``FragmentStats`` (:19-49), ``ImageBuffer``
(:52-64), ``computation_model`` (:204-208) and the module constants
(:15-16).  Scenes and cameras are duck-typed against tilesplat.scene
(Scene/Gaussian3D/Camera, src/tilesplat/scene.py:24-80), so the reference's own
objects are accepted unchanged.

There is exactly one implementation behind it (sm_100a CUDA through the C
ABI); the backend string only selects a compile-time alpha mode of the same
blend kernel.  Nothing here computes pixels on the CPU.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _abi

ALPHA_CULL_THRESHOLD = 1.0 / 255.0  # src/tilesplat/raster.py:15
TERMINATION_THRESHOLD = 0.0001      # src/tilesplat/raster.py:16
TILE_SIZE = 16                      # src/tilesplat/tiling.py:11


@dataclass
class FragmentStats:
    """Counts of blended, culled, and skipped fragments plus exp calls (src/tilesplat/raster.py:19-49)."""

    f_blend: int = 0
    f_cull: int = 0
    f_skip: int = 0
    exp_calls: int = 0
    n_splats: int = 0
    dropped: int = 0
    pixels_terminated: int = 0
    stage_ms: dict = field(default_factory=dict)
    n_visible: int = 0

    @property
    def total_fragments(self) -> int:
        return self.f_blend + self.f_cull + self.f_skip

    def counts(self) -> tuple[int, int, int, int]:
        return (self.f_blend, self.f_cull, self.f_skip, self.exp_calls)

    def to_dict(self) -> dict:
        return {
            "f_blend": self.f_blend,
            "f_cull": self.f_cull,
            "f_skip": self.f_skip,
            "exp_calls": self.exp_calls,
            "N": self.n_splats,
            "dropped": self.dropped,
            "pixels_terminated": self.pixels_terminated,
            "stage_ms": dict(self.stage_ms),
        }


@dataclass
class ImageBuffer:
    """Row-major float RGB image in [0, 1] (src/tilesplat/raster.py:52-64), plus the final
    transmittance ``T`` and per-pixel contributor counts ``n_contrib``."""

    rgb: np.ndarray  # (height, width, 3) float64
    T: np.ndarray | None = None
    n_contrib: np.ndarray | None = None

    @property
    def width(self) -> int:
        return self.rgb.shape[1]

    @property
    def height(self) -> int:
        return self.rgb.shape[0]


@dataclass(frozen=True)
class Backend:
    """Selects the alpha mode of the single B200 blend kernel.

    ``arith`` says what the kernel computes (it is not the reference's emulation model):
    ``"fp32"`` (CUDA-core quadratic form), ``"fp16-hilo"`` (tcgen05 fp16, hi/lo split vector, ~22 bits),
    ``"fp16"`` (tcgen05 fp16, the paper's length-8 vector); ``coords`` is "local" (G2L) or "global".
    """

    name: str
    alpha_mode: int
    early_cull: bool = True
    coords: str = "local"
    arith: str = "fp16-hilo"

    def tile_evaluator(self, *a, **k):  # the per-fragment protocol (raster.py:86-107) is not crossed
        raise NotImplementedError("the B200 renderer blends whole tiles on the GPU; use render()")


# This package's own specs: spec -> (alpha mode, arith)
_SPECS = {
    "tcgs": (_abi.ALPHA_TC_HILO, "fp16-hilo"),
    "tcgs-hilo": (_abi.ALPHA_TC_HILO, "fp16-hilo"),
    "tcgs-fp16": (_abi.ALPHA_TC_K8, "fp16"),
    "tcgs-k8": (_abi.ALPHA_TC_K8, "fp16"),
    "tcgs-ffma": (_abi.ALPHA_FFMA, "fp32"),
}
# The reference's spellings (src/tilesplat/raster.py:149-158, cli.py:15).
REFERENCE_SPECS = ("reference", "frag2mat", "frag2mat-fp16", "frag2mat-tf32")


def make_backend(spec: str = "tcgs", coords: str | None = None, batch_width: int = 16,
                 use_early_cull: bool = True) -> Backend:
    """Backend factory mirroring src/tilesplat/raster.py:149-158 (ValueError on unknown specs, coordinate modes
    and batch widths, as src/tilesplat/tensor_path.py:175-181).  ``coords=None`` is the reference's default
    ("global") for the reference's spellings and "local" for this package's own ``tcgs*`` specs.

    How each reference spelling maps onto the one B200 kernel (nothing is silently approximated):

    * ``"reference"`` -- ReferenceBackend (raster.py:77-107): alpha = o exp(-q/2) for every active fragment,
      cull on alpha < 1/255 afterwards (EarlyCull off), in fp32 on CUDA cores.  ``coords`` and
      ``use_early_cull`` are ignored, as the reference ignores them.
    * ``"frag2mat"`` -- exact arithmetic (float64 in the reference) is served by the fp32 CUDA-core form in
      tile-local coordinates whatever ``coords`` says: exact global and local evaluation agree to 1e-5
      (the reference's own criterion 1, tests/test_acceptance.py:44-68), and fp32 global coordinates would
      only lose precision.  ``use_early_cull`` selects the cull order (tensor_path.py:148-160).
    * ``"frag2mat-fp16"`` -- the paper's fp16 length-8 vector on tcgen05, in local (G2L) or global
      coordinates (the precision ablation).
    * ``"frag2mat-tf32"`` -- not reproduced: ValueError.
    * ``"tcgs"`` (this package's default), ``"tcgs-fp16"``, ``"tcgs-ffma"`` -- hi/lo fp16 tcgen05, paper
      K8, fp32 CUDA cores; tile-local coordinates only.

    ``batch_width`` only validates: the kernel's batch (32 live Gaussians per MMA) does not change the
    output, which the reference requires of every batch width (tests/test_tensor_path.py:155-165).
    """
    own = spec in _SPECS
    if coords is None:
        coords = "local" if own else "global"
    if coords not in ("global", "local"):
        raise ValueError(f"unknown coordinate mode {coords!r}")
    if batch_width < 1:
        raise ValueError("batch width must be positive")
    if spec == "reference":
        return Backend("reference", _abi.ALPHA_FFMA, False, "local", "fp32")
    if spec == "frag2mat":
        return Backend(f"frag2mat-exact-{coords}", _abi.ALPHA_FFMA, bool(use_early_cull), "local", "fp32")
    if spec == "frag2mat-fp16":
        mode = _abi.ALPHA_TC_K8 if coords == "local" else _abi.ALPHA_TC_K8_GLOBAL
        return Backend(f"frag2mat-fp16-{coords}", mode, bool(use_early_cull), coords, "fp16")
    if spec == "frag2mat-tf32":
        raise ValueError("backend 'frag2mat-tf32': the B200 kernel does not reproduce the tf32 arithmetic model "
                         "(use 'frag2mat' for exact or 'frag2mat-fp16' for the paper's fp16 path)")
    if spec not in _SPECS:
        raise ValueError(f"unknown backend {spec!r}")
    if coords != "local":
        raise ValueError(f"backend {spec!r} evaluates in tile-local coordinates only (global coordinates: "
                         "'frag2mat-fp16' with coords='global')")
    mode, arith = _SPECS[spec]
    return Backend(spec, mode, bool(use_early_cull), "local", arith)


def computation_model(stats: FragmentStats, k_alpha: float, k_cull: float, k_blend: float) -> float:
    """Fragment-cost model (src/tilesplat/raster.py:204-208)."""
    if k_alpha < 0 or k_cull < 0 or k_blend < 0:
        raise ValueError("cost constants must be non-negative")
    return k_blend * stats.f_blend + (k_cull + k_alpha) * (stats.f_blend + stats.f_cull)


# ----------------------------------------------------------------------------- scene / camera packing

@dataclass
class GaussianCloud:
    """Device-resident SoA Gaussians (the layout libtcgs.so consumes).

    ``features`` is RGB [P,3] when ``sh_degree == -1`` (the reference's
    Gaussian3D.color) or SH coefficients [P,(d+1)^2,3] for degree d.
    """

    means: torch.Tensor
    scales: torch.Tensor
    rotations: torch.Tensor
    opacities: torch.Tensor
    features: torch.Tensor
    sh_degree: int = -1

    @property
    def P(self) -> int:
        return int(self.means.shape[0])

    @property
    def dtype_code(self) -> int:
        return _abi.F64 if self.means.dtype == torch.float64 else _abi.F32

    @classmethod
    def from_arrays(cls, d: dict, device=None, dtype=None) -> "GaussianCloud":
        """From a dict of arrays (paper_2505_24796_b200.synthetic scenes)."""
        device = torch.device(device or "cuda")
        sh = int(d.get("sh_degree", 0))
        feats = d["features"] if (sh > 0 and "features" in d) else d["colors"]
        sh_code = sh if (sh > 0 and "features" in d) else -1
        if dtype is None:
            dtype = torch.float64 if np.asarray(d["means"]).dtype == np.float64 else torch.float32

        def t(x):
            return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype).to(device).contiguous()

        return cls(t(d["means"]), t(d["scales"]), t(d["rotations"]), t(np.asarray(d["opacities"]).reshape(-1)),
                   t(feats), sh_code)

    @classmethod
    def from_scene(cls, scene, device=None) -> "GaussianCloud":
        """From a reference ``tilesplat.Scene`` (float64, colours used directly)."""
        g = tuple(scene.gaussians)
        if len(g) == 0:
            z = np.zeros((0, 3))
            return cls.from_arrays({"means": z, "scales": z, "rotations": np.zeros((0, 4)),
                                    "opacities": np.zeros(0), "colors": z}, device, torch.float64)
        arr = {
            "means": np.array([x.mean for x in g], np.float64),
            "scales": np.array([x.scale for x in g], np.float64),
            "rotations": np.array([x.rotation for x in g], np.float64),
            "opacities": np.array([x.opacity for x in g], np.float64),
            "colors": np.array([x.color for x in g], np.float64),
        }
        return cls.from_arrays(arr, device, torch.float64)

    def _c(self) -> _abi.Scene:
        s = _abi.Scene()
        s.P = self.P
        s.sh_degree = self.sh_degree
        s.dtype = self.dtype_code
        for name in ("means", "scales", "rotations", "opacities", "features"):
            t = getattr(self, name)
            if not t.is_contiguous():
                raise ValueError(f"{name} must be contiguous")
            if t.dtype != self.means.dtype:
                raise ValueError("all Gaussian arrays must share one dtype")
            setattr(s, name, t.data_ptr() if t.numel() else 0)
        return s


def camera_struct(cam) -> _abi.Camera:
    """Pack a tilesplat.Camera-like object (src/tilesplat/scene.py:50-68)."""
    c = _abi.Camera()
    v = np.asarray(cam.view, dtype=np.float64).reshape(16)
    for i in range(16):
        c.view[i] = float(v[i])
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.near_plane = float(getattr(cam, "near", 0.2))
    c.width, c.height = int(cam.width), int(cam.height)
    if c.width <= 0 or c.height <= 0:
        raise ValueError("image dimensions must be positive")
    if not (c.fx > 0 and c.fy > 0):
        raise ValueError("focal lengths must be positive")
    if not c.near_plane > 0:
        raise ValueError("near clip must be positive")
    return c


# ----------------------------------------------------------------------------- the renderer

@dataclass
class Frame:
    rgb: torch.Tensor        # [H,W,3] f32 (device)
    T: torch.Tensor          # [H,W]   f32 (device)
    n_contrib: torch.Tensor  # [H,W]   i32 (device)
    stats: FragmentStats | None


class Renderer:
    """Owns the device workspace and the output buffers; renders frames stream-ordered.

    The library allocates nothing: the workspace is a torch uint8 tensor sized by
    tcgs_workspace_size and grown (with one re-render) when a frame overflows
    the splat capacity.
    """

    def __init__(self, device=None, backend="tcgs", max_splats: int | None = None, coverage: str = "square",
                 schedule: str = "dynamic"):
        if coverage not in _abi.COVERAGE:
            raise ValueError(f"coverage must be one of {sorted(_abi.COVERAGE)}")
        if schedule not in _abi.SCHEDULE:
            raise ValueError(f"schedule must be one of {sorted(_abi.SCHEDULE)}")
        self.coverage = _abi.COVERAGE[coverage]  # "square": the reference's tiles; "ellipse": opt-in, fewer splats
        # K7 tile assignment: "dynamic" (a global queue; best for a lone frame) or "static" (frames in flight)
        self.schedule = _abi.SCHEDULE[schedule]
        self.lib = _abi.load()
        self.device = torch.device(device or "cuda")
        if self.device.type != "cuda":
            raise ValueError("the B200 renderer needs a CUDA device")
        with torch.cuda.device(self.device):
            _abi.check(self.lib.tcgs_device_check(), "device check")
        self.backend = backend if isinstance(backend, Backend) else make_backend(backend)
        self.max_splats = max_splats
        self.ws = None
        self.ws_key = None
        self._out = {}
        self._timing = False  # render_frame: the library times the stages (tcgs_opts.timing)
        self._dump = None     # (beta, class) device tensors: the K7 debug dump (dump_frame / blend_lists)

    def _opts(self, band=None, debug=False, defer_colour=False) -> _abi.Opts:
        o = _abi.Opts()
        o.timing = 1 if self._timing else 0
        if self._dump is not None:
            o.dump_beta, o.dump_class = self._dump[0].data_ptr(), self._dump[1].data_ptr()
        o.defer_colour = 1 if defer_colour else 0
        o.tile_row_begin, o.tile_row_end = (band if band is not None else (0, 0))
        o.alpha_mode = self.backend.alpha_mode
        o.early_cull = 1 if self.backend.early_cull else 0
        o.debug = 1 if debug else 0
        o.coverage = self.coverage
        o.schedule = self.schedule
        return o

    def workspace(self, P: int, W: int, H: int, cap: int, min_bytes: int = 0) -> torch.Tensor:
        need = max(int(self.lib.tcgs_workspace_size(P, W, H, cap)), int(min_bytes))
        if self.ws is None or self.ws.numel() < need:
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        self.ws_key = (P, W, H, cap)
        return self.ws

    def outputs(self, W: int, H: int):
        key = (W, H)
        if key not in self._out:
            self._out[key] = (torch.zeros((H, W, 3), dtype=torch.float32, device=self.device),
                              torch.ones((H, W), dtype=torch.float32, device=self.device),
                              torch.zeros((H, W), dtype=torch.int32, device=self.device))
        return self._out[key]

    def capacity(self, P: int) -> int:
        if self.max_splats is None:
            self.max_splats = max(1 << 16, 16 * P)
        return self.max_splats

    def launch(self, cloud: GaussianCloud, cam, band=None, debug=False, outputs=None, timers=None):
        """Enqueue K1..K7 on the current stream (no host synchronisation)."""
        ev = timers
        if ev:
            ev[0].record()
        self.preprocess(cloud, cam, band, debug)
        if ev:
            ev[1].record()
        return self.bin_blend(cloud, cam, band, outputs, ev)

    def preprocess(self, cloud: GaussianCloud, cam, band=None, debug=False, defer_colour=False) -> None:
        """K1 (band-agnostic: its tile rectangles serve any band binned afterwards).  ``defer_colour``: geometry
        only -- call ``colour`` for the band before binning it."""
        c = camera_struct(cam)
        cap = self.capacity(cloud.P)
        ws = self.workspace(cloud.P, c.width, c.height, cap)
        st = torch.cuda.current_stream(self.device).cuda_stream
        _abi.check(self.lib.tcgs_preprocess(cloud._c(), c, self._opts(band, debug, defer_colour), ws.data_ptr(),
                                            ws.numel(), cap, st), "tcgs_preprocess")

    def colour(self, cloud: GaussianCloud, cam, band=None) -> None:
        """The deferred colours of the Gaussians whose tile rectangle meets ``band`` (tile rows [y0, y1))."""
        c = camera_struct(cam)
        st = torch.cuda.current_stream(self.device).cuda_stream
        _abi.check(self.lib.tcgs_colour(cloud._c(), c, self._opts(band), self.ws.data_ptr(), self.ws.numel(),
                                        self.capacity(cloud.P), st), "tcgs_colour")

    def bin_blend(self, cloud: GaussianCloud, cam, band=None, outputs=None, timers=None):
        """K2-K6 and K7 for ``band`` (tile rows [y0, y1); None = the whole frame) after ``preprocess``."""
        c = camera_struct(cam)
        cap = self.capacity(cloud.P)
        ws = self.ws
        rgb, T, cnt = outputs if outputs is not None else self.outputs(c.width, c.height)
        o = self._opts(band)
        st = torch.cuda.current_stream(self.device).cuda_stream
        ev = timers
        _abi.check(self.lib.tcgs_bin(cloud.P, c, o, ws.data_ptr(), ws.numel(), cap, st), "tcgs_bin")
        if ev:
            ev[2].record()
        _abi.check(self.lib.tcgs_blend(cloud.P, c, o, ws.data_ptr(), ws.numel(), cap, rgb.data_ptr(), T.data_ptr(),
                                       cnt.data_ptr(), st), "tcgs_blend")
        if ev:
            ev[3].record()
        return rgb, T, cnt

    def read_stats(self, P: int, band=None) -> tuple[int, FragmentStats]:
        st_ = _abi.Stats()
        o = self._opts(band)
        rc = self.lib.tcgs_read_stats(self.ws.data_ptr(), P, o, st_, torch.cuda.current_stream(self.device).cuda_stream)
        fs = FragmentStats(f_blend=st_.f_blend, f_cull=st_.f_cull, f_skip=st_.f_skip, exp_calls=st_.exp_calls,
                           n_splats=st_.n_splats, dropped=st_.dropped, pixels_terminated=st_.pixels_terminated,
                           n_visible=st_.n_visible)
        if o.timing:  # src/tilesplat/raster.py:196-200: exactly these three keys
            fs.stage_ms = {"preprocess": float(st_.ms_preprocess), "sorting": float(st_.ms_sort),
                           "blending": float(st_.ms_blend)}
        return rc, fs

    def finish(self, cloud: GaussianCloud, cam, band=None, with_stats=True, outputs=None) -> Frame:
        """K2-K7 for ``band`` after ``preprocess`` + the frame's stats (re-running K1 if the splat
        capacity had to grow)."""
        for _attempt in range(3):
            rgb, T, cnt = self.bin_blend(cloud, cam, band, outputs=outputs)
            rc, fs = self.read_stats(cloud.P, band)
            if rc == _abi.TCGS_ERR_CAPACITY:
                self.max_splats = int(fs.n_splats * 1.25) + 1024
                self.preprocess(cloud, cam, band)
                continue
            _abi.check(rc, "tcgs_read_stats")
            return Frame(rgb, T, cnt, fs)
        raise RuntimeError("splat capacity could not be satisfied")

    def render_frame(self, cloud: GaussianCloud, cam, band=None, debug=False, timed=True) -> Frame:
        """One frame, synchronously, with its FragmentStats (stage device times from the library when
        ``timed``: tcgs_opts.timing -> tcgs_stats.ms_*)."""
        with torch.cuda.device(self.device):
            self._timing = bool(timed)
            try:
                for _attempt in range(3):
                    rgb, T, cnt = self.launch(cloud, cam, band, debug)
                    rc, fs = self.read_stats(cloud.P, band)
                    if rc == _abi.TCGS_ERR_CAPACITY:
                        self.max_splats = int(fs.n_splats * 1.25) + 1024
                        continue
                    _abi.check(rc, "tcgs_read_stats")
                    return Frame(rgb, T, cnt, fs)
            finally:
                self._timing = False
        raise RuntimeError("splat capacity could not be satisfied")

    def dump_frame(self, cloud: GaussianCloud, cam, band=None, host: bool = True):
        """Debug: render one frame with K7's beta/classification dump (the a19 tolerance oracle).

        Returns (Frame, beta float32 [N,256], cls uint8 [N,256]) as numpy: for tile-list entry e (the order of
        ``tile_lists``) and tile pixel i = 16 row + col, beta = K7's exponent in log2 units and cls = 1 cull /
        2 blend / 3 terminate / 4 dead on the whole tile (box test) / 0 not evaluated (NaN beta)."""
        f = self.render_frame(cloud, cam, band, timed=False)  # sizes the workspace and learns N
        n = max(int(f.stats.n_splats), 1)
        beta = torch.full((n, 256), float("nan"), dtype=torch.float32, device=self.device)
        cls = torch.zeros((n, 256), dtype=torch.uint8, device=self.device)
        self._dump = (beta, cls)
        try:
            f = self.render_frame(cloud, cam, band, timed=False)
        finally:
            self._dump = None
        n = int(f.stats.n_splats)
        if not host:  # device tensors (full-size frames: the caller fetches the rows it needs)
            return f, beta[:n], cls[:n]
        return f, beta[:n].cpu().numpy(), cls[:n].cpu().numpy()

    # -- debug accessors (tests) ------------------------------------------------------------
    def tile_lists(self, P: int, cam, band=None):
        """(offsets int64 [n_tiles+1], ids int32 [N]) of the last frame, as numpy (CSR, row-major tiles)."""
        c = camera_struct(cam)
        o = self._opts(band)
        rc, fs = self.read_stats(P, band)
        _abi.check(rc, "tcgs_read_stats")
        n = fs.n_splats
        ids = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        ty0, ty1 = band if band is not None else (0, (c.height + 15) // 16)
        nt = ((c.width + 15) // 16) * (ty1 - ty0)
        ranges = torch.empty((max(nt, 1), 2), dtype=torch.int32, device=self.device)
        st = torch.cuda.current_stream(self.device).cuda_stream
        _abi.check(self.lib.tcgs_copy_lists(self.ws.data_ptr(), P, c, o, self.max_splats, ids.data_ptr(),
                                            ranges.data_ptr(), st), "tcgs_copy_lists")
        r = ranges[:nt].cpu().numpy().astype(np.int64)
        counts = np.where(r[:, 1] > r[:, 0], r[:, 1] - r[:, 0], 0)
        offsets = np.zeros(nt + 1, np.int64)
        np.cumsum(counts, out=offsets[1:])
        ids_np = ids[:n].cpu().numpy()
        # ranges are contiguous and ordered, so CSR offsets index ids directly
        assert all(r[t, 0] == offsets[t] for t in range(nt) if counts[t] > 0)
        return offsets, ids_np

    def projection(self, P: int, cam):
        c = camera_struct(cam)
        d = self.device
        vis = torch.empty(max(P, 1), dtype=torch.uint8, device=d)
        m2 = torch.empty((max(P, 1), 2), dtype=torch.float64, device=d)
        con = torch.empty((max(P, 1), 3), dtype=torch.float64, device=d)
        dep = torch.empty(max(P, 1), dtype=torch.float64, device=d)
        rad = torch.empty(max(P, 1), dtype=torch.int32, device=d)
        rgb = torch.empty((max(P, 1), 3), dtype=torch.float32, device=d)
        st = torch.cuda.current_stream(d).cuda_stream
        _abi.check(self.lib.tcgs_copy_projection(self.ws.data_ptr(), P, c, self.max_splats, vis.data_ptr(),
                                                 m2.data_ptr(), con.data_ptr(), dep.data_ptr(), rad.data_ptr(),
                                                 rgb.data_ptr(), st), "tcgs_copy_projection")
        torch.cuda.synchronize(d)
        return {k: v[:P].cpu().numpy() for k, v in
                dict(visible=vis, mean2d=m2, inv_cov=con, depth=dep, radius=rad, rgb=rgb).items()}

    def blend_lists(self, mean2d, conic, opacity, colors, offsets, ids, cam, band=None, dump=False):
        """K7 alone on caller-given projected records and CSR tile lists (tests/KATs).  ``dump``: also return
        K7's beta / classification per (list entry, tile pixel), as ``dump_frame`` does."""
        d = self.device
        c = camera_struct(cam)
        P = int(np.asarray(mean2d).reshape(-1, 2).shape[0])

        def t(x, dt):
            return torch.as_tensor(np.ascontiguousarray(x), dtype=dt, device=d).contiguous()

        m2 = t(np.asarray(mean2d, np.float64).reshape(-1, 2), torch.float64)
        con = t(np.asarray(conic, np.float64).reshape(-1, 3), torch.float64)
        op = t(np.asarray(opacity, np.float64).reshape(-1), torch.float64)
        col = t(np.asarray(colors, np.float32).reshape(-1, 3), torch.float32)
        off = t(np.asarray(offsets, np.int64), torch.int64)
        idt = t(np.asarray(ids, np.int32).reshape(-1) if np.size(ids) else np.zeros(1, np.int32), torch.int32)
        ws = self.workspace(P, c.width, c.height, 1)
        rgb = torch.zeros((c.height, c.width, 3), dtype=torch.float32, device=d)
        T = torch.ones((c.height, c.width), dtype=torch.float32, device=d)
        cnt = torch.zeros((c.height, c.width), dtype=torch.int32, device=d)
        n = max(int(np.size(ids)), 1)
        if dump:
            self._dump = (torch.full((n, 256), float("nan"), dtype=torch.float32, device=d),
                          torch.zeros((n, 256), dtype=torch.uint8, device=d))
        o = self._opts(band)
        dumped, self._dump = self._dump, None
        st = torch.cuda.current_stream(d).cuda_stream
        with torch.cuda.device(d):
            _abi.check(self.lib.tcgs_blend_lists(P, m2.data_ptr(), con.data_ptr(), op.data_ptr(), col.data_ptr(),
                                                 off.data_ptr(), idt.data_ptr(), c, o, ws.data_ptr(), ws.numel(),
                                                 rgb.data_ptr(), T.data_ptr(), cnt.data_ptr(), st), "tcgs_blend_lists")
            rc, fs = self.read_stats(P, band)
            _abi.check(rc, "tcgs_read_stats")
        if dump:
            m = int(np.size(ids))
            return Frame(rgb, T, cnt, fs), dumped[0][:m].cpu().numpy(), dumped[1][:m].cpu().numpy()
        return Frame(rgb, T, cnt, fs)


class ViewRenderer:
    """Renders many independent views of one scene with ``n_streams`` workspaces on as many CUDA streams.

    Frame i runs on stream i % n_streams, so the latency-bound stages of one view (K1, the sort passes)
    overlap the tail of the previous view's K7 instead of leaving SMs idle between frames.  Views are
    independent (the reference renders each camera separately, src/tilesplat/raster.py:161), so this
    changes no result.  ``join()`` makes the caller's current stream wait for every view.
    """

    def __init__(self, device=None, backend="tcgs", n_streams: int = 2, coverage: str = "square"):
        self.device = torch.device(device or "cuda")
        # several frames share the GPU: K7's static schedule leaves a staggered tail the other streams fill
        self.renderers = [Renderer(self.device, backend, coverage=coverage, schedule="static")
                          for _ in range(n_streams)]
        self.streams = [torch.cuda.Stream(self.device) for _ in range(n_streams)]
        self.outputs = [None] * n_streams
        self.k = 0

    @property
    def lib(self):
        return self.renderers[0].lib

    def warm(self, cloud: GaussianCloud, cam) -> FragmentStats:
        """Size every workspace (one synchronous frame each); returns the stats of ``cam``."""
        st = None
        for r, s in zip(self.renderers, self.streams):
            with torch.cuda.stream(s):
                st = r.render_frame(cloud, cam, timed=False).stats
        return st

    def launch(self, cloud: GaussianCloud, cam, timers=None):
        """Enqueue one view on the next stream (ordered after the caller's current stream)."""
        i = self.k % len(self.streams)
        self.k += 1
        s = self.streams[i]
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            return self.renderers[i].launch(cloud, cam, timers=timers)

    def launch_group(self, cloud: GaussianCloud, cams, timers=None):
        """Enqueue ``len(cams)`` views (at most the stream count and ``_abi.MAX_VIEWS_PER_PASS``) with ONE
        fused K1 pass (``tcgs_preprocess_views``: each Gaussian's inputs are read once for every camera),
        then each view's K2-K7 on its own stream.  Returns the views' (rgb, T, n_contrib) outputs.
        ``timers`` (4 events) bracket the fused K1 and the last view's binning / blending."""
        n = len(cams)
        if not 1 <= n <= min(len(self.streams), _abi.MAX_VIEWS_PER_PASS):
            raise ValueError(f"a view group holds 1..{min(len(self.streams), _abi.MAX_VIEWS_PER_PASS)} cameras")
        idx = [(self.k + j) % len(self.streams) for j in range(n)]
        self.k += n
        rs = [self.renderers[i] for i in idx]
        ss = [self.streams[i] for i in idx]
        cs = [camera_struct(c) for c in cams]
        cap = max(r.capacity(cloud.P) for r in rs)  # one workspace layout for the whole pass
        # the pass checks every view against ONE ws_bytes: grow each workspace to the largest view's need
        need = max(int(self.lib.tcgs_workspace_size(cloud.P, c.width, c.height, cap)) for c in cs)
        wss = []
        for r, c in zip(rs, cs):
            r.max_splats = cap
            wss.append(r.workspace(cloud.P, c.width, c.height, cap, min_bytes=need))
        ps = ss[0]  # the fused K1 runs on the first view's stream, after every view's previous frame
        ps.wait_stream(torch.cuda.current_stream(self.device))
        for s in ss[1:]:
            ps.wait_stream(s)
        cam_arr = (_abi.Camera * n)(*cs)
        ws_arr = (ctypes.c_void_p * n)(*[w.data_ptr() for w in wss])
        ev = timers
        with torch.cuda.stream(ps):
            if ev:
                ev[0].record()
            _abi.check(self.lib.tcgs_preprocess_views(cloud._c(), cam_arr, n, rs[0]._opts(), ws_arr,
                                                      min(w.numel() for w in wss), cap, ps.cuda_stream),
                       "tcgs_preprocess_views")
            if ev:
                ev[1].record()
        outs = []
        for j, (r, s, cam) in enumerate(zip(rs, ss, cams)):
            s.wait_stream(ps)
            with torch.cuda.stream(s):
                outs.append(r.bin_blend(cloud, cam, timers=ev if (ev and j == n - 1) else None))
        return outs

    def join(self):
        cur = torch.cuda.current_stream(self.device)
        for s in self.streams:
            cur.wait_stream(s)


_DEFAULT = {}


def _renderer(device, backend) -> Renderer:
    key = (str(device), backend if isinstance(backend, Backend) else make_backend(backend))
    if key not in _DEFAULT:
        _DEFAULT[key] = Renderer(device, backend)
    return _DEFAULT[key]


def render(scene, cam, backend="reference", device=None) -> tuple[ImageBuffer, FragmentStats]:
    """Drop-in for ``tilesplat.render(scene, cam, backend="reference")`` (src/tilesplat/raster.py:161-201).

    ``scene`` is a reference ``Scene`` (or a ``GaussianCloud``); background is
    black; boundary tiles are full 16x16 tiles with out-of-image pixels masked.
    The default backend is the reference's ("reference": alpha for every active
    fragment, the cull on alpha afterwards); pass ``"tcgs"`` for the tensor-core
    path with EarlyCull.  ``stats.stage_ms`` holds exactly the reference's keys
    (preprocess / sorting / blending), as device times.  Returns float64 RGB
    like the reference plus ``T``/``n_contrib`` extras.
    """
    if isinstance(backend, str):
        backend = make_backend(backend)
    device = torch.device(device or "cuda")
    cloud = scene if isinstance(scene, GaussianCloud) else GaussianCloud.from_scene(scene, device)
    r = _renderer(device, backend)
    frame = r.render_frame(cloud, cam)
    img = ImageBuffer(frame.rgb.double().cpu().numpy(), frame.T.double().cpu().numpy(),
                      frame.n_contrib.cpu().numpy())
    return img, frame.stats


def rasterize(means, scales, rotations, opacities, features, sh_degree: int, cameras, backend="tcgs",
              band=None, renderer: Renderer | None = None, n_streams: int = 8) -> dict:
    """Batched entry: render every camera of ``cameras`` from device tensors.

    Views are independent, so they run ``n_streams`` at a time on their own workspaces and CUDA
    streams (``ViewRenderer``), in groups of up to ``n_streams // 2`` (<= 8) that share one fused K1
    pass (``tcgs_preprocess_views``); every view's outputs are copied out on its own stream and its
    FragmentStats snapshotted without a host sync.  Returns ``rgb [V,H,W,3] f32``, ``T [V,H,W] f32``,
    ``n_contrib [V,H,W] i32`` (device tensors) and per-view FragmentStats.
    """
    import ctypes

    cloud = GaussianCloud(means.contiguous(), scales.contiguous(), rotations.contiguous(),
                          opacities.reshape(-1).contiguous(), features.contiguous(), int(sh_degree))
    cams = list(cameras)
    if not cams:
        raise ValueError("no cameras")
    if renderer is not None or band is not None or n_streams <= 1:
        r = renderer or Renderer(means.device, backend)
        frames = [r.render_frame(cloud, cam, band=band) for cam in cams[:1]]
        out = [(frames[0].rgb.clone(), frames[0].T.clone(), frames[0].n_contrib.clone(), frames[0].stats)]
        for cam in cams[1:]:
            f = r.render_frame(cloud, cam, band=band)
            out.append((f.rgb.clone(), f.T.clone(), f.n_contrib.clone(), f.stats))
    else:
        vr = ViewRenderer(means.device, backend, n_streams)
        vr.warm(cloud, cams[0])
        nb = int(vr.lib.tcgs_counters_bytes())
        snaps = torch.empty((len(cams), nb), dtype=torch.uint8).pin_memory()
        outs = []
        # groups of views share one fused K1 pass; two groups in flight (the next group's K1 overlaps this
        # group's binning and blending)
        group = max(1, min(_abi.MAX_VIEWS_PER_PASS, len(vr.streams) // 2))
        for v0 in range(0, len(cams), group):
            n = len(vr.streams)
            idx = [(vr.k + j) % n for j in range(min(group, len(cams) - v0))]
            res = vr.launch_group(cloud, cams[v0:v0 + len(idx)])
            for j, (i, (rgb, T, cnt)) in enumerate(zip(idx, res)):
                with torch.cuda.stream(vr.streams[i]):
                    outs.append((rgb.clone(), T.clone(), cnt.clone()))
                    _abi.check(vr.lib.tcgs_snapshot_stats(ctypes.c_void_p(vr.renderers[i].ws.data_ptr()),
                                                          ctypes.c_void_p(snaps[v0 + j].data_ptr()),
                                                          ctypes.c_void_p(vr.streams[i].cuda_stream)), "snapshot")
        vr.join()
        torch.cuda.current_stream(means.device).synchronize()
        out = []
        for v, cam in enumerate(cams):
            st = _abi.Stats()
            rc = vr.lib.tcgs_decode_stats(ctypes.c_void_p(snaps[v].data_ptr()), vr.renderers[0]._opts(), st)
            if rc == _abi.TCGS_ERR_CAPACITY:  # this view needed a bigger workspace: redo it synchronously
                f = vr.renderers[0].render_frame(cloud, cam, timed=False)
                out.append((f.rgb.clone(), f.T.clone(), f.n_contrib.clone(), f.stats))
                continue
            _abi.check(rc, "tcgs_decode_stats")
            out.append((*outs[v], FragmentStats(f_blend=st.f_blend, f_cull=st.f_cull, f_skip=st.f_skip,
                                                exp_calls=st.exp_calls, n_splats=st.n_splats, dropped=st.dropped,
                                                pixels_terminated=st.pixels_terminated, n_visible=st.n_visible)))
    return {"rgb": torch.stack([o[0] for o in out]), "T": torch.stack([o[1] for o in out]),
            "n_contrib": torch.stack([o[2] for o in out]), "stats": [o[3] for o in out]}
