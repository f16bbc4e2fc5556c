"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the TC-GS render path.

A float64 restatement of the reference renderer ``tilesplat``
(/root/reference/pkg/src/tilesplat; see tcgs_oracle.c for the per-function
file:line citations).  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package, and only as the checker / the timed CPU baseline -- never as
the thing measured or shipped.  The product path (``paper_2505_24796_b200``)
never imports it and fails loudly when its CUDA extension is missing.

Parity is pinned against golden vectors the reference itself produced
(tests/golden/make_golden.py, tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
BUILD_DIR = os.path.join(HERE, "_build")
LIB_PATH = os.path.join(BUILD_DIR, "libtcgs_oracle.so")
SRC_PATH = os.path.join(HERE, "tcgs_oracle.c")

TILE_SIZE = 16
ALPHA_CULL_THRESHOLD = 1.0 / 255.0
TERMINATION_THRESHOLD = 0.0001

_lib = None


def build(force: bool = False) -> str:
    """Compile the C restatement (gcc, -ffp-contract=off keeps numpy's op order)."""
    if not force and os.path.exists(LIB_PATH) and os.path.getmtime(LIB_PATH) >= os.path.getmtime(SRC_PATH):
        return LIB_PATH
    os.makedirs(BUILD_DIR, exist_ok=True)
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
           SRC_PATH, "-o", tmp, "-lm"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


class _OCam(ctypes.Structure):
    _fields_ = [("view", ctypes.c_double * 16), ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double), ("near_", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        lib.oracle_project.restype = ctypes.c_int64
        lib.oracle_project.argtypes = [ctypes.c_int64, P, P, P, ctypes.POINTER(_OCam), P, P, P, P, P]
        lib.oracle_tile_counts.restype = ctypes.c_int64
        lib.oracle_tile_counts.argtypes = [ctypes.c_int64, P, P, P, ctypes.c_int, ctypes.c_int, P]
        lib.oracle_tile_lists.restype = None
        lib.oracle_tile_lists.argtypes = [ctypes.c_int64, P, P, P, P, ctypes.c_int, ctypes.c_int, P, P]
        lib.oracle_blend.restype = None
        lib.oracle_blend.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P, P, P,
                                     P, P, P, P]
        lib.oracle_classify.restype = None
        lib.oracle_classify.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, P, P, P, P, P, P]
        lib.oracle_blend_const_alpha.restype = None
        lib.oracle_blend_const_alpha.argtypes = [ctypes.c_int, P, P, P, P, P, P]
        lib.oracle_sh_color.restype = None
        lib.oracle_sh_color.argtypes = [ctypes.c_int64, ctypes.c_int, P, P, P, P]
        lib.oracle_py_hypot.restype = ctypes.c_double
        lib.oracle_py_hypot.argtypes = [ctypes.c_double, ctypes.c_double]
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def _f64(a, shape_tail=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a


@dataclass
class OCamera:
    """Mirror of tilesplat.scene.Camera (src/tilesplat/scene.py:50-68)."""

    view: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float = 0.2

    @classmethod
    def from_any(cls, cam) -> "OCamera":
        return cls(np.asarray(cam.view, dtype=np.float64).reshape(4, 4), float(cam.fx), float(cam.fy),
                   float(cam.cx), float(cam.cy), int(cam.width), int(cam.height), float(cam.near))

    def _c(self) -> _OCam:
        c = _OCam()
        v = np.ascontiguousarray(self.view, dtype=np.float64).reshape(16)
        for i in range(16):
            c.view[i] = float(v[i])
        c.fx, c.fy, c.cx, c.cy, c.near_ = self.fx, self.fy, self.cx, self.cy, self.near
        c.width, c.height = self.width, self.height
        return c

    @property
    def tiles_x(self) -> int:
        return (self.width + TILE_SIZE - 1) // TILE_SIZE

    @property
    def tiles_y(self) -> int:
        return (self.height + TILE_SIZE - 1) // TILE_SIZE


@dataclass
class Projection:
    visible: np.ndarray   # bool [P]
    mean2d: np.ndarray    # f64 [P,2]
    inv_cov: np.ndarray   # f64 [P,3]  (s11, s12, s22)
    depth: np.ndarray     # f64 [P]
    radius: np.ndarray    # i32 [P]
    dropped: int


def project(means, scales, rotations, cam) -> Projection:
    """src/tilesplat/projection.py:68-134 (project, project_scene)."""
    lib = _load()
    means = _f64(means).reshape(-1, 3)
    scales = _f64(scales).reshape(-1, 3)
    rotations = _f64(rotations).reshape(-1, 4)
    P = means.shape[0]
    cam = OCamera.from_any(cam)
    vis = np.zeros(P, np.uint8)
    mean2d = np.zeros((P, 2))
    inv = np.zeros((P, 3))
    depth = np.zeros(P)
    rad = np.zeros(P, np.int32)
    c = cam._c()
    dropped = lib.oracle_project(P, _p(means), _p(scales), _p(rotations), ctypes.byref(c), _p(vis), _p(mean2d),
                                 _p(inv), _p(depth), _p(rad))
    return Projection(vis.astype(bool), mean2d, inv, depth, rad, int(dropped))


def build_tiles(proj: Projection, cam):
    """src/tilesplat/tiling.py:46-59 -> CSR (offsets[n_tiles+1] int64, ids[N] int32 original ids)."""
    lib = _load()
    cam = OCamera.from_any(cam)
    vis = np.ascontiguousarray(proj.visible.astype(np.uint8))
    P = vis.shape[0]
    nt = cam.tiles_x * cam.tiles_y
    counts = np.zeros(nt, np.int64)
    n = lib.oracle_tile_counts(P, _p(vis), _p(proj.mean2d), _p(proj.radius), cam.tiles_x, cam.tiles_y, _p(counts))
    offsets = np.zeros(nt + 1, np.int64)
    np.cumsum(counts, out=offsets[1:])
    ids = np.zeros(max(int(n), 1), np.int32)
    lib.oracle_tile_lists(P, _p(vis), _p(proj.mean2d), _p(proj.radius), _p(proj.depth), cam.tiles_x, cam.tiles_y,
                          _p(offsets), _p(ids))
    return offsets, ids[: int(n)]


@dataclass
class OracleStats:
    """Mirror of tilesplat.raster.FragmentStats (src/tilesplat/raster.py:19-49)."""

    f_blend: int = 0
    f_cull: int = 0
    f_skip: int = 0
    exp_calls: int = 0
    n_splats: int = 0
    dropped: int = 0
    pixels_terminated: int = 0
    stage_ms: dict = field(default_factory=dict)

    def counts(self):
        return (self.f_blend, self.f_cull, self.f_skip, self.exp_calls)


@dataclass
class OracleFrame:
    rgb: np.ndarray        # f64 [H,W,3]
    T: np.ndarray          # f64 [H,W]
    n_contrib: np.ndarray  # i32 [H,W]
    stats: OracleStats
    offsets: np.ndarray
    ids: np.ndarray
    proj: Projection


def blend(proj: Projection, offsets, ids, opacity, colors, cam, band=None):
    """src/tilesplat/raster.py:110-146 blend_tile over every tile (or a tile-row band)."""
    lib = _load()
    cam = OCamera.from_any(cam)
    H, W = cam.height, cam.width
    r0, r1 = band if band is not None else (0, cam.tiles_y)
    rgb = np.zeros((H, W, 3))
    T = np.ones((H, W))
    cnt = np.zeros((H, W), np.int32)
    st = np.zeros(5, np.int64)
    opacity = _f64(opacity).reshape(-1)
    colors = _f64(colors).reshape(-1, 3)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    if ids.size == 0:
        ids = np.zeros(1, np.int32)
    lib.oracle_blend(W, H, r0, r1, _p(offsets), _p(ids), _p(proj.mean2d), _p(proj.inv_cov), _p(opacity),
                     _p(colors), _p(rgb), _p(T), _p(cnt), _p(st))
    return rgb, T, cnt, st


def render(means, scales, rotations, opacities, colors, cam, early_cull: bool = True) -> OracleFrame:
    """src/tilesplat/raster.py:161-201 render(scene, cam, "reference"), returning T and counts too.

    ``exp_calls`` follows the TC-GS EarlyCull accounting (f_blend +
    pixels_terminated, src/tilesplat/tensor_path.py:148-154) when
    ``early_cull`` else the reference backend's (every active fragment,
    src/tilesplat/raster.py:94).
    """
    import time

    t0 = time.perf_counter()
    proj = project(means, scales, rotations, cam)
    t1 = time.perf_counter()
    offsets, ids = build_tiles(proj, cam)
    t2 = time.perf_counter()
    rgb, T, cnt, st = blend(proj, offsets, ids, opacities, colors, cam)
    t3 = time.perf_counter()
    fb, fc, fs, pt, ns = (int(x) for x in st)
    stats = OracleStats(f_blend=fb, f_cull=fc, f_skip=fs, n_splats=int(ids.size), dropped=proj.dropped,
                        pixels_terminated=pt,
                        exp_calls=(fb + pt) if early_cull else (fb + fc + pt),
                        stage_ms={"preprocess": (t1 - t0) * 1e3, "sorting": (t2 - t1) * 1e3,
                                  "blending": (t3 - t2) * 1e3})
    return OracleFrame(rgb, T, cnt, stats, offsets, ids, proj)


def classify(proj: Projection, offsets, ids, opacity, cam, band=None) -> np.ndarray:
    """Per-fragment classes of the reference blend loop: uint8 [N, 256] (1 cull, 2 blend, 3 terminate, 0 not
    reached / out of the image) for tile-list entry j and tile pixel 16 row + col (tcgs_oracle.c)."""
    lib = _load()
    cam = OCamera.from_any(cam)
    r0, r1 = band if band is not None else (0, cam.tiles_y)
    offsets = np.ascontiguousarray(offsets, dtype=np.int64)
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    n = ids.size
    cls = np.zeros((max(n, 1), 256), np.uint8)
    if n == 0:
        return cls[:0]
    lib.oracle_classify(cam.width, cam.height, r0, r1, _p(offsets), _p(ids), _p(proj.mean2d), _p(proj.inv_cov),
                        _p(_f64(opacity).reshape(-1)), _p(cls))
    return cls


def blend_const_alpha(alphas, colors):
    """Single full tile with per-splat constant alpha (tests/test_raster.py:21-29 evaluator)."""
    lib = _load()
    a = _f64(alphas).reshape(-1)
    c = _f64(colors).reshape(-1, 3)
    n = a.shape[0]
    if n == 0:
        a = np.zeros(1)
        c = np.zeros((1, 3))
    rgb = np.zeros((256, 3))
    T = np.zeros(256)
    cnt = np.zeros(256, np.int32)
    st = np.zeros(4, np.int64)
    lib.oracle_blend_const_alpha(n, _p(a), _p(c), _p(rgb), _p(T), _p(cnt), _p(st))
    return rgb, T, cnt, tuple(int(x) for x in st)


def sh_color(means, feats, sh_degree: int, view) -> np.ndarray:
    """3DGS SH colour restatement (parity UNPINNED for degree >= 1)."""
    lib = _load()
    means = _f64(means).reshape(-1, 3)
    K = (sh_degree + 1) ** 2
    feats = _f64(feats).reshape(-1, K, 3)
    view = _f64(view).reshape(16)
    out = np.zeros((means.shape[0], 3))
    lib.oracle_sh_color(means.shape[0], sh_degree, _p(means), _p(feats), _p(view), _p(out))
    return out


def py_hypot(x: float, y: float) -> float:
    return float(_load().oracle_py_hypot(x, y))


# src/tilesplat/images.py:37-48
def psnr(a: np.ndarray, b: np.ndarray) -> float:
    if a.shape != b.shape:
        raise ValueError(f"image shapes differ: {a.shape} vs {b.shape}")
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(1.0 / mse)


def max_channel_diff(a: np.ndarray, b: np.ndarray) -> float:
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)))) if np.size(a) else 0.0
