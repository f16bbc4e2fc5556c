"""Synthetic scenes and cameras for the BASELINE configs.

``make_camera`` / ``make_scene`` reproduce the reference's test fixtures
(/root/reference/pkg/tests/conftest.py:28-60) draw for draw, so a seed names
the same scene in both code bases.  ``gen_uniform`` (G), ``gen_anisotropic``
(G') and ``gen_ball`` (B) + ``orbit_cameras`` are the BASELINE config
generators; every array is rounded to float32 once so the GPU path and the
float64 reference consume identical values.

Scenes are returned as a plain dict of SoA numpy arrays:
means [P,3], scales [P,3], rotations [P,4] (w,x,y,z), opacities [P],
colors [P,3] and, for sh_degree >= 1, features [P,(d+1)^2,3].
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SH_C0 = 0.28209479177387814  # src/tilesplat/scene.py:11


@dataclass(frozen=True)
class CameraSpec:
    """Pinhole camera, world->camera ``view`` row-major (src/tilesplat/scene.py:50-68)."""

    view: np.ndarray
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int
    near: float = 0.2


def make_camera(width=256, height=256, focal=None, near=0.2) -> CameraSpec:
    """tests/conftest.py:28-39 of the reference."""
    focal = focal or width * 1.2
    return CameraSpec(np.eye(4), float(focal), float(focal), width / 2.0, height / 2.0, width, height, near)


def make_scene(seed, n, depth_range=(4.0, 9.0), xy_spread=1.6, scale_range=(0.15, 0.5),
               opacity_range=(0.15, 0.5)) -> dict:
    """tests/conftest.py:42-60 of the reference, draw order preserved (float64 values)."""
    rng = np.random.default_rng(seed)
    means = np.zeros((n, 3))
    scales = np.zeros((n, 3))
    rots = np.zeros((n, 4))
    opac = np.zeros(n)
    cols = np.zeros((n, 3))
    for i in range(n):
        q = rng.normal(size=4)
        rots[i] = q / np.linalg.norm(q)
        means[i, 0] = rng.uniform(-xy_spread, xy_spread)
        means[i, 1] = rng.uniform(-xy_spread, xy_spread)
        means[i, 2] = rng.uniform(*depth_range)
        scales[i] = rng.uniform(*scale_range, size=3)
        opac[i] = float(rng.uniform(*opacity_range))
        cols[i] = rng.uniform(0.0, 1.0, size=3)
    return {"means": means, "scales": scales, "rotations": rots, "opacities": opac, "colors": cols,
            "sh_degree": 0}


def _finish(d: dict, rng, sh_degree: int) -> dict:
    if sh_degree > 0:
        K = (sh_degree + 1) ** 2
        feats = np.zeros((d["means"].shape[0], K, 3))
        feats[:, 0, :] = (d["colors"] - 0.5) / SH_C0
        feats[:, 1:, :] = rng.normal(0.0, 0.05, size=(d["means"].shape[0], K - 1, 3))
        d["features"] = feats
    d["sh_degree"] = sh_degree
    for k in ("means", "scales", "rotations", "opacities", "colors", "features"):
        if k in d:
            d[k] = np.ascontiguousarray(d[k].astype(np.float32))
    return d


def gen_uniform(P: int, W: int, H: int, seed: int, sh_degree: int = 3, anisotropic: bool = False) -> dict:
    """Generator G (configs 2, 3) and G' (config 5, ``anisotropic``): SURVEY.md Appendix B."""
    rng = np.random.default_rng(seed)
    f = 1.2 * W
    z = rng.uniform(2.0, 20.0, P)
    x = rng.uniform(-1.05, 1.05, P) * z * (W / 2) / f
    y = rng.uniform(-1.05, 1.05, P) * z * (H / 2) / f
    q = rng.normal(size=(P, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    if anisotropic:
        long_ax = np.exp(rng.uniform(math.log(2.0), math.log(16.0), P))
        short = np.exp(rng.uniform(math.log(0.1), math.log(0.5), (P, 2)))
        sigma_px = np.concatenate([long_ax[:, None], short], axis=1)
        opac = rng.uniform(0.01, 0.1, P)
    else:
        sigma_px = np.exp(rng.uniform(math.log(0.5), math.log(8.0), (P, 3)))
        opac = rng.uniform(0.05, 0.95, P)
    scales = sigma_px * (z / f)[:, None]
    colors = rng.uniform(0.0, 1.0, (P, 3))
    d = {"means": np.stack([x, y, z], 1), "scales": scales, "rotations": q, "opacities": opac, "colors": colors}
    return _finish(d, rng, sh_degree)


def gen_ball(P: int, seed: int = 4, sh_degree: int = 3) -> dict:
    """Generator B (config 4): points in a radius-1.5 ball, SURVEY.md Appendix B."""
    rng = np.random.default_rng(seed)
    dirs = rng.normal(size=(P, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    r = 1.5 * rng.uniform(0.0, 1.0, P) ** (1.0 / 3.0)
    means = dirs * r[:, None]
    q = rng.normal(size=(P, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    scales = np.exp(rng.uniform(math.log(0.001), math.log(0.015), (P, 3)))
    opac = rng.uniform(0.05, 0.95, P)
    colors = rng.uniform(0.0, 1.0, (P, 3))
    d = {"means": means, "scales": scales, "rotations": q, "opacities": opac, "colors": colors}
    return _finish(d, rng, sh_degree)


def look_at_view(eye) -> np.ndarray:
    """World->camera view with +z forward, +y down, looking at the origin."""
    eye = np.asarray(eye, dtype=np.float64)
    f = -eye / np.linalg.norm(eye)
    r = np.cross(np.array([0.0, 1.0, 0.0]), f)
    r /= np.linalg.norm(r)
    d = np.cross(f, r)
    R = np.stack([r, d, f])
    view = np.eye(4)
    view[:3, :3] = R
    view[:3, 3] = -R @ eye
    return view


def orbit_cameras(n_views: int = 256, W: int = 1920, H: int = 1080, radius: float = 4.0,
                  height: float = -1.0) -> list:
    """Config 4: n_views cameras on an orbit."""
    f = 1.2 * W
    cams = []
    for k in range(n_views):
        th = 2.0 * math.pi * k / n_views
        eye = (radius * math.cos(th), height, radius * math.sin(th))
        cams.append(CameraSpec(look_at_view(eye), f, f, W / 2.0, H / 2.0, W, H))
    return cams


CONFIGS = {
    # name: (description, builder)
    "c1": "synthetic 10k random Gaussians, SH0, 256x256 (reference conftest make_scene(0, 10000))",
    "c2": "synthetic 1M Gaussians, SH3, 1920x1080, single camera",
    "c3": "synthetic 3M Gaussians, SH3, 3840x2160, tile bands",
    "c4": "synthetic 1M Gaussians, SH3, 256 orbit cameras at 1920x1080",
    "c5": "synthetic 6M anisotropic low-opacity Gaussians, SH3, 1920x1080",
}


def config_scene(name: str, scale: float = 1.0):
    """(scene dict, [cameras]) for a BASELINE config; ``scale`` shrinks P for quick runs."""
    if name == "c1":
        s = make_scene(0, max(1, int(10_000 * scale)))
        for k in ("means", "scales", "rotations", "opacities", "colors"):
            s[k] = np.ascontiguousarray(s[k])
        return s, [make_camera(256, 256)]
    if name == "c2":
        return gen_uniform(int(1_000_000 * scale), 1920, 1080, seed=2), [make_camera(1920, 1080)]
    if name == "c3":
        return gen_uniform(int(3_000_000 * scale), 3840, 2160, seed=3), [make_camera(3840, 2160)]
    if name == "c4":
        return gen_ball(int(1_000_000 * scale), seed=4), orbit_cameras(256)
    if name == "c5":
        return gen_uniform(int(6_000_000 * scale), 1920, 1080, seed=5, anisotropic=True), [make_camera(1920, 1080)]
    raise ValueError(f"unknown config {name!r}")
