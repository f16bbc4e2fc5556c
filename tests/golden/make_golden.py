"""Generate golden vectors by running the REFERENCE renderer (tilesplat).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py c1 rot      # a subset

Each fixture ``<name>.npz`` holds the scene inputs (float64), the camera, the
reference's projection records for the survivors (``project_scene``,
src/tilesplat/projection.py:119), its per-tile lists mapped to original
Gaussian ids (``build_tiles``, src/tilesplat/tiling.py:46), the rendered
image and FragmentStats (``render``, src/tilesplat/raster.py:161), plus the
final transmittance T and per-pixel contributor counts, which ``render`` does
not return: they come from re-driving the reference's own ``blend_tile``
tile by tile with a counting evaluator wrapper and a culled sentinel splat
(SURVEY.md section 8(c)).

The fixtures are the pin for the oracle (tests/test_oracle_golden.py) and a
direct parity target for the GPU path (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import tilesplat  # noqa: E402
from tilesplat.projection import project_scene  # noqa: E402
from tilesplat.raster import FragmentStats, ReferenceBackend, blend_tile, render  # noqa: E402
from tilesplat.scene import Camera, Gaussian3D, Scene  # noqa: E402
from tilesplat.tiling import TILE_SIZE, build_tiles  # noqa: E402

import conftest as ref_conftest  # noqa: E402  (reference fixtures: make_scene/make_camera)

from oracle import sh_color  # noqa: E402  (SH restatement: parity unpinned, colours fed to the reference)
from paper_2505_24796_b200 import synthetic  # noqa: E402


class CountingEvaluator:
    """Wraps a reference evaluator; a pixel blends j iff active_j & ~culled_j & active_{j+1}."""

    def __init__(self, inner, n):
        self.inner = inner
        self.n = n
        self.count = np.zeros(256, np.int32)
        self.prev_cand = np.zeros(256, bool)
        self.sentinel_seen = False

    def fragment(self, j, active):
        self.count -= (self.prev_cand & ~active).astype(np.int32)  # terminated at j-1: not a blend
        if j == self.n:
            self.sentinel_seen = True
            self.prev_cand = np.zeros(256, bool)
            return np.ones(256, bool), np.zeros(256), 0
        culled, alpha, n_exp = self.inner.fragment(j, active)
        cand = active & ~culled
        self.count += cand.astype(np.int32)
        self.prev_cand = cand
        return culled, alpha, n_exp

    def finish(self):
        if not self.sentinel_seen:  # blend_tile broke early: every candidate terminated
            self.count -= self.prev_cand.astype(np.int32)


def reference_T_and_counts(projected, grid, cam):
    """Mirror of src/tilesplat/raster.py:177-193 that keeps T and per-pixel counts."""
    backend = ReferenceBackend()
    T = np.ones((cam.height, cam.width))
    counts = np.zeros((cam.height, cam.width), np.int32)
    rgb = np.zeros((cam.height, cam.width, 3))
    for ty in range(grid.tiles_y):
        ys = ty * TILE_SIZE + np.arange(TILE_SIZE)
        for tx in range(grid.tiles_x):
            idx = grid.tile_list(tx, ty)
            if not idx:
                continue
            xs = tx * TILE_SIZE + np.arange(TILE_SIZE)
            in_image = (np.tile(xs, TILE_SIZE) < cam.width) & (np.repeat(ys, TILE_SIZE) < cam.height)
            splats = [projected[j] for j in idx]
            colors = np.array([pg.color for pg in splats])
            ev = CountingEvaluator(backend.tile_evaluator(tx, ty, splats), len(splats))
            scratch = FragmentStats()
            big_c, big_t = blend_tile(ev, len(splats) + 1, in_image, np.vstack([colors, np.zeros((1, 3))]), scratch)
            ev.finish()
            h = min(TILE_SIZE, cam.height - ty * TILE_SIZE)
            w = min(TILE_SIZE, cam.width - tx * TILE_SIZE)
            sl = (slice(ty * TILE_SIZE, ty * TILE_SIZE + h), slice(tx * TILE_SIZE, tx * TILE_SIZE + w))
            T[sl] = big_t.reshape(TILE_SIZE, TILE_SIZE)[:h, :w]
            counts[sl] = ev.count.reshape(TILE_SIZE, TILE_SIZE)[:h, :w]
            rgb[sl] = big_c.reshape(TILE_SIZE, TILE_SIZE, 3)[:h, :w]
    return rgb, T, counts


def scene_from_arrays(d):
    gs = tuple(
        Gaussian3D(mean=d["means"][i].astype(np.float64), scale=d["scales"][i].astype(np.float64),
                   rotation=d["rotations"][i].astype(np.float64), opacity=float(d["opacities"][i]),
                   color=d["colors"][i].astype(np.float64))
        for i in range(d["means"].shape[0]))
    return Scene(gs)


def arrays_from_scene(scene):
    g = scene.gaussians
    return {
        "means": np.array([x.mean for x in g]).reshape(-1, 3),
        "scales": np.array([x.scale for x in g]).reshape(-1, 3),
        "rotations": np.array([x.rotation for x in g]).reshape(-1, 4),
        "opacities": np.array([x.opacity for x in g], dtype=np.float64),
        "colors": np.array([x.color for x in g]).reshape(-1, 3),
    }


def rot_view(ax, ay, az, t):
    cx, sx, cy, sy, cz, sz = np.cos(ax), np.sin(ax), np.cos(ay), np.sin(ay), np.cos(az), np.sin(az)
    Rx = np.array([[1, 0, 0], [0, cx, -sx], [0, sx, cx]])
    Ry = np.array([[cy, 0, sy], [0, 1, 0], [-sy, 0, cy]])
    Rz = np.array([[cz, -sz, 0], [sz, cz, 0], [0, 0, 1]])
    v = np.eye(4)
    v[:3, :3] = Rz @ Ry @ Rx
    v[:3, 3] = t
    return v


def fixture_specs():
    mc, ms = ref_conftest.make_camera, ref_conftest.make_scene
    specs = {
        # config 1 of BASELINE.json
        "c1": lambda: (ms(0, 10000), mc(256, 256)),
        # acceptance criterion 1 scenes (tests/test_acceptance.py:35-41)
        "acc101": lambda: (ms(101, 10), mc(256, 256)),
        "acc102": lambda: (ms(102, 100), mc(256, 256)),
        "acc103": lambda: (ms(103, 400, scale_range=(0.08, 0.2)), mc(512, 512)),
        "acc104": lambda: (ms(104, 700, scale_range=(0.05, 0.15)), mc(768, 768)),
        "acc105": lambda: (ms(105, 1000, scale_range=(0.03, 0.1)), mc(1024, 1024)),
        # criterion 7 scenes (tests/test_acceptance.py:299-306)
        "sem701": lambda: (ms(701, 20, opacity_range=(0.2, 0.95)), mc(64, 64)),
        "sem702": lambda: (ms(702, 60, opacity_range=(0.2, 0.95)), mc(64, 64)),
        "sem703": lambda: (ms(703, 100, opacity_range=(0.2, 0.95)), mc(64, 64)),
        # partial boundary tiles (tests/test_raster.py:149-162)
        "partial": lambda: (ms(9, 15), mc(40, 24)),
        # dense scene, criterion 9 (tests/test_acceptance.py:289-299)
        "dense909": lambda: (ms(909, 150, xy_spread=0.5, scale_range=(0.3, 0.8), opacity_range=(0.7, 0.95)),
                             mc(256, 256)),
        # fp16 stress scene from SURVEY.md Appendix C: small anisotropic low-opacity splats (eigen clamp active)
        "stress": lambda: (ms(5, 8000, xy_spread=1.0, scale_range=(0.002, 0.06), opacity_range=(0.02, 0.4)), mc(160, 160)),
        # near-plane / off-screen / huge Gaussians, wide depth range (tests/test_projection.py:126-135 style)
        "wide": lambda: (ms(21, 400, scale_range=(0.01, 2.0), depth_range=(0.1, 30.0)), mc(200, 136)),
    }

    def rot():  # general (non-identity) view: exercises gemv/gemm operation order and float64 depth ties
        scene = ms(31, 3000, xy_spread=2.5, depth_range=(-2.0, 2.0))
        cam = Camera(view=rot_view(0.3, -0.4, 0.2, [0.1, -0.2, 7.0]), fx=140.0, fy=150.0, cx=70.5, cy=47.25,
                     width=144, height=96)
        return scene, cam

    def dense_rot():  # many splats per tile, fp32 depth keys would mis-order
        scene = ms(77, 10000, xy_spread=0.8, depth_range=(3.0, 5.0), scale_range=(0.02, 0.08))
        cam = Camera(view=rot_view(0.05, 0.1, -0.3, [0.0, 0.0, 1.0]), fx=60.0, fy=60.0, cx=32.0, cy=32.0,
                     width=64, height=64)
        return scene, cam

    def sh3():  # SH degree 3: colours from the oracle's SH restatement (unpinned) fed to the reference
        d = synthetic.gen_uniform(3000, 128, 96, seed=12, sh_degree=3)
        view = rot_view(0.02, -0.03, 0.01, [0.05, 0.0, 0.3])
        d = {k: (v.astype(np.float64) if isinstance(v, np.ndarray) else v) for k, v in d.items()}
        d["colors"] = sh_color(d["means"], d["features"], 3, view)
        cam = Camera(view=view, fx=1.2 * 128, fy=1.2 * 128, cx=64.0, cy=48.0, width=128, height=96)
        return d, cam

    def f32gen():  # float32-valued generator G at small scale (the BASELINE config-2 family)
        d = synthetic.gen_uniform(8000, 240, 136, seed=2, sh_degree=0)
        cam = ref_conftest.make_camera(240, 136)
        return d, cam

    def aniso():  # float32-valued generator G' (config-5 family): clamp-heavy, elongated, low opacity
        d = synthetic.gen_uniform(12000, 160, 96, seed=5, sh_degree=0, anisotropic=True)
        cam = ref_conftest.make_camera(160, 96)
        return d, cam

    specs["rot"] = rot
    specs["dense_rot"] = dense_rot
    specs["sh3"] = sh3
    specs["f32gen"] = f32gen
    specs["aniso"] = aniso
    return specs


def make_fixture(name, builder):
    t0 = time.time()
    obj, cam = builder()
    extra = {}
    if isinstance(obj, dict):
        arrays = {k: obj[k] for k in ("means", "scales", "rotations", "opacities", "colors")}
        if "features" in obj:
            extra["features"] = obj["features"]
            extra["sh_degree"] = np.int32(obj["sh_degree"])
        scene = scene_from_arrays(arrays)
    else:
        scene = obj
        arrays = arrays_from_scene(scene)
    img, stats = render(scene, cam, "reference")
    projected, dropped = project_scene(scene.gaussians, cam)
    # survivors keep input order; recover their original indices
    surv = []
    pi = 0
    for i, g in enumerate(scene.gaussians):
        if pi < len(projected) and tilesplat.project(g, cam) is not None:
            surv.append(i)
            pi += 1
    surv = np.array(surv, np.int32)
    assert surv.size == len(projected)
    grid = build_tiles(projected, cam)
    offsets = np.zeros(len(grid.lists) + 1, np.int64)
    offsets[1:] = np.cumsum([len(lst) for lst in grid.lists])
    ids = np.array([surv[j] for lst in grid.lists for j in lst], np.int32)
    rgb2, T, counts = reference_T_and_counts(projected, grid, cam)
    assert np.array_equal(rgb2, img.rgb), name
    assert int(counts.sum()) == stats.f_blend, name
    out = dict(
        means=arrays["means"], scales=arrays["scales"], rotations=arrays["rotations"],
        opacities=arrays["opacities"], colors=arrays["colors"],
        view=np.asarray(cam.view, np.float64), intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.near]),
        size=np.array([cam.width, cam.height], np.int32),
        surv=surv,
        mean2d=np.array([pg.mean2d for pg in projected]).reshape(-1, 2),
        inv_cov=np.array([pg.inv_cov for pg in projected], np.float64).reshape(-1, 3),
        depth=np.array([pg.depth for pg in projected], np.float64),
        radius=np.array([pg.radius for pg in projected], np.int32),
        offsets=offsets, ids=ids, rgb=img.rgb, T=T, counts=counts,
        stats=np.array([stats.f_blend, stats.f_cull, stats.f_skip, stats.exp_calls, stats.n_splats, stats.dropped,
                        stats.pixels_terminated], np.int64),
        **extra,
    )
    if cam.width * cam.height > 256 * 256:
        # large frames (criterion-1 scenes 103-105): the float64 mantissa noise does not compress (25 MB for
        # 1024^2), so the image and T are stored as 16-bit fixed point (tests/conftest.py:load_golden decodes
        # them) and tests hold the oracle to them within img_tol (half a quantum; the reference's own criterion-1
        # bound is 1e-5, tests/test_acceptance.py:56)
        for k in ("rgb", "T"):
            out[k + "_q16"] = np.round(np.clip(out.pop(k), 0.0, 1.0) * 65535.0).astype(np.uint16)
        out["img_tol"] = np.float64(0.5 / 65535.0 + 1e-12)
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **out)
    print(f"{name}: P={arrays['means'].shape[0]} N={stats.n_splats} {cam.width}x{cam.height} "
          f"stats={stats.counts()} terminated={stats.pixels_terminated} -> {os.path.getsize(path)/1e6:.2f} MB "
          f"({time.time()-t0:.1f}s)", flush=True)


def main(argv):
    specs = fixture_specs()
    names = argv or list(specs)
    for n in names:
        make_fixture(n, specs[n])


if __name__ == "__main__":
    main(sys.argv[1:])
