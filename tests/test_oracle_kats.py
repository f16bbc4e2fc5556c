"""The reference's own known-answer tests, replayed against the CPU oracle.

Each test cites the reference test it mirrors.  Together with
test_oracle_golden.py this pins the oracle before it is trusted as the GPU
path's checker.
"""

import math
import os

import numpy as np
import pytest

import oracle
from paper_2505_24796_b200 import synthetic


class Cam:
    def __init__(self, width=64, height=64, view=None, fx=1.0, fy=1.0, cx=0.0, cy=0.0, near=0.2):
        self.view = np.eye(4) if view is None else view
        self.fx, self.fy, self.cx, self.cy, self.near = fx, fy, cx, cy, near
        self.width, self.height = width, height


def proj_from(mean2d, radius, depth=None):
    """Hand-built projection records (tests/test_tiling.py:9-17 `splat`)."""
    n = len(mean2d)
    return oracle.Projection(np.ones(n, bool), np.asarray(mean2d, np.float64).reshape(n, 2),
                             np.tile([1.0, 0.0, 1.0], (n, 1)),
                             np.asarray(depth if depth is not None else np.ones(n), np.float64),
                             np.asarray(radius, np.int32), 0)


def lists(offsets, ids, tiles_x, tx, ty):
    t = ty * tiles_x + tx
    return tuple(int(i) for i in ids[offsets[t]:offsets[t + 1]])


# ---- tests/test_tiling.py ---------------------------------------------------

def test_single_tile_coverage():  # tests/test_tiling.py:20-25
    cam = synthetic.make_camera(64, 64)
    off, ids = oracle.build_tiles(proj_from([(8.0, 8.0)], [1]), cam)
    assert ids.size == 1 and lists(off, ids, 4, 0, 0) == (0,)


def test_corner_covers_four_tiles():  # tests/test_tiling.py:28-34
    cam = synthetic.make_camera(64, 64)
    off, ids = oracle.build_tiles(proj_from([(16.0, 16.0)], [1]), cam)
    assert ids.size == 4
    for tx, ty in ((0, 0), (1, 0), (0, 1), (1, 1)):
        assert lists(off, ids, 4, tx, ty) == (0,)


def test_coverage_clipped_to_grid():  # tests/test_tiling.py:36-39
    cam = synthetic.make_camera(32, 32)
    off, ids = oracle.build_tiles(proj_from([(0.0, 0.0)], [40]), cam)
    assert ids.size == 4


def test_covered_tiles_matches_interval_overlap():  # tests/test_tiling.py:42-56
    rng = np.random.default_rng(5)
    cam = synthetic.make_camera(128, 128)
    for _ in range(200):
        mean = rng.uniform(-20.0, 148.0, 2)
        radius = int(rng.integers(0, 40))
        off, ids = oracle.build_tiles(proj_from([mean], [radius]), cam)
        got = {(t % 8, t // 8) for t in range(64) if off[t + 1] > off[t]}
        expect = set()
        for ty in range(8):
            for tx in range(8):
                xo = mean[0] + radius >= tx * 16 and mean[0] - radius < (tx + 1) * 16
                yo = mean[1] + radius >= ty * 16 and mean[1] - radius < (ty + 1) * 16
                if xo and yo:
                    expect.add((tx, ty))
        assert got == expect


def test_depth_order_is_ascending_and_stable():  # tests/test_tiling.py:59-69
    cam = synthetic.make_camera(16, 16)
    pr = proj_from([(8.0, 8.0), (8.0, 8.0), (7.0, 8.0), (8.0, 8.0)], [1, 1, 1, 1], [5.0, 2.0, 5.0, 1.0])
    off, ids = oracle.build_tiles(pr, cam)
    assert lists(off, ids, 1, 0, 0) == (3, 1, 0, 2)


def test_census_empty_grid():  # tests/test_tiling.py:72-77
    cam = synthetic.make_camera(32, 32)
    off, ids = oracle.build_tiles(proj_from(np.zeros((0, 2)), []), cam)
    assert ids.size == 0 and off[-1] == 0


# ---- tests/test_raster.py blend goldens (ConstantAlphaEvaluator) ----------

def test_blend_two_half_alpha_splats():  # tests/test_raster.py:37-45
    c, t, cnt, (fb, fc, fs, pt) = oracle.blend_const_alpha([0.5, 0.5], [[1, 0, 0], [0, 1, 0]])
    assert np.allclose(c, [0.5, 0.25, 0.0]) and np.allclose(t, 0.25)
    assert fb == 512 and fc == 0 and fs == 0 and np.all(cnt == 2)


def test_blend_culls_tiny_alpha():  # tests/test_raster.py:48-55
    c, t, cnt, (fb, fc, fs, pt) = oracle.blend_const_alpha([1.0 / 512.0], [[1, 1, 1]])
    assert np.all(c == 0.0) and np.all(t == 1.0) and fc == 256 and fb == 0


def test_opaque_splat_terminates_before_compositing():  # tests/test_raster.py:58-69
    c, t, cnt, (fb, fc, fs, pt) = oracle.blend_const_alpha([1.0, 0.5], np.ones((2, 3)))
    assert np.all(c == 0.0) and np.all(t == 1.0)
    assert pt == 256 and fb == 0 and fs == 512


def test_blend_skips_after_termination_accounting():  # tests/test_raster.py:72-80
    c, t, cnt, (fb, fc, fs, pt) = oracle.blend_const_alpha([0.5, 1.0, 0.5], np.ones((3, 3)))
    assert fb == 256 and pt == 256 and fs == 512 and fb + fc + fs == 3 * 256


def test_empty_scene_renders_black():  # tests/test_raster.py:83-89
    cam = synthetic.make_camera(48, 48)
    fr = oracle.render(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 4)), np.zeros(0), np.zeros((0, 3)), cam)
    assert fr.rgb.shape == (48, 48, 3) and np.all(fr.rgb == 0.0)
    assert fr.stats.counts() == (0, 0, 0, 0) and fr.stats.n_splats == 0


def test_stats_closure_against_tile_lists():  # tests/test_raster.py:138-162
    for (w, h, seed, n) in ((80, 80, 17, 30), (40, 24, 9, 15)):
        cam = synthetic.make_camera(w, h)
        s = synthetic.make_scene(seed, n)
        fr = oracle.render(s["means"], s["scales"], s["rotations"], s["opacities"], s["colors"], cam)
        expected = 0
        tx_n = (w + 15) // 16
        for t in range(fr.offsets.size - 1):
            tx, ty = t % tx_n, t // tx_n
            expected += int(fr.offsets[t + 1] - fr.offsets[t]) * min(16, w - 16 * tx) * min(16, h - 16 * ty)
        st = fr.stats
        assert st.f_blend + st.f_cull + st.f_skip == expected


def test_brightest_pixel_at_projected_mean():  # tests/test_raster.py:106-120
    cam = synthetic.make_camera(64, 64)
    fr = oracle.render([[0.05, -0.08, 5.0]], [[0.2, 0.2, 0.2]], [[1.0, 0.0, 0.0, 0.0]], [0.9], [[1.0, 1.0, 1.0]],
                       cam)
    lum = fr.rgb.sum(axis=2)
    y, x = np.unravel_index(np.argmax(lum), lum.shape)
    assert x == round(fr.proj.mean2d[0, 0]) and y == round(fr.proj.mean2d[0, 1])


# ---- tests/test_projection.py ----------------------------------------------

def test_project_unit_gaussian_on_axis():  # tests/test_projection.py:54-65
    pr = oracle.project([[0.0, 0.0, 1.0]], [[1.0, 1.0, 1.0]], [[1.0, 0, 0, 0]], Cam())
    assert pr.visible[0]
    assert np.allclose(pr.mean2d[0], [0.0, 0.0])
    assert pr.inv_cov[0, 0] == pytest.approx(1.0 / 1.3) and pr.inv_cov[0, 2] == pytest.approx(1.0 / 1.3)
    assert pr.inv_cov[0, 1] == pytest.approx(0.0, abs=1e-15)
    assert pr.depth[0] == 1.0 and pr.radius[0] == math.ceil(3.0 * math.sqrt(1.3))


def test_project_isotropic_radius():  # tests/test_projection.py:68-73
    pr = oracle.project([[0.0, 0.0, 1.0]], [[0.5, 0.5, 0.5]], [[1.0, 0, 0, 0]], Cam())
    var = 0.25 + 0.3
    assert pr.inv_cov[0, 0] == pytest.approx(1.0 / var) and pr.radius[0] == math.ceil(3.0 * math.sqrt(var))


def test_project_frustum_cull():  # tests/test_projection.py:76-80 (equality culls)
    pr = oracle.project([[0, 0, 0.1], [0, 0, -2.0], [0, 0, 0.2], [0, 0, 2.0]], np.ones((4, 3)),
                        np.tile([1.0, 0, 0, 0], (4, 1)), Cam())
    assert list(pr.visible) == [False, False, False, True] and pr.dropped == 3


def test_project_pixel_center_offset():  # tests/test_projection.py:91-97
    cam = Cam(64, 48, fx=100.0, fy=100.0, cx=32.0, cy=24.0)
    pr = oracle.project([[0.5, -0.25, 2.0]], np.ones((1, 3)), [[1.0, 0, 0, 0]], cam)
    assert pr.mean2d[0, 0] == pytest.approx(32.0 + 100.0 * 0.5 / 2.0)
    assert pr.mean2d[0, 1] == pytest.approx(24.0 - 100.0 * 0.25 / 2.0)


def test_projected_inverse_covariance_stays_in_range():  # tests/test_projection.py:126-135
    cam = synthetic.make_camera(256, 256)
    s = synthetic.make_scene(21, 150, scale_range=(0.01, 2.0), depth_range=(0.5, 30.0))
    pr = oracle.project(s["means"], s["scales"], s["rotations"], cam)
    inv = pr.inv_cov[pr.visible]
    tr = inv[:, 0] + inv[:, 2]
    assert np.all(tr > 0) and np.all(tr <= 4.0 + 1e-12)


def test_py_hypot_matches_math_hypot():
    rng = np.random.default_rng(0)
    for scale in (1.0, 1e-3, 1e3, 1e-300, 1e300):
        a = rng.normal(size=2000) * scale
        b = rng.normal(size=2000) * scale * rng.choice([1, 1e-6, 1e6, 0.0], size=2000)
        for x, y in zip(a, b):
            assert oracle.py_hypot(x, y) == math.hypot(x, y)


# ---- the reference fixtures' generators ------------------------------------

@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/tests"), reason="reference tree absent")
def test_make_scene_matches_reference_conftest():
    import importlib.util
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    spec = importlib.util.spec_from_file_location("ref_conftest", "/root/reference/pkg/tests/conftest.py")
    ref = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(ref)
    s = synthetic.make_scene(3, 50, scale_range=(0.1, 0.2))
    r = ref.make_scene(3, 50, scale_range=(0.1, 0.2))
    assert np.array_equal(s["means"], np.array([g.mean for g in r.gaussians]))
    assert np.array_equal(s["rotations"], np.array([g.rotation for g in r.gaussians]))
    assert np.array_equal(s["colors"], np.array([g.color for g in r.gaussians]))


def test_make_scene_matches_golden_c1_inputs():
    from conftest import load_golden
    g = load_golden("c1")
    s = synthetic.make_scene(0, 10000)
    for k in ("means", "scales", "rotations", "opacities", "colors"):
        assert np.array_equal(s[k], g[k]), k
