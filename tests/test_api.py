"""Host-side mirror of the reference render API (src/tilesplat/raster.py), on CPU: backend factory,
FragmentStats, computation_model, camera packing and argument validation (no GPU needed)."""

import numpy as np
import pytest

import paper_2505_24796_b200 as tcgs
from paper_2505_24796_b200 import _abi, synthetic
from paper_2505_24796_b200.raster import FragmentStats, camera_struct, computation_model, make_backend


def test_constants_match_reference():  # src/tilesplat/raster.py:15-16, tiling.py:11
    assert tcgs.ALPHA_CULL_THRESHOLD == 1.0 / 255.0
    assert tcgs.TERMINATION_THRESHOLD == 0.0001
    assert tcgs.TILE_SIZE == 16


@pytest.mark.parametrize("spec,mode,early,name", [
    ("tcgs", _abi.ALPHA_TC_HILO, True, "tcgs"), ("tcgs-fp16", _abi.ALPHA_TC_K8, True, "tcgs-fp16"),
    ("tcgs-ffma", _abi.ALPHA_FFMA, True, "tcgs-ffma"),
    # the reference's spellings keep its default coords="global" (src/tilesplat/raster.py:149)
    ("frag2mat", _abi.ALPHA_FFMA, True, "frag2mat-exact-global"),
    ("frag2mat-fp16", _abi.ALPHA_TC_K8_GLOBAL, True, "frag2mat-fp16-global"),
    ("reference", _abi.ALPHA_FFMA, False, "reference")])
def test_backend_specs(spec, mode, early, name):
    b = make_backend(spec)
    assert (b.name, b.alpha_mode, b.early_cull) == (name, mode, early)
    # EarlyCull off is a different kernel (alpha for every active fragment), not only a different count;
    # the reference backend has no EarlyCull at all
    assert make_backend(spec, use_early_cull=False).early_cull is False


def test_reference_spellings_and_coordinates():
    # G2L for the paper's fp16 vector; exact arithmetic ignores coords (criterion 1: global == local to 1e-5)
    assert make_backend("frag2mat-fp16", coords="local").alpha_mode == _abi.ALPHA_TC_K8
    assert make_backend("frag2mat", coords="local").alpha_mode == _abi.ALPHA_FFMA
    assert make_backend("reference", coords="global").alpha_mode == _abi.ALPHA_FFMA
    assert make_backend("reference", coords="local", use_early_cull=True).early_cull is False
    assert make_backend("frag2mat-fp16", coords="global").coords == "global"


def test_backend_errors():  # reference tests/test_raster.py:165-167 ("splatzilla"), tensor_path.py:175-181
    with pytest.raises(ValueError):
        make_backend("splatzilla")
    with pytest.raises(ValueError):
        make_backend("frag2mat", coords="polar")
    with pytest.raises(ValueError):
        make_backend("frag2mat", batch_width=0)
    with pytest.raises(ValueError):  # tf32 arithmetic is not reproduced: refused, not approximated
        make_backend("frag2mat-tf32")
    with pytest.raises(ValueError):  # this package's own specs are tile-local only
        make_backend("tcgs", coords="global")
    with pytest.raises(NotImplementedError):
        make_backend("tcgs").tile_evaluator(0, 0, [])


def test_render_defaults_to_the_reference_backend():
    import inspect

    assert inspect.signature(tcgs.render).parameters["backend"].default == "reference"


def test_fragment_stats_contract():  # src/tilesplat/raster.py:19-49
    st = FragmentStats(f_blend=2, f_cull=3, f_skip=5, exp_calls=7, n_splats=11, dropped=1, pixels_terminated=4,
                       stage_ms={"preprocess": 1.0})
    assert st.total_fragments == 10 and st.counts() == (2, 3, 5, 7)
    assert st.to_dict() == {"f_blend": 2, "f_cull": 3, "f_skip": 5, "exp_calls": 7, "N": 11, "dropped": 1,
                            "pixels_terminated": 4, "stage_ms": {"preprocess": 1.0}}


def test_computation_model():  # reference tests/test_raster.py:93-103
    assert computation_model(FragmentStats(), 1.0, 1.0, 1.0) == 0.0
    assert computation_model(FragmentStats(f_blend=1, f_cull=2), 1.0, 1.0, 1.0) == 1.0 + 2.0 * 3
    with pytest.raises(ValueError):
        computation_model(FragmentStats(), -1.0, 1.0, 1.0)


def test_camera_packing_and_validation():
    cam = synthetic.make_camera(640, 360)
    c = camera_struct(cam)
    assert (c.width, c.height, c.fx, c.cx, c.near_plane) == (640, 360, 768.0, 320.0, 0.2)
    assert list(c.view) == list(np.eye(4).reshape(-1))
    for bad in (synthetic.make_camera(0, 10), synthetic.CameraSpec(np.eye(4), -1.0, 1.0, 0, 0, 8, 8),
                synthetic.CameraSpec(np.eye(4), 1.0, 1.0, 0, 0, 8, 8, near=0.0)):
        with pytest.raises(ValueError):
            camera_struct(bad)


def test_renderer_requires_cuda_device():
    with pytest.raises(ValueError):
        tcgs.Renderer("cpu")
