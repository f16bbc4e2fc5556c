"""The C-ABI boundary on CPU: libtcgs.so loads, exports every function include/tcgs.h declares with
the ctypes signature the Python mirror binds, and its host-only entry points behave.  No compute
calls (there is no GPU here)."""

import ctypes
import os
import re

import pytest

from paper_2505_24796_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tcgs.h")
PKG = os.path.join(ROOT, "paper_2505_24796_b200")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^[A-Za-z_][\w\s\*]*?\b(tcgs_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_abi.LIB_PATH):
        from paper_2505_24796_b200 import build

        build.build()
    return _abi.load(build_if_missing=False)


def test_header_declares_the_render_path():
    names = declared_functions()
    for n in ("tcgs_preprocess", "tcgs_bin", "tcgs_blend", "tcgs_render", "tcgs_read_stats", "tcgs_blend_lists",
              "tcgs_tile_row_counts", "tcgs_workspace_size", "tcgs_error_string", "tcgs_launch_count"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, f"libtcgs.so lacks {missing}"
    assert sorted(_abi.SIGNATURES) == names, "ctypes mirror out of sync with include/tcgs.h"


def test_host_only_entry_points(lib):
    assert lib.tcgs_version() >= 1
    assert lib.tcgs_error_string(0) == b"ok"
    assert b"capacity" in lib.tcgs_error_string(_abi.TCGS_ERR_CAPACITY)
    assert lib.tcgs_error_string(-99) == b"unknown error"
    small = lib.tcgs_workspace_size(1000, 256, 256, 64000)
    big = lib.tcgs_workspace_size(1_000_000, 1920, 1080, 6_500_000)
    assert 0 < small < big
    assert lib.tcgs_workspace_size(0, 16, 16, 1) > 0
    assert isinstance(lib.tcgs_launch_count(), int)


def test_invalid_arguments_are_rejected_before_any_launch(lib):
    cam = _abi.Camera()
    cam.width, cam.height, cam.fx, cam.fy, cam.near_plane = 0, 16, 1.0, 1.0, 0.2
    ws = ctypes.create_string_buffer(16)
    n0 = lib.tcgs_launch_count()
    rc = lib.tcgs_bin(10, ctypes.byref(cam), None, ctypes.cast(ws, ctypes.c_void_p), 16, 100, None)
    assert rc == _abi.TCGS_ERR_INVALID_ARG
    assert b"dimensions" in lib.tcgs_last_error()
    cam.width = 16
    rc = lib.tcgs_bin(10, ctypes.byref(cam), None, ctypes.cast(ws, ctypes.c_void_p), 16, 100, None)
    assert rc == _abi.TCGS_ERR_WORKSPACE  # 16 bytes is far below tcgs_workspace_size
    with pytest.raises(ValueError):
        _abi.check(rc, "tcgs_bin")
    o = _abi.Opts()
    o.coverage = 7
    rc = lib.tcgs_bin(10, ctypes.byref(cam), ctypes.byref(o), ctypes.cast(ws, ctypes.c_void_p), 16, 100, None)
    assert rc == _abi.TCGS_ERR_INVALID_ARG and b"coverage" in lib.tcgs_last_error()
    assert lib.tcgs_launch_count() == n0


def test_preprocess_views_rejects_bad_view_groups(lib):
    scene = _abi.Scene()
    scene.P, scene.sh_degree, scene.dtype = 0, 0, 0
    cams = (_abi.Camera * 2)()
    for c in cams:
        c.width, c.height, c.fx, c.fy, c.near_plane = 64, 64, 50.0, 50.0, 0.2
    need = lib.tcgs_workspace_size(0, 64, 64, 1024)
    bufs = [ctypes.create_string_buffer(need) for _ in range(2)]
    ws = (ctypes.c_void_p * 2)(*[ctypes.cast(b, ctypes.c_void_p).value for b in bufs])
    n0 = lib.tcgs_launch_count()
    for n in (0, _abi.MAX_VIEWS_PER_PASS + 1):
        assert lib.tcgs_preprocess_views(ctypes.byref(scene), cams, n, None, ws, need, 1024, None) == \
            _abi.TCGS_ERR_INVALID_ARG
    same = (ctypes.c_void_p * 2)(ws[0], ws[0])
    assert lib.tcgs_preprocess_views(ctypes.byref(scene), cams, 2, None, same, need, 1024, None) == \
        _abi.TCGS_ERR_INVALID_ARG
    assert b"distinct" in lib.tcgs_last_error()
    cams[1].width = 0
    assert lib.tcgs_preprocess_views(ctypes.byref(scene), cams, 2, None, ws, need, 1024, None) == \
        _abi.TCGS_ERR_INVALID_ARG
    assert lib.tcgs_launch_count() == n0


def test_colour_pass_rejects_bad_arguments(lib):
    cam = _abi.Camera()
    cam.width, cam.height, cam.fx, cam.fy, cam.near_plane = 64, 64, 50.0, 50.0, 0.2
    ws = ctypes.create_string_buffer(16)
    n0 = lib.tcgs_launch_count()
    assert lib.tcgs_colour(None, ctypes.byref(cam), None, ctypes.cast(ws, ctypes.c_void_p), 16, 100, None) == \
        _abi.TCGS_ERR_INVALID_ARG
    scene = _abi.Scene()
    scene.P, scene.sh_degree, scene.dtype = 0, 0, 0
    assert lib.tcgs_colour(ctypes.byref(scene), ctypes.byref(cam), None, ctypes.cast(ws, ctypes.c_void_p), 16, 100,
                           None) == _abi.TCGS_ERR_WORKSPACE
    scene.sh_degree = 7
    assert lib.tcgs_colour(ctypes.byref(scene), ctypes.byref(cam), None, ctypes.cast(ws, ctypes.c_void_p), 16, 100,
                           None) == _abi.TCGS_ERR_INVALID_ARG
    assert lib.tcgs_launch_count() == n0


def test_product_package_never_touches_the_oracle():
    """Only tests/, smoke() and bench.py may use oracle/: the shipped package must not import it."""
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", text, flags=re.M), f
                assert not re.search(r"#include\s*[<\"].*oracle", text), f
                assert not re.search(r"CDLL\(.*oracle|libtcgs_oracle", text), f


def test_c_example_compiles_and_links(lib):
    """examples/render_c.c uses only include/tcgs.h and links libtcgs.so from plain C (gcc, C11)."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None or shutil.which("make") is None:
        pytest.skip("no gcc/make")
    ex = os.path.join(ROOT, "examples")
    r = subprocess.run(["make", "-B", "-C", ex], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    assert "warning" not in r.stderr.lower(), r.stderr
    assert os.access(os.path.join(ex, "render_c"), os.X_OK)
