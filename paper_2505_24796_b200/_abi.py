"""ctypes binding of libtcgs.so (include/tcgs.h).  The product path has no fallback:
if the library cannot be loaded every render raises."""

from __future__ import annotations

import ctypes
import os
import shutil

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TCGS_LIB") or os.path.join(HERE, "_lib", "libtcgs.so")  # TCGS_LIB: A/B builds

TCGS_OK = 0
TCGS_ERR_INVALID_ARG = -1
TCGS_ERR_CUDA = -2
TCGS_ERR_CAPACITY = -3
TCGS_ERR_DEVICE = -4
TCGS_ERR_WORKSPACE = -5

ALPHA_TC_HILO = 0
ALPHA_TC_K8 = 1
ALPHA_FFMA = 2
ALPHA_TC_K8_GLOBAL = 3

IPC_HANDLE_BYTES = 64

F32 = 0
F64 = 1


class Scene(ctypes.Structure):
    _fields_ = [("P", ctypes.c_int64), ("sh_degree", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("means", ctypes.c_void_p), ("scales", ctypes.c_void_p), ("rotations", ctypes.c_void_p),
                ("opacities", ctypes.c_void_p), ("features", ctypes.c_void_p)]


class Camera(ctypes.Structure):
    _fields_ = [("view", ctypes.c_double * 16), ("fx", ctypes.c_double), ("fy", ctypes.c_double),
                ("cx", ctypes.c_double), ("cy", ctypes.c_double), ("near_plane", ctypes.c_double),
                ("width", ctypes.c_int32), ("height", ctypes.c_int32)]


class Opts(ctypes.Structure):
    _fields_ = [("tile_row_begin", ctypes.c_int32), ("tile_row_end", ctypes.c_int32),
                ("alpha_mode", ctypes.c_int32), ("early_cull", ctypes.c_int32), ("debug", ctypes.c_int32),
                ("coverage", ctypes.c_int32), ("defer_colour", ctypes.c_int32), ("schedule", ctypes.c_int32),
                ("timing", ctypes.c_int32), ("reserved", ctypes.c_int32), ("dump_beta", ctypes.c_void_p),
                ("dump_class", ctypes.c_void_p)]


SCHEDULE = {"dynamic": 0, "static": 1}  # enum tcgs_schedule (include/tcgs.h)


COVERAGE = {"square": 0, "box": 1, "ellipse": 2}  # enum tcgs_coverage (include/tcgs.h)


class Stats(ctypes.Structure):
    _fields_ = [("n_splats", ctypes.c_int64), ("dropped", ctypes.c_int64), ("f_blend", ctypes.c_int64),
                ("f_cull", ctypes.c_int64), ("f_skip", ctypes.c_int64), ("exp_calls", ctypes.c_int64),
                ("pixels_terminated", ctypes.c_int64), ("n_visible", ctypes.c_int64),
                ("max_splats_needed", ctypes.c_int64), ("ms_preprocess", ctypes.c_float), ("ms_sort", ctypes.c_float),
                ("ms_blend", ctypes.c_float), ("reserved", ctypes.c_float)]


# name -> (restype, argtypes); every symbol include/tcgs.h declares
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
MAX_VIEWS_PER_PASS = 8  # TCGS_MAX_VIEWS_PER_PASS (include/tcgs.h)

SIGNATURES = {
    "tcgs_workspace_size": (ctypes.c_size_t, [_I64, ctypes.c_int32, ctypes.c_int32, _I64]),
    "tcgs_preprocess": (ctypes.c_int, [ctypes.POINTER(Scene), ctypes.POINTER(Camera), ctypes.POINTER(Opts), _P,
                                       ctypes.c_size_t, _I64, _P]),
    "tcgs_colour": (ctypes.c_int, [ctypes.POINTER(Scene), ctypes.POINTER(Camera), ctypes.POINTER(Opts), _P,
                                   ctypes.c_size_t, _I64, _P]),
    "tcgs_preprocess_views": (ctypes.c_int, [ctypes.POINTER(Scene), ctypes.POINTER(Camera), ctypes.c_int32,
                                             ctypes.POINTER(Opts), ctypes.POINTER(_P), ctypes.c_size_t, _I64, _P]),
    "tcgs_bin": (ctypes.c_int, [_I64, ctypes.POINTER(Camera), ctypes.POINTER(Opts), _P, ctypes.c_size_t, _I64, _P]),
    "tcgs_blend": (ctypes.c_int, [_I64, ctypes.POINTER(Camera), ctypes.POINTER(Opts), _P, ctypes.c_size_t, _I64,
                                  _P, _P, _P, _P]),
    "tcgs_render": (ctypes.c_int, [ctypes.POINTER(Scene), ctypes.POINTER(Camera), ctypes.POINTER(Opts), _P,
                                   ctypes.c_size_t, _I64, _P, _P, _P, _P]),
    "tcgs_read_stats": (ctypes.c_int, [_P, _I64, ctypes.POINTER(Opts), ctypes.POINTER(Stats), _P]),
    "tcgs_counters_bytes": (ctypes.c_size_t, []),
    "tcgs_snapshot_stats": (ctypes.c_int, [_P, _P, _P]),
    "tcgs_decode_stats": (ctypes.c_int, [_P, ctypes.POINTER(Opts), ctypes.POINTER(Stats)]),
    "tcgs_frame_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "tcgs_frame_free": (ctypes.c_int, [_P]),
    "tcgs_ipc_get_handle": (ctypes.c_int, [_P, _P]),
    "tcgs_ipc_open": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_void_p)]),
    "tcgs_ipc_close": (ctypes.c_int, [_P]),
    "tcgs_blend_lists": (ctypes.c_int, [_I64, _P, _P, _P, _P, _P, _P, ctypes.POINTER(Camera), ctypes.POINTER(Opts),
                                        _P, ctypes.c_size_t, _P, _P, _P, _P]),
    "tcgs_copy_lists": (ctypes.c_int, [_P, _I64, ctypes.POINTER(Camera), ctypes.POINTER(Opts), _I64, _P, _P, _P]),
    "tcgs_copy_projection": (ctypes.c_int, [_P, _I64, ctypes.POINTER(Camera), _I64, _P, _P, _P, _P, _P, _P, _P]),
    "tcgs_tile_row_counts": (ctypes.c_int, [_P, _I64, ctypes.POINTER(Camera), _I64, _P, _P]),
    "tcgs_device_check": (ctypes.c_int, []),
    "tcgs_error_string": (ctypes.c_char_p, [ctypes.c_int]),
    "tcgs_last_error": (ctypes.c_char_p, []),
    "tcgs_version": (ctypes.c_int, []),
    "tcgs_launch_count": (ctypes.c_ulonglong, []),
}

_lib = None


def load(build_if_missing: bool = True):
    """Load libtcgs.so (building it in-tree with nvcc if it is absent and nvcc exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH) and build_if_missing and shutil.which(
            os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")):
        from . import build as _build
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libtcgs.so not found at {LIB_PATH}: run `python -m paper_2505_24796_b200.build` "
                           "(the B200 renderer has no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == TCGS_OK:
        return
    lib = load()
    msg = f"{what}: {lib.tcgs_error_string(rc).decode()} ({lib.tcgs_last_error().decode()})"
    if rc in (TCGS_ERR_INVALID_ARG, TCGS_ERR_WORKSPACE):
        raise ValueError(msg)
    if rc == TCGS_ERR_CAPACITY:
        raise CapacityError(msg)
    raise RuntimeError(msg)


class CapacityError(RuntimeError):
    pass
