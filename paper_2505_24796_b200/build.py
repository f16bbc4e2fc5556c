"""Build libtcgs.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB_DIR = os.path.join(HERE, "_lib")
LIB_PATH = os.path.join(LIB_DIR, "libtcgs.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

SOURCES = ["abi.cu", "preprocess.cu", "binning.cu", "render.cu", "render.cu:few", "render.cu:heavy"]
# render.cu is compiled three times: the default K7 (4 CTAs/SM x 2 producer warps), the few-tiles K7 (3 x 4) and the
# heavy K7 (the default residency reading the compacted live lists of producer-heavy frames)
VARIANT_FLAGS = {"few": ["-DTCGS_K7_ENTRY=launch_render_k7_few", "-DTCGS_K7_CTAS=3", "-DTCGS_K7_PRODUCERS=4",
                         "-DTCGS_K7_SECOND_BUILD"],
                 "heavy": ["-DTCGS_K7_ENTRY=launch_render_k7_heavy", "-DTCGS_K7_COMPACT", "-DTCGS_K7_SECOND_BUILD"]}
# preprocess.cu must not contract a*b+c into FMA: it reproduces numpy's float64 operation order.
PER_FILE_FLAGS = {"preprocess.cu": ["--fmad=false"]}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fno-fast-math",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "tcgs.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile libtcgs.so (``out``/``defines``: an experiment variant, e.g. -DTCGS_K7_WAIT_HINT=0)."""
    if out is None and not force and not _stale():
        return LIB_PATH
    lib_path = out or LIB_PATH
    obj_dir = os.path.join(os.path.dirname(lib_path), "obj" if out is None else "obj_" + os.path.basename(lib_path))
    os.makedirs(obj_dir, exist_ok=True)
    objs = []
    for entry in SOURCES:
        src, _, variant = entry.partition(":")
        obj = os.path.join(obj_dir, src.replace(".cu", f"_{variant}.o" if variant else ".o"))
        cmd = [NVCC, *ARCH, *COMMON, *defines, *PER_FILE_FLAGS.get(src, []), *VARIANT_FLAGS.get(variant, []), "-c",
               os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(obj)
    tmp = lib_path + f".tmp{os.getpid()}"
    subprocess.run([NVCC, *ARCH, "-shared", "-cudart", "static", *objs, "-o", tmp], check=True)
    os.replace(tmp, lib_path)
    return lib_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
