import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")
GOLDEN_NAMES = sorted(f[:-4] for f in os.listdir(GOLDEN_DIR) if f.endswith(".npz"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libtcgs.so")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_golden(name):
    with np.load(os.path.join(GOLDEN_DIR, f"{name}.npz")) as z:
        g = {k: z[k] for k in z.files}
    for k in ("rgb", "T"):  # large frames store the image as 16-bit fixed point (make_golden.py)
        if k + "_q16" in g:
            g[k] = g.pop(k + "_q16").astype(np.float64) / 65535.0
    return g


class GoldenCam:
    def __init__(self, g):
        self.view = g["view"]
        self.fx, self.fy, self.cx, self.cy, self.near = (float(x) for x in g["intr"])
        self.width, self.height = (int(x) for x in g["size"])


@pytest.fixture(params=GOLDEN_NAMES)
def golden(request):
    g = load_golden(request.param)
    g["name"] = request.param
    return g
