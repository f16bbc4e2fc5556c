"""PLY ingestion (paper_2505_24796_b200/ply.py): the reference's load_ply semantics
(src/tilesplat/scene.py:141-212, its tests at tests/test_scene.py:49-120) plus SH f_rest bands."""

import os
import struct
import sys

import numpy as np
import pytest

from paper_2505_24796_b200 import ply, synthetic

PROPS = ["x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
         "rot_0", "rot_1", "rot_2", "rot_3"]
REF_SRC = "/root/reference/pkg/src"


def write_rows(path, rows, props=None):
    props = props or PROPS
    header = ["ply", "format binary_little_endian 1.0", f"element vertex {len(rows)}"]
    header += [f"property float {n}" for n in props] + ["end_header"]
    with open(path, "wb") as fh:
        fh.write(("\n".join(header) + "\n").encode("ascii"))
        for row in rows:
            fh.write(struct.pack(f"<{len(row)}f", *row))


def row(**kw):
    base = {n: 0.0 for n in PROPS}
    base["rot_0"] = 1.0
    base.update(kw)
    return [base[n] for n in PROPS]


def test_activations(tmp_path):  # reference tests/test_scene.py:49-59
    p = tmp_path / "one.ply"
    write_rows(p, [row()])
    d = ply.read_ply(str(p))
    assert d["opacities"][0] == pytest.approx(0.5)
    assert np.allclose(d["scales"], 1.0) and np.allclose(d["colors"], 0.5)
    assert np.allclose(d["rotations"], [1.0, 0.0, 0.0, 0.0]) and d["sh_degree"] == 0


def test_dc_colour_and_clamp(tmp_path):  # tests/test_scene.py:62-76
    p = tmp_path / "c.ply"
    write_rows(p, [row(f_dc_0=1.0, f_dc_1=-1.0), row(f_dc_0=10.0, f_dc_1=-10.0)])
    c = ply.read_ply(str(p))["colors"]
    assert c[0, 0] == pytest.approx(0.5 + ply.SH_C0) and c[0, 1] == pytest.approx(0.5 - ply.SH_C0)
    assert c[1, 0] == 1.0 and c[1, 1] == 0.0


def test_quaternion_normalised(tmp_path):  # tests/test_scene.py:79-83
    p = tmp_path / "q.ply"
    write_rows(p, [row(rot_0=3.0, rot_1=4.0)])
    assert np.allclose(ply.read_ply(str(p))["rotations"], [0.6, 0.8, 0.0, 0.0])


@pytest.mark.parametrize("case", ["missing", "zero", "notply", "truncated", "zeroquat"])
def test_errors(tmp_path, case):  # tests/test_scene.py:92-120
    p = tmp_path / "bad.ply"
    if case == "missing":
        props = [n for n in PROPS if n != "opacity"]
        write_rows(p, [[0.0] * len(props)], props)
        with pytest.raises(ply.SceneFormatError, match="opacity"):
            ply.read_ply(str(p))
    elif case == "zero":
        write_rows(p, [])
        with pytest.raises(ply.SceneValidationError):
            ply.read_ply(str(p))
    elif case == "notply":
        p.write_bytes(b"hello world")
        with pytest.raises(ply.SceneFormatError):
            ply.read_ply(str(p))
    elif case == "truncated":
        write_rows(p, [row()])
        p.write_bytes(p.read_bytes()[:-4])
        with pytest.raises(ply.SceneFormatError, match="truncated"):
            ply.read_ply(str(p))
    else:
        write_rows(p, [row(rot_0=0.0)])
        with pytest.raises(ply.SceneValidationError, match="quaternion"):
            ply.read_ply(str(p))
    assert issubclass(ply.SceneFormatError, ValueError) and issubclass(ply.SceneValidationError, ValueError)


@pytest.mark.parametrize("deg", [0, 1, 2, 3])
def test_sh_bands_round_trip(tmp_path, deg):
    """write_ply / read_ply keep every SH band in the 3DGS channel-major f_rest layout."""
    s = synthetic.gen_uniform(500, 128, 96, seed=deg)
    K = (deg + 1) ** 2
    s["sh_degree"] = deg
    s["features"] = np.ascontiguousarray(s["features"][:, :K, :])
    p = tmp_path / f"sh{deg}.ply"
    ply.write_ply(str(p), s)
    d = ply.read_ply(str(p))
    assert d["sh_degree"] == deg and d["features"].shape == (500, K, 3)
    f32 = lambda x: np.asarray(x, np.float32).astype(np.float64)  # noqa: E731 (the file stores float)
    assert np.array_equal(d["features"], f32(s["features"]))
    assert np.array_equal(d["means"], f32(s["means"]))
    assert np.allclose(d["scales"], s["scales"], rtol=1e-6)
    assert np.allclose(d["opacities"], s["opacities"], rtol=1e-5)
    assert np.allclose(d["rotations"], s["rotations"], atol=1e-6)


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present")
def test_matches_reference_load_ply(tmp_path):
    """Same arrays as the reference's own loader on the same file (float64, bit for bit)."""
    sys.path.insert(0, REF_SRC)
    from tilesplat.scene import load_ply as ref_load

    s = synthetic.gen_uniform(300, 128, 96, seed=7)
    s["sh_degree"] = 3
    p = tmp_path / "r.ply"
    ply.write_ply(str(p), s)
    d = ply.read_ply(str(p))
    g = ref_load(str(p)).gaussians
    for key, attr in (("means", "mean"), ("scales", "scale"), ("rotations", "rotation"), ("colors", "color")):
        assert np.array_equal(d[key], np.array([getattr(x, attr) for x in g])), key
    assert np.array_equal(d["opacities"], np.array([x.opacity for x in g]))
