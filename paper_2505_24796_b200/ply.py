"""3DGS PLY checkpoints -> device-resident Gaussians.

The reference reads binary little-endian PLY in the 3DGS layout, keeping only
the SH DC term (``tilesplat.scene.load_ply``, src/tilesplat/scene.py:141-212).
This loader keeps the reference's activations, exception types and messages; its header parser is its own
(a statement regex grouped by element):

* opacity = sigmoid(stored);
* scale = exp(stored);
* quaternion normalised, where a zero quaternion raises ``SceneValidationError``;
* colour = clip(0.5 + SH_C0 * f_dc, 0, 1);
* ``SceneFormatError`` for a bad header, missing properties or a truncated
  body;
* ``SceneValidationError`` for zero vertices or out-of-range values.

In addition it keeps the higher SH bands. ``f_rest_*`` is stored
channel-major: ``f_rest_{c*(K-1) + k-1}`` holds channel c, coefficient k, as
3DGS's ``save_ply`` transposes it. The result is features [P, K, 3] with
K = (d+1)^2, so the B200 preprocess (K1) evaluates view-dependent colour.
Parsing is one vectorised ``np.frombuffer`` over the vertex block. Uploads go
through pinned host memory with non-blocking copies.
"""

from __future__ import annotations

import re

import numpy as np
import torch

from .raster import GaussianCloud

SH_C0 = 0.28209479177387814  # src/tilesplat/scene.py:11
QUAT_NORM_TOL = 1e-6          # src/tilesplat/scene.py:13


class SceneFormatError(ValueError):
    """A scene file cannot be parsed (src/tilesplat/scene.py:16-17)."""


class SceneValidationError(ValueError):
    """Scene contents violate an invariant (src/tilesplat/scene.py:20-21)."""


_REQUIRED = ("x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
             "rot_0", "rot_1", "rot_2", "rot_3")  # src/tilesplat/scene.py:108-123
_TYPES = {  # src/tilesplat/scene.py:125-138
    "float": "<f4", "float32": "<f4", "double": "<f8", "float64": "<f8", "uchar": "<u1", "uint8": "<u1",
    "int": "<i4", "int32": "<i4", "uint": "<u4", "uint32": "<u4", "short": "<i2", "ushort": "<u2",
}
_REST_COUNT_TO_DEGREE = {0: 0, 9: 1, 24: 2, 45: 3}


_HEADER_END = re.compile(rb"^end_header\r?\n", re.M)
# one header statement per line: a keyword and its arguments (PLY 1.0 header grammar)
_STATEMENT = re.compile(r"^\s*(format|element|property|comment|obj_info)\b\s*(.*?)\s*$", re.M)


def _split_header(path: str, data: bytes) -> tuple[str, bytes]:
    """(header text, body bytes); SceneFormatError unless the file starts with the PLY magic and has an end."""
    m = _HEADER_END.search(data)
    if not data.startswith(b"ply") or m is None:
        raise SceneFormatError(f"{path}: not a PLY file")
    return data[: m.start()].decode("ascii", errors="replace"), data[m.end():]


def _vertex_layout(path: str, head: str) -> tuple[int, list[tuple[str, str]]]:
    """Vertex count and the vertex element's (name, numpy type) fields, with the reference's checks
    (src/tilesplat/scene.py:148-193: binary little-endian, scalar properties of known types, the 3DGS fields)."""
    stmts = [(m.group(1), m.group(2).split()) for m in _STATEMENT.finditer(head)]
    formats = [a for k, a in stmts if k == "format"]
    if not formats or not formats[-1] or formats[-1][0] != "binary_little_endian":
        raise SceneFormatError(f"{path}: expected binary_little_endian format")
    # group property statements under the element statement that precedes them
    elements: dict[str, tuple[int, list[list[str]]]] = {}
    current = None
    for kind, args in stmts:
        if kind == "element":
            current = args[0] if args else ""
            elements[current] = (int(args[1]) if len(args) > 1 else 0, [])
        elif kind == "property" and current is not None:
            elements[current][1].append(args)
    if "vertex" not in elements:
        raise SceneFormatError(f"{path}: no vertex element")
    count, props = elements["vertex"]
    if count == 0:
        raise SceneValidationError(f"{path}: scene contains zero vertices")
    fields = []
    for args in props:
        if args and args[0] == "list":
            raise SceneFormatError(f"{path}: list properties unsupported")
        if not args or args[0] not in _TYPES:
            raise SceneFormatError(f"{path}: unsupported property type {args[0] if args else ''}")
        fields.append((args[1], _TYPES[args[0]]))
    missing = [p for p in _REQUIRED if p not in {n for n, _ in fields}]
    if missing:
        raise SceneFormatError(f"{path}: missing vertex property '{missing[0]}'")
    return count, fields


def read_ply(path: str) -> dict:
    """Parse a 3DGS PLY into SoA float64 arrays (reference activations) plus SH features.

    Returns ``means [P,3], scales [P,3], rotations [P,4] (w,x,y,z), opacities [P],
    colors [P,3]`` (the reference's Gaussian3D fields), ``sh_degree`` and
    ``features [P,(d+1)^2,3]`` (raw SH coefficients, DC first).
    """
    with open(path, "rb") as fh:
        data = fh.read()
    head, body = _split_header(path, data)
    count, fields = _vertex_layout(path, head)
    names = [n for n, _ in fields]
    dt = np.dtype(fields)
    if len(body) < count * dt.itemsize:
        raise SceneFormatError(f"{path}: truncated vertex data")
    v = np.frombuffer(body[: count * dt.itemsize], dtype=dt)

    def cols(*keys):
        return np.stack([v[k] for k in keys], axis=1).astype(np.float64)

    rest = sorted((n for n in names if n.startswith("f_rest_")), key=lambda n: int(n[len("f_rest_"):]))
    if len(rest) not in _REST_COUNT_TO_DEGREE:
        raise SceneFormatError(f"{path}: {len(rest)} f_rest properties (expected 0, 9, 24 or 45)")
    deg = _REST_COUNT_TO_DEGREE[len(rest)]
    K = (deg + 1) ** 2
    f_dc = cols("f_dc_0", "f_dc_1", "f_dc_2")
    feats = np.empty((count, K, 3), np.float64)
    feats[:, 0, :] = f_dc
    if K > 1:
        fr = cols(*rest).reshape(count, 3, K - 1)  # channel-major (3DGS save_ply transpose)
        feats[:, 1:, :] = fr.transpose(0, 2, 1)
    quats = cols("rot_0", "rot_1", "rot_2", "rot_3")
    norms = np.linalg.norm(quats, axis=1, keepdims=True)
    if np.any(norms == 0):
        raise SceneValidationError(f"{path}: zero quaternion")
    out = {
        "means": cols("x", "y", "z"),
        "scales": np.exp(cols("scale_0", "scale_1", "scale_2")),
        "rotations": quats / norms,
        "opacities": 1.0 / (1.0 + np.exp(-v["opacity"].astype(np.float64))),
        "colors": np.clip(0.5 + SH_C0 * f_dc, 0.0, 1.0),
        "features": feats,
        "sh_degree": deg,
    }
    validate(out, path)
    return out


def validate(d: dict, where: str = "scene") -> None:
    """Gaussian3D.validate over every Gaussian (src/tilesplat/scene.py:37-47), vectorised."""
    n = np.linalg.norm(d["rotations"], axis=1)
    checks = [
        (np.abs(n - 1.0) > QUAT_NORM_TOL, "quaternion not normalized"),
        (~((d["opacities"] > 0.0) & (d["opacities"] <= 1.0)), "opacity must lie in (0, 1]"),
        (np.any(d["scales"] <= 0.0, axis=1), "scale components must be positive"),
        (np.any((d["colors"] < 0.0) | (d["colors"] > 1.0), axis=1), "color components must lie in [0, 1]"),
    ]
    for bad, msg in checks:
        if np.any(bad):
            raise SceneValidationError(f"{msg} (gaussian {int(np.argmax(bad))}) in {where}")


def load_ply(path: str, device=None, dtype=torch.float32, sh: bool = True) -> GaussianCloud:
    """PLY -> device GaussianCloud (pinned-memory, non-blocking upload).

    ``sh=True`` keeps the full SH bands (view-dependent colour evaluated by K1).
    ``sh=False`` gives the reference's behaviour: DC colour only, clamped at load.
    ``dtype`` is the device storage type: float64 reproduces the reference's
    arrays bit for bit; float32 halves the upload.
    """
    d = read_ply(path)
    feats, deg = (d["features"], d["sh_degree"]) if sh else (d["colors"], -1)
    dev = torch.device(device or "cuda")

    def up(x):
        t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(dtype)
        if dev.type == "cuda":
            t = t.pin_memory().to(dev, non_blocking=True)
        return t.contiguous()

    cloud = GaussianCloud(up(d["means"]), up(d["scales"]), up(d["rotations"]), up(d["opacities"]), up(feats), deg)
    if dev.type == "cuda":
        torch.cuda.current_stream(dev).synchronize()
    return cloud


def write_ply(path: str, d: dict) -> None:
    """Write a scene dict (read_ply / synthetic layout) as a 3DGS binary PLY (inverse activations).

    ``features`` (if present, with ``sh_degree``) are stored as f_dc + channel-major f_rest.  Otherwise
    the DC term is derived from ``colors`` (colour = 0.5 + SH_C0 f_dc).
    """
    P = int(np.asarray(d["means"]).shape[0])
    deg = int(d.get("sh_degree", 0)) if "features" in d else 0
    K = (deg + 1) ** 2
    if "features" in d:
        feats = np.asarray(d["features"], np.float64).reshape(P, K, 3)
    else:
        feats = ((np.asarray(d["colors"], np.float64) - 0.5) / SH_C0).reshape(P, 1, 3)
    op = np.clip(np.asarray(d["opacities"], np.float64).reshape(P), 1e-12, 1.0 - 1e-12)
    cols = {
        "x": d["means"][:, 0], "y": d["means"][:, 1], "z": d["means"][:, 2],
        "f_dc_0": feats[:, 0, 0], "f_dc_1": feats[:, 0, 1], "f_dc_2": feats[:, 0, 2],
    }
    rest = feats[:, 1:, :].transpose(0, 2, 1).reshape(P, 3 * (K - 1))
    for i in range(3 * (K - 1)):
        cols[f"f_rest_{i}"] = rest[:, i]
    cols["opacity"] = np.log(op / (1.0 - op))
    for i in range(3):
        cols[f"scale_{i}"] = np.log(np.asarray(d["scales"], np.float64)[:, i])
    for i in range(4):
        cols[f"rot_{i}"] = np.asarray(d["rotations"], np.float64)[:, i]
    names = list(cols)
    rec = np.empty(P, dtype=np.dtype([(n, "<f4") for n in names]))
    for n in names:
        rec[n] = cols[n]
    header = ["ply", "format binary_little_endian 1.0", f"element vertex {P}"]
    header += [f"property float {n}" for n in names] + ["end_header"]
    with open(path, "wb") as fh:
        fh.write(("\n".join(header) + "\n").encode("ascii"))
        fh.write(rec.tobytes())
