"""Helpers shared by the GPU parity tests (test infrastructure).

``explain_count_mismatches`` implements the north-star rule for per-pixel
contributor counts: they must be identical "except where alpha lies within
fp16 error of the cutoff".  For every pixel whose GPU count differs from the
reference, the pixel's fragment sequence is replayed in float64 and the
mismatch is accepted only if some reached fragment sits within the
arithmetic's error band of the EarlyCull cutoff (|beta + ln 255| small) or of
the termination threshold (T (1 - alpha) close to 1e-4).
"""

from __future__ import annotations

import math

import numpy as np

LN255 = math.log(255.0)

# beta error band per alpha mode: fp16 K8 (paper layout, src/tilesplat/precision.py:166 error_bound with
# eps_H = 2^-11 over the length-8 dot) vs the hi/lo K16 split (~2^-22 relative) vs FP32 FFMA.
def beta_band(mode: str, S: float) -> float:
    if mode == "k8":
        return 2.0 * (2.0 ** -11) * S * 1.5 + 1e-4
    if mode == "hilo":
        return 64.0 * (2.0 ** -24) * S + 2e-5
    return 32.0 * (2.0 ** -24) * S + 2e-5


def gaussian_vector(mx, my, s11, s12, s22, o, ox, oy):
    dmx, dmy = mx - ox, my - oy
    v0 = math.log(o) - 0.5 * (s11 * dmx * dmx + 2.0 * s12 * dmx * dmy + s22 * dmy * dmy)
    return np.array([v0, s11 * dmx + s12 * dmy, s12 * dmx + s22 * dmy, -0.5 * s11, -s12, -0.5 * s22])


def explain_count_mismatches(gpu_counts, ref_counts, offsets, ids, mean2d, inv_cov, opacity, width, mode,
                             max_report=20):
    """Returns (n_mismatch, list of unexplained pixel descriptions)."""
    tiles_x = (width + 15) // 16
    ys, xs = np.nonzero(gpu_counts != ref_counts)
    unexplained = []
    for y, x in zip(ys, xs):
        t = (y // 16) * tiles_x + (x // 16)
        ox, oy = (x // 16) * 16 + 8.0, (y // 16) * 16 + 8.0
        u = np.array([1.0, x - ox, y - oy, (x - ox) ** 2, (x - ox) * (y - oy), (y - oy) ** 2])
        T = 1.0
        rel_T = 0.0  # first-order relative error of T accumulated through the blended fragments
        near = False
        for g in ids[offsets[t]:offsets[t + 1]]:
            v = gaussian_vector(mean2d[g, 0], mean2d[g, 1], *inv_cov[g], opacity[g], ox, oy)
            beta = float(u @ v)
            band = beta_band(mode, float(np.sum(np.abs(u * v))))
            if abs(beta + LN255) <= band:
                near = True
                break
            if beta < -LN255:
                continue
            a = min(math.exp(beta), 1.0)
            tn = T - a * T
            err = tn * rel_T + T * a * (math.exp(band) - 1.0) + 1e-7
            if abs(tn - 1e-4) <= err:
                near = True
                break
            if tn < 1e-4:
                break
            rel_T += a * band / max(1.0 - a, 1e-6) + 2e-7
            T = tn
        if not near:
            unexplained.append((int(x), int(y), int(gpu_counts[y, x]), int(ref_counts[y, x])))
            if len(unexplained) >= max_report:
                break
    return len(ys), unexplained


def psnr(a, b) -> float:
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)
