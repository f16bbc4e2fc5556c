"""Helpers shared by the GPU parity tests (test infrastructure).

Two checks implement the north-star rule for the alpha path -- "per-pixel contributor counts identical
except where alpha lies within fp16 error of the cutoff" -- on top of K7's debug dump (tcgs_opts.dump_beta /
dump_class: the exponent K7 evaluated and the class it gave every (tile-list entry, tile pixel)):

* ``check_betas``: the a19 tolerance oracle.  Every exponent K7 evaluated is held to
  ``exact_dot(u, v) +- error_bound`` -- the reference's rigorous dot-product bound
  (src/tilesplat/precision.py:151-185: S ((1 + eps_in)^2 (1 + eps_acc)^n - 1)) with the GPU's own input and
  accumulation precisions (``BOUND_MODELS``).  The paper's fp16 K8 vector uses the reference's FP16 bound
  literally.
* ``first_divergences``: for every pixel, the first tile-list entry whose class (cull / blend / terminate)
  differs between K7 and the reference blend loop (oracle_classify, a C restatement of
  src/tilesplat/raster.py:110-146).  Later entries legitimately diverge; the first one must lie inside the
  error band of the cut it straddles: the EarlyCull cut (|beta - (-log2 255)| <= bound) or the termination
  test (|T (1 - alpha) - 1e-4| within the propagated fp32 error of T and alpha).

All exponents are in log2 units (K7 pre-scales the Gaussian vector by log2 e).
"""

from __future__ import annotations

import math

import numpy as np

LN255 = math.log(255.0)
LOG2E = 1.0 / math.log(2.0)
CUT_LOG2 = -LN255 * LOG2E   # EarlyCull: beta' < -log2 255 culls (src/tilesplat/tensor_path.py:79-81)
EX2_REL = 2.0 ** -21        # ex2.approx.ftz.f32: relative error of alpha (log2 units: ~2^-21 / ln 2)

# GPU arithmetic per alpha mode, restating precision.py:166-185's bound S ((1+eps_in)^2 (1+eps_acc)^n - 1):
#   eps_in  -- relative error of each vector entry as K7 feeds it to the dot product:
#              hi/lo:  the fp32 coefficient (<= 8 roundings, 2^-21 of its terms' magnitude) + the two-piece fp16
#                      split (residual <= 2^-22);
#              ffma:   the fp32 coefficient only;
#   eps_acc -- one accumulation step in fp32 (2^-23: one ulp, truncating accumulation allowed);
#   n       -- terms accumulated (16 for the K = 16 hi/lo MMA, 6 for the FFMA chain).
# S' sums the magnitudes of the terms each entry is computed from (no cancellation credit), and an absolute
# fp16-subnormal term covers tiny hi/lo pieces.  "k8" is the reference's own FP16 model (eps_H = 2^-10 covers the
# fp32 -> fp16 double rounding), plus the fp32 pre-rounding of the coefficient.
BOUND_MODELS = {
    "hilo": dict(eps_in=2.0 ** -21, eps_acc=2.0 ** -23, n=16),
    "ffma": dict(eps_in=2.0 ** -21, eps_acc=2.0 ** -23, n=6),
}


def _terms(mean2d, inv_cov, opacity, ids_e, tile_e, tiles_x):
    """Per entry: (dmx, dmy) = mean - tile centre, conic, ln o (float64 [E])."""
    g = ids_e
    tx = tile_e % tiles_x
    ty = tile_e // tiles_x
    dmx = mean2d[g, 0] - (16.0 * tx + 8.0)
    dmy = mean2d[g, 1] - (16.0 * ty + 8.0)
    s11, s12, s22 = inv_cov[g, 0], inv_cov[g, 1], inv_cov[g, 2]
    return dmx, dmy, s11, s12, s22, np.log(opacity[g])


_UX = np.tile(np.arange(16, dtype=np.float64), 16) - 8.0   # tile pixel i = 16 row + col
_UY = np.repeat(np.arange(16, dtype=np.float64), 16) - 8.0


def beta_and_bound(mode, mean2d, inv_cov, opacity, ids_e, tile_e, tiles_x):
    """Exact beta (log2 units, float64; gaussian_vector . pixel_vector in tile-local coordinates,
    src/tilesplat/tensor_path.py:25-53) and K7's rigorous error bound for entries ``ids_e`` x 256 pixels."""
    dmx, dmy, s11, s12, s22, lno = (x[:, None] for x in _terms(mean2d, inv_cov, opacity, ids_e, tile_e, tiles_x))
    ux, uy = _UX[None, :], _UY[None, :]
    ex, ey = dmx - ux, dmy - uy  # mean - pixel (alpha_reference, src/tilesplat/raster.py:67-74)
    beta = (lno - 0.5 * (s11 * ex * ex + 2.0 * s12 * ex * ey + s22 * ey * ey)) * LOG2E
    t0 = np.abs(lno) + 0.5 * (np.abs(s11) * dmx * dmx + 2.0 * np.abs(s12 * dmx * dmy) + np.abs(s22) * dmy * dmy)
    t1 = np.abs(ux) * (np.abs(s11 * dmx) + np.abs(s12 * dmy))
    t2 = np.abs(uy) * (np.abs(s12 * dmx) + np.abs(s22 * dmy))
    t3 = 0.5 * np.abs(s11) * ux * ux + np.abs(s12 * ux * uy) + 0.5 * np.abs(s22) * uy * uy
    s_mag = (t0 + t1 + t2 + t3) * LOG2E
    au, av = np.abs(ux), np.abs(uy)
    if mode == "k8":
        # the reference's error_bound(u, v, FP16).rigorous on the padded length-8 vectors
        v0 = (lno - 0.5 * (s11 * dmx * dmx + 2.0 * s12 * dmx * dmy + s22 * dmy * dmy))
        v1, v2 = s11 * dmx + s12 * dmy, s12 * dmx + s22 * dmy
        S = (np.abs(v0) + np.abs(v1) * au + np.abs(v2) * av + 0.5 * np.abs(s11) * ux * ux
             + np.abs(s12 * ux * uy) + 0.5 * np.abs(s22) * uy * uy) * LOG2E
        eh, ef = 2.0 ** -10, 2.0 ** -24
        b = S * ((1.0 + eh) ** 2 * (1.0 + ef) ** 8 - 1.0) + 2.0 ** -21 * s_mag
        b = b + 2.0 ** -25 * (3.0 + au + av + au * au + au * av + av * av)  # fp16 subnormal spacing
    else:
        m = BOUND_MODELS[mode]
        b = s_mag * ((1.0 + m["eps_in"]) ** 2 * (1.0 + m["eps_acc"]) ** m["n"] - 1.0)
        if mode == "hilo":
            b = b + 2.0 ** -24 * (4.0 + 2.0 * (au + av + au * au + au * av + av * av))
    return beta, b


def tiles_of_entries(offsets):
    n_t = len(offsets) - 1
    return np.repeat(np.arange(n_t, dtype=np.int64), np.diff(np.asarray(offsets, np.int64)))


def check_betas(beta_gpu, cls_gpu, offsets, ids, mean2d, inv_cov, opacity, width, mode, chunk=1 << 15):
    """a19: every evaluated exponent within exact +- bound.  Returns (n_checked, n_violations, max |err|/bound)."""
    tiles_x = (width + 15) // 16
    tile_e = tiles_of_entries(offsets)
    ids = np.asarray(ids, np.int64)
    n_chk = n_bad = 0
    worst = 0.0
    for e0 in range(0, len(ids), chunk):
        e1 = min(e0 + chunk, len(ids))
        beta, b = beta_and_bound(mode, mean2d, inv_cov, opacity, ids[e0:e1], tile_e[e0:e1], tiles_x)
        ev = (cls_gpu[e0:e1] > 0) & (cls_gpu[e0:e1] < 4)
        err = np.abs(beta_gpu[e0:e1].astype(np.float64) - beta)
        n_chk += int(ev.sum())
        n_bad += int(np.count_nonzero(ev & ~(err <= b)))
        if ev.any():
            worst = max(worst, float(np.max(err[ev] / b[ev])))
    return n_chk, n_bad, worst


def merge_dead(cls_gpu, cls_ref):
    """K7's class 4 marks a Gaussian its producer found dead on the whole tile (box test): a cull where the pixel is
    still live, nothing after it terminated -- it agrees with a reference cull (1) or unreached entry (0)."""
    g = cls_gpu.copy()
    wild = (g == 4) & (cls_ref <= 1)
    g[wild] = cls_ref[wild]
    return g


def replay_T(mode, ids_list, tile, i, mean2d, inv_cov, opacity, upto, tiles_x):
    """Reference transmittance before list position ``upto`` at tile pixel ``i`` of ``tile`` (float64,
    raster.py:110-146), and the first-order relative error K7's fp32 T has accumulated by then: each blend
    multiplies T by (1 - alpha) with alpha known to (2^b - 1) + ex2 error, plus one fp32 rounding."""
    T, rel = 1.0, 0.0
    if upto == 0:
        return T, rel
    lst = np.asarray(ids_list[:upto], np.int64)
    beta, b = beta_and_bound(mode, mean2d, inv_cov, opacity, lst, np.full(upto, tile, np.int64), tiles_x)
    tx, ty = tile % tiles_x, tile // tiles_x
    px, py = 16 * tx + i % 16, 16 * ty + i // 16
    for j in range(upto):
        g = lst[j]
        s11, s12, s22 = inv_cov[g]
        dx, dy = mean2d[g, 0] - px, mean2d[g, 1] - py
        a = opacity[g] * math.exp(-0.5 * (s11 * dx * dx + 2.0 * s12 * dx * dy + s22 * dy * dy))
        if a < 1.0 / 255.0:
            continue
        if T - a * T < 1e-4:
            break
        d_a = (2.0 ** float(b[j, i]) - 1.0) + EX2_REL
        rel += a * d_a / max(1.0 - a, 1e-12) + 2.0 ** -23
        T -= a * T
    return T, rel


def first_divergences(cls_gpu, cls_ref, beta_gpu, offsets, ids, mean2d, inv_cov, opacity, width, height, mode,
                      max_report=20):
    """For every pixel, the first entry where K7's class differs from the reference's must lie in the error band
    of the cut it straddles.  Returns (n_divergent_pixels, unexplained [(x, y, entry, gpu, ref, why)])."""
    tiles_x = (width + 15) // 16
    g = merge_dead(cls_gpu, cls_ref)
    diff_e, diff_i = np.nonzero(g != cls_ref)
    if diff_e.size == 0:
        return 0, []
    tile_e = tiles_of_entries(offsets)
    key = tile_e[diff_e] * 256 + diff_i
    _, first = np.unique(key, return_index=True)  # nonzero() is row-major: the first hit has the smallest entry
    ids = np.asarray(ids, np.int64)
    unexplained = []
    for k in first.tolist():
        e, i = int(diff_e[k]), int(diff_i[k])
        t = int(tile_e[e])
        px, py = (t % tiles_x) * 16 + i % 16, (t // tiles_x) * 16 + i // 16
        beta, b = beta_and_bound(mode, mean2d, inv_cov, opacity, ids[e:e + 1], tile_e[e:e + 1], tiles_x)
        beta, b = float(beta[0, i]), float(b[0, i])
        cg, cr = int(g[e, i]), int(cls_ref[e, i])
        ok = False
        why = ""
        if cg == 4:  # K7 found the Gaussian dead on the whole tile where the reference passes it
            why = f"dead-box cull of a passing fragment (beta = {beta:.6g}, cut {CUT_LOG2:.6g})"
        elif 1 in (cg, cr) and cg != cr:  # a pass/cull flip at the EarlyCull (or alpha) cut
            ok = abs(beta - CUT_LOG2) <= b + EX2_REL * LOG2E
            why = f"cull flip: |beta - cut| = {abs(beta - CUT_LOG2):.3g} vs bound {b:.3g}"
        elif {cg, cr} == {2, 3}:  # blend vs terminate
            lst = ids[offsets[t]:offsets[t + 1]]
            T, rel = replay_T(mode, lst, t, i, mean2d, inv_cov, opacity, e - int(offsets[t]), tiles_x)
            a = 2.0 ** beta
            d_a = (2.0 ** b - 1.0) + EX2_REL
            tn = T - a * T
            tol = abs(tn) * rel + T * a * d_a + 2.0 ** -23 * T + 1e-12
            ok = abs(tn - 1e-4) <= tol
            why = f"termination flip: |T(1-a) - 1e-4| = {abs(tn - 1e-4):.3g} vs {tol:.3g}"
        else:
            why = "not a cut flip"
        if not ok:
            unexplained.append((px, py, e, cg, cr, why))
            if len(unexplained) >= max_report:
                break
    return len(first), unexplained


def psnr(a, b) -> float:
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(1.0 / mse)
