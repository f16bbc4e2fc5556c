/*
 * tcgs_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, float64 restatement of the reference renderer `tilesplat`
 * (arxiv 2505.24796 reference package, /root/reference/pkg/src/tilesplat).
 * It is the CHECKER for the B200 product path (libtcgs.so): only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it.  Nothing in the product imports, links or executes it.
 *
 * Parity of this restatement is PINNED against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py imports tilesplat and records
 * projection records, tile lists, images, transmittance, per-pixel
 * contributor counts and FragmentStats), see tests/test_oracle_golden.py.
 *
 * Arithmetic follows the reference operation by operation:
 *   - numpy scalar/elementwise ops are plain IEEE double ops (no contraction:
 *     build with -ffp-contract=off);
 *   - numpy `@` on the small matrices goes through OpenBLAS 0.3.30 whose
 *     dgemm computes every entry as fma(a2,b2,fma(a1,b1,a0*b0)) and whose
 *     dgemv (3x3 @ 3) computes fma(a2,b2,fma(a0,b0,a1*b1)) -- measured in this
 *     container, see DESIGN.md "bit-exact preprocess";
 *   - np.linalg.norm of a 2-vector is sqrt(fma(v1,v1,v0*v0)) (ddot);
 *   - math.hypot is CPython 3.12's vector_norm (correctly rounded, with a
 *     differential correction), restated in py_hypot() below;
 *   - np.exp is approximated by libm exp (<= 1 ulp apart; only measure-zero
 *     threshold flips can result, which the golden tests would expose).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TILE 16
#define COV_DILATION 0.3          /* src/tilesplat/projection.py:14 */
#define MIN_EIGENVALUE 0.5        /* src/tilesplat/projection.py:18 */
#define ALPHA_CULL (1.0 / 255.0)  /* src/tilesplat/raster.py:15 */
#define TERM_THRESHOLD 0.0001     /* src/tilesplat/raster.py:16 */

typedef struct {
    double view[16]; /* row-major world->camera, src/tilesplat/scene.py:50-68 */
    double fx, fy, cx, cy, near_;
    int32_t width, height;
} ocam;

/* ---------------------------------------------------------------- helpers */
typedef struct { double hi, lo; } dl;
static inline dl dl_mul(double x, double y) { dl r; r.hi = x * y; r.lo = fma(x, y, -r.hi); return r; }
static inline dl dl_fast_sum(double a, double b) { dl r; r.hi = a + b; double z = r.hi - a; r.lo = b - z; return r; }

/* CPython 3.12 math.hypot (Modules/mathmodule.c vector_norm, n = 2). */
double py_hypot(double x, double y) {
    x = fabs(x); y = fabs(y);
    double mx = x > y ? x : y;
    if (isinf(mx)) return mx;
    if (isnan(x) || isnan(y)) return NAN;
    if (mx == 0.0) return mx;
    int max_e; frexp(mx, &max_e);
    if (max_e < -1023) return DBL_MIN * py_hypot(x / DBL_MIN, y / DBL_MIN);
    double scale = ldexp(1.0, -max_e);
    double csum = 1.0, frac1 = 0.0, frac2 = 0.0, v[2] = {x, y};
    for (int i = 0; i < 2; i++) {
        double t = v[i] * scale;
        dl pr = dl_mul(t, t);
        dl sm = dl_fast_sum(csum, pr.hi);
        csum = sm.hi; frac1 += pr.lo; frac2 += sm.lo;
    }
    double h = sqrt(csum - 1.0 + (frac1 + frac2));
    dl pr = dl_mul(-h, h);
    dl sm = dl_fast_sum(csum, pr.hi);
    csum = sm.hi; frac1 += pr.lo; frac2 += sm.lo;
    double xx = csum - 1.0 + (frac1 + frac2);
    h += xx / (2.0 * h);
    return h / scale;
}

/* OpenBLAS dgemm entry order for K = 3 (see header). */
static inline double dot3_gemm(double a0, double a1, double a2, double b0, double b1, double b2) {
    return fma(a2, b2, fma(a1, b1, a0 * b0));
}
/* OpenBLAS dgemv entry order for a 3x3 @ 3 product. */
static inline double dot3_gemv(double a0, double a1, double a2, double b0, double b1, double b2) {
    return fma(a2, b2, fma(a0, b0, a1 * b1));
}

/* src/tilesplat/scene.py:83-92 rotation_matrix, then :95-101 covariance_of. */
static void covariance_of(const double s[3], const double q[4], double cov[3][3]) {
    double w = q[0], x = q[1], y = q[2], z = q[3];
    double r[3][3] = {
        {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
        {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
        {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)},
    };
    double s2[3] = {s[0] * s[0], s[1] * s[1], s[2] * s[2]};
    double m[3][3], c[3][3];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) m[i][j] = r[i][j] * s2[j];
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) c[i][j] = dot3_gemm(m[i][0], m[i][1], m[i][2], r[j][0], r[j][1], r[j][2]);
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) cov[i][j] = (c[i][j] + c[j][i]) / 2.0;
}

/* src/tilesplat/projection.py:45-65 _clamp_eigenvalues (in place on a,b,c). */
static void clamp_eigenvalues(double *pa, double *pb, double *pc, double floor_) {
    double a = *pa, b = *pb, c = *pc;
    double mid = (a + c) / 2.0;
    double half = py_hypot((a - c) / 2.0, b);
    double lo = mid - half, hi = mid + half;
    if (lo >= floor_) return;
    double lo_c = lo > floor_ ? lo : floor_;
    double hi_c = hi > floor_ ? hi : floor_;
    if (half == 0.0) { *pa = lo_c; *pb = 0.0; *pc = lo_c; return; }
    double v0, v1;
    if (fabs(b) > 1e-300) { v0 = b; v1 = hi - a; }
    else if (a >= c) { v0 = 1.0; v1 = 0.0; }
    else { v0 = 0.0; v1 = 1.0; }
    double nrm = sqrt(fma(v1, v1, v0 * v0));
    v0 = v0 / nrm; v1 = v1 / nrm;
    double u0 = -v1, u1 = v0;
    /* hi_c * outer(v, v) + lo_c * outer(u, u) */
    *pa = hi_c * (v0 * v0) + lo_c * (u0 * u0);
    *pb = hi_c * (v0 * v1) + lo_c * (u0 * u1);
    *pc = hi_c * (v1 * v1) + lo_c * (u1 * u1);
}

/*
 * src/tilesplat/projection.py:68-116 project() for every Gaussian.
 * visible[i] = 0 where project() returns None (tz <= near, det <= 0).
 * Returns the dropped count (src/tilesplat/projection.py:119-134).
 */
int64_t oracle_project(int64_t P, const double *means, const double *scales, const double *quats,
                       const ocam *cam, uint8_t *visible, double *mean2d, double *inv_cov, double *depth,
                       int32_t *radius) {
    int64_t dropped = 0;
    const double *V = cam->view;
#pragma omp parallel for reduction(+ : dropped) schedule(static)
    for (int64_t i = 0; i < P; i++) {
        const double *mu = means + 3 * i;
        double t[3];
        for (int k = 0; k < 3; k++)
            t[k] = dot3_gemv(V[4 * k + 0], V[4 * k + 1], V[4 * k + 2], mu[0], mu[1], mu[2]) + V[4 * k + 3];
        double tz = t[2];
        visible[i] = 0;
        if (tz <= cam->near_) { dropped++; continue; }
        double mx = cam->fx * t[0] / tz + cam->cx;
        double my = cam->fy * t[1] / tz + cam->cy;
        double j00 = cam->fx / tz, j02 = -cam->fx * t[0] / (tz * tz);
        double j11 = cam->fy / tz, j12 = -cam->fy * t[1] / (tz * tz);
        double jac[2][3] = {{j00, 0.0, j02}, {0.0, j11, j12}};
        double cov[3][3];
        covariance_of(scales + 3 * i, quats + 4 * i, cov);
        double m[2][3], mc[2][3], sg[2][2];
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++)
                m[a][b] = dot3_gemm(jac[a][0], jac[a][1], jac[a][2], V[0 * 4 + b], V[1 * 4 + b], V[2 * 4 + b]);
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++)
                mc[a][b] = dot3_gemm(m[a][0], m[a][1], m[a][2], cov[0][b], cov[1][b], cov[2][b]);
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 2; b++) sg[a][b] = dot3_gemm(mc[a][0], mc[a][1], mc[a][2], m[b][0], m[b][1], m[b][2]);
        double sa = (sg[0][0] + sg[0][0]) / 2.0;
        double sb = (sg[0][1] + sg[1][0]) / 2.0;
        double sc = (sg[1][1] + sg[1][1]) / 2.0;
        sa += COV_DILATION;
        sc += COV_DILATION;
        clamp_eigenvalues(&sa, &sb, &sc, MIN_EIGENVALUE);
        double mid = (sa + sc) / 2.0;
        double lam_max = mid + py_hypot((sa - sc) / 2.0, sb);
        int32_t rad = (int32_t)ceil(3.0 * sqrt(lam_max));
        double det = sa * sc - sb * sb;
        if (det <= 0.0) { dropped++; continue; }
        visible[i] = 1;
        mean2d[2 * i + 0] = mx;
        mean2d[2 * i + 1] = my;
        inv_cov[3 * i + 0] = sc / det;
        inv_cov[3 * i + 1] = -sb / det;
        inv_cov[3 * i + 2] = sa / det;
        depth[i] = tz;
        radius[i] = rad;
    }
    return dropped;
}

/* src/tilesplat/tiling.py:34-43 covered_tiles as a clipped closed rectangle. */
static inline void tile_rect(double mx, double my, int32_t r, int tiles_x, int tiles_y, int *x0, int *x1, int *y0,
                             int *y1) {
    double fx0 = floor((mx - r) / TILE), fx1 = floor((mx + r) / TILE);
    double fy0 = floor((my - r) / TILE), fy1 = floor((my + r) / TILE);
    *x0 = fx0 < 0 ? 0 : (int)fx0;
    *y0 = fy0 < 0 ? 0 : (int)fy0;
    *x1 = fx1 > tiles_x - 1 ? tiles_x - 1 : (int)fx1;
    *y1 = fy1 > tiles_y - 1 ? tiles_y - 1 : (int)fy1;
}

typedef struct { double d; int64_t i; } dkey;
static int cmp_dkey(const void *a, const void *b) {
    const dkey *x = a, *y = b;
    if (x->d < y->d) return -1;
    if (x->d > y->d) return 1;
    return x->i < y->i ? -1 : (x->i > y->i);
}

/*
 * src/tilesplat/tiling.py:46-59 build_tiles: per-tile lists of Gaussian ids
 * (original indices; the reference stores survivor indices, which map 1:1
 * in order), each sorted ascending by float64 depth, stable by index.
 * Phase 1 (offsets == NULL ids == NULL) returns N and fills counts[n_tiles].
 */
int64_t oracle_tile_counts(int64_t P, const uint8_t *visible, const double *mean2d, const int32_t *radius,
                           int tiles_x, int tiles_y, int64_t *counts) {
    memset(counts, 0, sizeof(int64_t) * (size_t)tiles_x * tiles_y);
    int64_t n = 0;
    for (int64_t i = 0; i < P; i++) {
        if (!visible[i]) continue;
        int x0, x1, y0, y1;
        tile_rect(mean2d[2 * i], mean2d[2 * i + 1], radius[i], tiles_x, tiles_y, &x0, &x1, &y0, &y1);
        for (int ty = y0; ty <= y1; ty++)
            for (int tx = x0; tx <= x1; tx++) { counts[ty * tiles_x + tx]++; n++; }
    }
    return n;
}

void oracle_tile_lists(int64_t P, const uint8_t *visible, const double *mean2d, const int32_t *radius,
                       const double *depth, int tiles_x, int tiles_y, const int64_t *offsets, int32_t *ids) {
    int64_t nt = (int64_t)tiles_x * tiles_y;
    int64_t nv = 0;
    for (int64_t i = 0; i < P; i++) nv += visible[i] != 0;
    dkey *order = malloc(sizeof(dkey) * (size_t)(nv ? nv : 1));
    int64_t k = 0;
    for (int64_t i = 0; i < P; i++)
        if (visible[i]) { order[k].d = depth[i]; order[k].i = i; k++; }
    qsort(order, (size_t)nv, sizeof(dkey), cmp_dkey);
    int64_t *cursor = malloc(sizeof(int64_t) * (size_t)(nt ? nt : 1));
    memcpy(cursor, offsets, sizeof(int64_t) * (size_t)nt);
    for (int64_t k2 = 0; k2 < nv; k2++) {
        int64_t i = order[k2].i;
        int x0, x1, y0, y1;
        tile_rect(mean2d[2 * i], mean2d[2 * i + 1], radius[i], tiles_x, tiles_y, &x0, &x1, &y0, &y1);
        for (int ty = y0; ty <= y1; ty++)
            for (int tx = x0; tx <= x1; tx++) ids[cursor[ty * tiles_x + tx]++] = (int32_t)i;
    }
    free(cursor);
    free(order);
}

/*
 * src/tilesplat/raster.py:110-146 blend_tile + :161-201 render, restated per
 * pixel (the structure of tests/test_acceptance.py:157-203 replay_reference,
 * which the reference proves equivalent).  Alpha is the reference backend's
 * alpha_reference (src/tilesplat/raster.py:67-94).
 *
 * Tiles in [tile_row_begin, tile_row_end) are rendered (a band); rgb/T/count
 * are full-frame arrays.  stats[0..4] = f_blend, f_cull, f_skip,
 * pixels_terminated, n_splats (band).
 */
void oracle_blend(int width, int height, int tile_row_begin, int tile_row_end, const int64_t *offsets,
                  const int32_t *ids, const double *mean2d, const double *inv_cov, const double *opacity,
                  const double *color, double *rgb, double *T_out, int32_t *count_out, int64_t *stats) {
    int tiles_x = (width + TILE - 1) / TILE;
    int64_t fb = 0, fc = 0, fs = 0, pt = 0, ns = 0;
#pragma omp parallel for reduction(+ : fb, fc, fs, pt, ns) schedule(dynamic, 1) collapse(2)
    for (int ty = tile_row_begin; ty < tile_row_end; ty++) {
        for (int tx = 0; tx < tiles_x; tx++) {
            int64_t t = (int64_t)ty * tiles_x + tx;
            int64_t b = offsets[t], e = offsets[t + 1];
            ns += e - b;
            for (int py = ty * TILE; py < ty * TILE + TILE && py < height; py++) {
                for (int px = tx * TILE; px < tx * TILE + TILE && px < width; px++) {
                    double T = 1.0, c0 = 0.0, c1 = 0.0, c2 = 0.0;
                    int32_t cnt = 0;
                    int64_t j = b;
                    for (; j < e; j++) {
                        int64_t g = ids[j];
                        double s11 = inv_cov[3 * g], s12 = inv_cov[3 * g + 1], s22 = inv_cov[3 * g + 2];
                        double dx = mean2d[2 * g] - (double)px;
                        double dy = mean2d[2 * g + 1] - (double)py;
                        double q = s11 * dx * dx + 2.0 * s12 * dx * dy + s22 * dy * dy;
                        double alpha = opacity[g] * exp(-0.5 * q);
                        if (alpha < ALPHA_CULL) { fc++; continue; }
                        if (T - alpha * T < TERM_THRESHOLD) { pt++; break; }
                        double w = alpha * T;
                        c0 += w * color[3 * g];
                        c1 += w * color[3 * g + 1];
                        c2 += w * color[3 * g + 2];
                        T = T - w;
                        cnt++;
                    }
                    fb += cnt;
                    fs += e - j; /* the terminating fragment and every later one */
                    int64_t p = (int64_t)py * width + px;
                    rgb[3 * p] = c0; rgb[3 * p + 1] = c1; rgb[3 * p + 2] = c2;
                    T_out[p] = T;
                    count_out[p] = cnt;
                }
            }
        }
    }
    stats[0] = fb; stats[1] = fc; stats[2] = fs; stats[3] = pt; stats[4] = ns;
}

/*
 * Single-tile blend with caller-given per-splat alpha (the ConstantAlpha
 * evaluator of tests/test_raster.py:21-29), for the reference's blend KATs.
 */
/* Per-fragment classification of the reference blend loop (src/tilesplat/raster.py:110-146 with
 * alpha_reference, :67-94): cls[j*256 + 16*row + col] for tile-list entry j and tile pixel (col, row) is
 * 1 cull (alpha < 1/255), 2 blend, 3 terminate (T - alpha T < 1e-4, checked before compositing); entries the
 * pixel never reaches (after its termination) and out-of-image pixels stay 0.  Test infrastructure: the
 * first-divergent-fragment check of the GPU's contributor counts (tests/parity_util.py). */
void oracle_classify(int width, int height, int tile_row_begin, int tile_row_end, const int64_t *offsets,
                     const int32_t *ids, const double *mean2d, const double *inv_cov, const double *opacity,
                     uint8_t *cls) {
    int tiles_x = (width + TILE - 1) / TILE;
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
    for (int ty = tile_row_begin; ty < tile_row_end; ty++) {
        for (int tx = 0; tx < tiles_x; tx++) {
            int64_t t = (int64_t)ty * tiles_x + tx;
            int64_t b = offsets[t], e = offsets[t + 1];
            for (int py = ty * TILE; py < ty * TILE + TILE && py < height; py++) {
                for (int px = tx * TILE; px < tx * TILE + TILE && px < width; px++) {
                    const int64_t pix = (int64_t)(py - ty * TILE) * TILE + (px - tx * TILE);
                    double T = 1.0;
                    for (int64_t j = b; j < e; j++) {
                        int64_t g = ids[j];
                        double s11 = inv_cov[3 * g], s12 = inv_cov[3 * g + 1], s22 = inv_cov[3 * g + 2];
                        double dx = mean2d[2 * g] - (double)px;
                        double dy = mean2d[2 * g + 1] - (double)py;
                        double q = s11 * dx * dx + 2.0 * s12 * dx * dy + s22 * dy * dy;
                        double alpha = opacity[g] * exp(-0.5 * q);
                        if (alpha < ALPHA_CULL) { cls[j * 256 + pix] = 1; continue; }
                        if (T - alpha * T < TERM_THRESHOLD) { cls[j * 256 + pix] = 3; break; }
                        cls[j * 256 + pix] = 2;
                        T = T - alpha * T;
                    }
                }
            }
        }
    }
}

void oracle_blend_const_alpha(int n, const double *alpha, const double *color, double *rgb, double *T_out,
                              int32_t *count_out, int64_t *stats) {
    int64_t fb = 0, fc = 0, fs = 0, pt = 0;
    for (int p = 0; p < TILE * TILE; p++) {
        double T = 1.0, c[3] = {0, 0, 0};
        int32_t cnt = 0;
        int j = 0;
        for (; j < n; j++) {
            double a = alpha[j];
            if (a < ALPHA_CULL) { fc++; continue; }
            if (T - a * T < TERM_THRESHOLD) { pt++; break; }
            double w = a * T;
            for (int k = 0; k < 3; k++) c[k] += w * color[3 * j + k];
            T = T - w;
            cnt++;
        }
        fb += cnt;
        fs += n - j;
        for (int k = 0; k < 3; k++) rgb[3 * p + k] = c[k];
        T_out[p] = T;
        count_out[p] = cnt;
    }
    stats[0] = fb; stats[1] = fc; stats[2] = fs; stats[3] = pt;
}

/*
 * Spherical-harmonics colour, degrees 0..3 (NOT in the reference: it only has
 * the DC term, src/tilesplat/scene.py:11,195-197; parity UNPINNED for degree
 * >= 1).  Restates the de-facto 3DGS convention:
 * dir = normalise(mu - campos), campos = -R^T t, colour = clip(sum + 0.5, 0, 1).
 * feats is [P, (deg+1)^2, 3].
 */
void oracle_sh_color(int64_t P, int deg, const double *means, const double *feats, const double *view,
                     double *out) {
    static const double C0 = 0.28209479177387814, C1 = 0.4886025119029199;
    static const double C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005, -1.0925484305920792,
                                 0.5462742152960396};
    static const double C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658, 0.3731763325901154,
                                 -0.4570457994644658, 1.445305721320277, -0.5900435899266435};
    double cp[3];
    for (int k = 0; k < 3; k++)
        cp[k] = -(view[0 * 4 + k] * view[3] + view[1 * 4 + k] * view[7] + view[2 * 4 + k] * view[11]);
    int K = (deg + 1) * (deg + 1);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < P; i++) {
        const double *sh = feats + (size_t)i * K * 3;
        double dx = means[3 * i] - cp[0], dy = means[3 * i + 1] - cp[1], dz = means[3 * i + 2] - cp[2];
        double nn = sqrt(dx * dx + dy * dy + dz * dz);
        double x = dx / nn, y = dy / nn, z = dz / nn;
        for (int ch = 0; ch < 3; ch++) {
            double r = C0 * sh[0 * 3 + ch];
            if (deg >= 1) r += -C1 * y * sh[1 * 3 + ch] + C1 * z * sh[2 * 3 + ch] - C1 * x * sh[3 * 3 + ch];
            if (deg >= 2) {
                double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
                r += C2[0] * xy * sh[4 * 3 + ch] + C2[1] * yz * sh[5 * 3 + ch] +
                     C2[2] * (2.0 * zz - xx - yy) * sh[6 * 3 + ch] + C2[3] * xz * sh[7 * 3 + ch] +
                     C2[4] * (xx - yy) * sh[8 * 3 + ch];
                if (deg >= 3) {
                    r += C3[0] * y * (3.0 * xx - yy) * sh[9 * 3 + ch] + C3[1] * xy * z * sh[10 * 3 + ch] +
                         C3[2] * y * (4.0 * zz - xx - yy) * sh[11 * 3 + ch] +
                         C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy) * sh[12 * 3 + ch] +
                         C3[4] * x * (4.0 * zz - xx - yy) * sh[13 * 3 + ch] + C3[5] * z * (xx - yy) * sh[14 * 3 + ch] +
                         C3[6] * x * (xx - 3.0 * yy) * sh[15 * 3 + ch];
                }
            }
            r += 0.5;
            out[3 * i + ch] = r < 0.0 ? 0.0 : (r > 1.0 ? 1.0 : r);
        }
    }
}

double oracle_py_hypot(double x, double y) { return py_hypot(x, y); }
