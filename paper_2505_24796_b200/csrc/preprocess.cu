// preprocess.cu -- K1: EWA projection of every Gaussian in float64 (sm_100a).
//
// Replaces tilesplat.projection.project / project_scene
// (/root/reference/pkg/src/tilesplat/projection.py:68-134), covariance_of
// (src/tilesplat/scene.py:83-101) and tiling.covered_tiles
// (src/tilesplat/tiling.py:34-43).  One thread per Gaussian; HBM-bound
// (reads 56 B of geometry + 12*(d+1)^2 B of SH, writes a 48 B render record,
// an 8 B tile rectangle, a 4 B tile count and an 8 B depth key).
//
// Bit-exactness: this translation unit is compiled with --fmad=false so every
// a*b+c below is two IEEE roundings exactly as numpy evaluates it; the
// explicit fma() calls reproduce OpenBLAS's dgemm/dgemv operation order
// for the reference's small matmuls (measured: DESIGN.md "bit-exact
// preprocess"), and py_hypot() restates CPython's math.hypot.  Radius, tile
// rectangles, mean2d and depth therefore equal the reference's bit for bit,
// which the binning parity test checks.
#include <float.h>

#include "tcgs_internal.cuh"

#ifndef TCGS_K1_THREADS
#define TCGS_K1_THREADS 256  // Gaussians (threads) per CTA, fp32 scenes
#endif

namespace tcgs {

namespace {

struct dl {
    double hi, lo;
};
__device__ __forceinline__ dl dl_mul(double x, double y) {
    dl r;
    r.hi = x * y;
    r.lo = fma(x, y, -r.hi);
    return r;
}
__device__ __forceinline__ dl dl_fast_sum(double a, double b) {
    dl r;
    r.hi = a + b;
    double z = r.hi - a;
    r.lo = b - z;
    return r;
}

// CPython 3.12 math.hypot for two arguments (vector_norm with differential correction).
__device__ double py_hypot(double x, double y) {
    x = fabs(x);
    y = fabs(y);
    double mx = x > y ? x : y;
    if (isinf(mx)) return mx;
    if (isnan(x) || isnan(y)) return __longlong_as_double(0x7ff8000000000000ll);
    if (mx == 0.0) return mx;
    int max_e;
    frexp(mx, &max_e);
    double pre = 1.0;
    if (max_e < -1023) {  // subnormal inputs: rescale (never hit by projected covariances)
        x /= DBL_MIN;
        y /= DBL_MIN;
        mx /= DBL_MIN;
        pre = DBL_MIN;
        frexp(mx, &max_e);
    }
    double scale = ldexp(1.0, -max_e);
    double csum = 1.0, frac1 = 0.0, frac2 = 0.0;
    double v[2] = {x, y};
#pragma unroll
    for (int i = 0; i < 2; i++) {
        double t = v[i] * scale;
        dl pr = dl_mul(t, t);
        dl sm = dl_fast_sum(csum, pr.hi);
        csum = sm.hi;
        frac1 += pr.lo;
        frac2 += sm.lo;
    }
    double h = sqrt(csum - 1.0 + (frac1 + frac2));
    dl pr = dl_mul(-h, h);
    dl sm = dl_fast_sum(csum, pr.hi);
    csum = sm.hi;
    frac1 += pr.lo;
    frac2 += sm.lo;
    double xx = csum - 1.0 + (frac1 + frac2);
    h += xx / (2.0 * h);
    return pre * (h / scale);
}

// OpenBLAS dgemm / dgemv entry order for K = 3.
__device__ __forceinline__ double dot3_gemm(double a0, double a1, double a2, double b0, double b1, double b2) {
    return fma(a2, b2, fma(a1, b1, a0 * b0));
}
__device__ __forceinline__ double dot3_gemv(double a0, double a1, double a2, double b0, double b1, double b2) {
    return fma(a2, b2, fma(a0, b0, a1 * b1));
}

template <typename T>
__device__ __forceinline__ double ld(const T *p, int64_t i) {  // p: shared memory (staged inputs)
    return static_cast<double>(p[i]);
}

// ---- input staging: every array segment of the CTA's Gaussians is copied into shared memory with one
// TMA bulk copy (cp.async.bulk, 16-B aligned segments) or, for a ragged tail, a coalesced cooperative loop;
// the per-thread AoS reads (e.g. 48 SH floats at a 192-B stride) then hit shared memory instead of L1.
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <typename T>
__device__ __forceinline__ bool bulk_ok(const T *src, int64_t elems) {
    return ((reinterpret_cast<uintptr_t>(src) & 15) == 0) && ((elems * (int64_t)sizeof(T)) % 16 == 0) && elems > 0;
}

// 3DGS spherical-harmonics colour (degree <= 3), NOT in the reference (parity unpinned, SURVEY.md
// Appendix E; oracle/tcgs_oracle.c:oracle_sh_color is the float64 restatement it is tested against).
// The basis is evaluated once per Gaussian and dotted with the three channels in fp32 FMA: the colour is
// stored as fp32 anyway, and the fp32 evaluation stays within ~1e-6 of the float64 restatement.
template <typename T>
__device__ void sh_color(const T *sh, int deg, double dx, double dy, double dz, float out[3]) {
    const float x = (float)dx, y = (float)dy, z = (float)dz;
    float b[16];
    b[0] = 0.28209479177387814f;
    int K = 1;
    if (deg >= 1) {
        const float C1 = 0.4886025119029199f;
        b[1] = -C1 * y;
        b[2] = C1 * z;
        b[3] = -C1 * x;
        K = 4;
    }
    if (deg >= 2) {
        const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
        b[4] = 1.0925484305920792f * xy;
        b[5] = -1.0925484305920792f * yz;
        b[6] = 0.31539156525252005f * (2.0f * zz - xx - yy);
        b[7] = -1.0925484305920792f * xz;
        b[8] = 0.5462742152960396f * (xx - yy);
        K = 9;
        if (deg >= 3) {
            b[9] = -0.5900435899266435f * y * (3.0f * xx - yy);
            b[10] = 2.890611442640554f * xy * z;
            b[11] = -0.4570457994644658f * y * (4.0f * zz - xx - yy);
            b[12] = 0.3731763325901154f * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
            b[13] = -0.4570457994644658f * x * (4.0f * zz - xx - yy);
            b[14] = 1.445305721320277f * z * (xx - yy);
            b[15] = -0.5900435899266435f * x * (xx - 3.0f * yy);
            K = 16;
        }
    }
    float r0 = 0.0f, r1 = 0.0f, r2 = 0.0f;
    if (sizeof(T) == 4 && K == 16) {
        // 48 floats per Gaussian = 12 LDS.128 (a 192-B per-thread stride: 4-way bank conflicts instead of
        // the 16-way of scalar loads)
        const float4 *v = reinterpret_cast<const float4 *>(sh);
#pragma unroll
        for (int q = 0; q < 12; q++) {
            const float4 f = v[q];
            const float e[4] = {f.x, f.y, f.z, f.w};
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const int idx = 4 * q + u, k = idx / 3, ch = idx % 3;
                float &acc = ch == 0 ? r0 : (ch == 1 ? r1 : r2);
                acc = __fmaf_rn(b[k], e[u], acc);
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < 16; k++)
            if (k < K) {
                r0 = __fmaf_rn(b[k], (float)sh[3 * k + 0], r0);
                r1 = __fmaf_rn(b[k], (float)sh[3 * k + 1], r1);
                r2 = __fmaf_rn(b[k], (float)sh[3 * k + 2], r2);
            }
    }
    out[0] = fminf(fmaxf(r0 + 0.5f, 0.0f), 1.0f);
    out[1] = fminf(fmaxf(r1 + 0.5f, 0.0f), 1.0f);
    out[2] = fminf(fmaxf(r2 + 0.5f, 0.0f), 1.0f);
}

struct PreArgs {
    tcgs_camera cam;
    double campos[3];
    int64_t P;
    int sh_degree;
    int tiles_x, tiles_y, band_y0, band_y1;
    int debug;
    int coverage;      // enum tcgs_coverage
    int defer_colour;  // 1: geometry only (no feature staging, no colour); tcgs_colour fills rgb later
    Rec *rec;
    short4 *rect;
    unsigned long long *keys;
    uint32_t *idx;
    int32_t *radius;
    double *dbg_conic;
    double *dbg_depth;
    double *dbg_mean2d;
    DevCounters *ctr;
};

// Views of one pass: every view reads the same staged Gaussians (multi-view fused preprocess, SURVEY.md
// §8(f) 2: the SH coefficients -- 192 B of the 236 B per Gaussian at SH3 -- are read once for NV cameras).
template <int NV>
struct PreViews {
    PreArgs v[NV];
    int n;
};

#ifndef TCGS_K1_VIEWS_MIN_CTAS
#define TCGS_K1_VIEWS_MIN_CTAS 3  // multi-view pass: resident CTAs per SM the register allocation must allow
#endif

template <typename T, int NV>
__global__ void __launch_bounds__(256, NV == 1 ? 1 : TCGS_K1_VIEWS_MIN_CTAS) preprocess_kernel(const __grid_constant__ PreViews<NV> pv,
                                                         const T *__restrict__ g_means,
                                                         const T *__restrict__ g_scales, const T *__restrict__ g_rots,
                                                         const T *__restrict__ g_opac, const T *__restrict__ g_feats) {
    const PreArgs &a0 = pv.v[0];  // scene-level fields (P, sh_degree) are the same in every view
    extern __shared__ __align__(16) unsigned char pre_smem[];
    // two transaction barriers: geometry (means, scales, rotations, opacity) and features (RGB or SH), so the
    // features' bulk copy -- most of the bytes at SH3 -- lands while the float64 projection runs
    __shared__ __align__(8) unsigned long long bar[2];
    const int NT = blockDim.x;
    const int64_t base = (int64_t)blockIdx.x * NT;
    const int n = (int)(a0.P - base < NT ? a0.P - base : NT);
    // features per Gaussian (none staged when the colour is deferred)
    const int F = a0.defer_colour ? 0 : (a0.sh_degree < 0 ? 3 : 3 * (a0.sh_degree + 1) * (a0.sh_degree + 1));
    // staged SoA segments, each 16-B aligned: means 3, scales 3, rotations 4, opacity 1, features F per Gaussian
    const int per[5] = {3, 3, 4, 1, F};
    const T *src[5] = {g_means, g_scales, g_rots, g_opac, g_feats};
    T *seg[5];
    {
        size_t off = 0;
        for (int q = 0; q < 5; q++) {
            seg[q] = reinterpret_cast<T *>(pre_smem + off);
            off += (((size_t)per[q] * NT * sizeof(T)) + 15) / 16 * 16;
        }
    }
    bool bulk[5];
    bool any_bulk[2] = {false, false};
    for (int q = 0; q < 5; q++) {
        bulk[q] = bulk_ok(src[q] + base * per[q], (int64_t)n * per[q]);
        any_bulk[q == 4] |= bulk[q];
    }
    if (threadIdx.x == 0) {
        for (int g = 0; g < 2; g++)
            if (any_bulk[g]) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[g])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int g = 0; g < 2; g++) {
            if (!any_bulk[g]) continue;
            uint32_t tx = 0;
            for (int q = g ? 4 : 0; q < (g ? 5 : 4); q++)
                if (bulk[q]) tx += (uint32_t)(n * per[q] * sizeof(T));
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[g])), "r"(tx)
                         : "memory");
            for (int q = g ? 4 : 0; q < (g ? 5 : 4); q++)
                if (bulk[q]) bulk_g2s(seg[q], src[q] + base * per[q], (uint32_t)(n * per[q] * sizeof(T)), &bar[g]);
        }
    }
    for (int q = 0; q < 5; q++)  // ragged / unaligned segments: coalesced cooperative copy
        if (!bulk[q])
            for (int e = threadIdx.x; e < n * per[q]; e += NT) seg[q][e] = src[q][base * per[q] + e];
    // PDL: the scene inputs are never written by a libtcgs kernel, so they stream in -- and the projection runs --
    // while the previous kernels of the stream finish; pdl_wait() comes right before the first workspace write
    pdl_launch();
    auto wait_bar = [&](int g) {
        if (any_bulk[g]) {
            asm volatile(
                "{\n"
                ".reg .pred P1;\n"
                "WAIT_%=:\n"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
                "@!P1 bra WAIT_%=;\n"
                "}\n" ::"r"(smem_u32(&bar[g]))
                : "memory");
        }
    };
    wait_bar(0);
    __syncthreads();
    const int l = threadIdx.x;
    const T *means = seg[0], *scales = seg[1], *rots = seg[2], *opac = seg[3], *feats = seg[4];
    const int64_t i = base + l;
    // covariance_of (src/tilesplat/scene.py:83-101): view-independent, computed once for every view of the pass
    double w, x, y, z;
    if (sizeof(T) == 4) {
        const float4 q4 = reinterpret_cast<const float4 *>(rots)[l];
        w = q4.x, x = q4.y, y = q4.z, z = q4.w;
    } else {
        w = ld(rots, 4 * l), x = ld(rots, 4 * l + 1), y = ld(rots, 4 * l + 2), z = ld(rots, 4 * l + 3);
    }
    const double r[3][3] = {
        {1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)},
        {2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)},
        {2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)},
    };
    const double s0 = ld(scales, 3 * l), s1 = ld(scales, 3 * l + 1), s2 = ld(scales, 3 * l + 2);
    const double sq[3] = {s0 * s0, s1 * s1, s2 * s2};
    double mm[3][3], c[3][3], cov[3][3];
#pragma unroll
    for (int p = 0; p < 3; p++)
#pragma unroll
        for (int q = 0; q < 3; q++) mm[p][q] = r[p][q] * sq[q];
#pragma unroll
    for (int p = 0; p < 3; p++)
#pragma unroll
        for (int q = 0; q < 3; q++) c[p][q] = dot3_gemm(mm[p][0], mm[p][1], mm[p][2], r[q][0], r[q][1], r[q][2]);
#pragma unroll
    for (int p = 0; p < 3; p++)
#pragma unroll
        for (int q = 0; q < 3; q++) cov[p][q] = (c[p][q] + c[q][p]) / 2.0;
    const int nv = NV == 1 ? 1 : pv.n;
    for (int vi = 0; vi < nv; vi++) {
        const PreArgs &a = pv.v[vi];
        const bool in_range = i < a.P;
        unsigned long long key = ~0ull;  // "touches nothing": rewritten by depth_key_fix
        uint32_t touched = 0;
        short4 rect = make_short4(0, 0, -1, -1);  // empty: touches no tile (binning reads the rectangle only)
        bool dropped = false;
        if (in_range) {
            const double *V = a.cam.view;
            const double m0 = ld(means, 3 * l), m1 = ld(means, 3 * l + 1), m2 = ld(means, 3 * l + 2);
            double t[3];
#pragma unroll
            for (int k = 0; k < 3; k++) t[k] = dot3_gemv(V[4 * k + 0], V[4 * k + 1], V[4 * k + 2], m0, m1, m2) + V[4 * k + 3];
            const double tz = t[2];
            if (a.debug) {  // the radius only feeds tcgs_copy_projection (debug)
                pdl_wait();
                a.radius[i] = -1;
            }
            if (!(tz > a.cam.near_plane)) {  // src/tilesplat/projection.py:76-78 (tz <= near culls)
                dropped = true;
            } else {
                const double fx = a.cam.fx, fy = a.cam.fy;
                const double mx = fx * t[0] / tz + a.cam.cx;
                const double my = fy * t[1] / tz + a.cam.cy;
                const double jac[2][3] = {{fx / tz, 0.0, -fx * t[0] / (tz * tz)}, {0.0, fy / tz, -fy * t[1] / (tz * tz)}};
                // sigma = (J W) Sigma (J W)^T  (src/tilesplat/projection.py:88-96)
                double m[2][3], mc[2][3], sg[2][2];
#pragma unroll
                for (int p = 0; p < 2; p++)
#pragma unroll
                    for (int q = 0; q < 3; q++) m[p][q] = dot3_gemm(jac[p][0], jac[p][1], jac[p][2], V[q], V[4 + q], V[8 + q]);
#pragma unroll
                for (int p = 0; p < 2; p++)
#pragma unroll
                    for (int q = 0; q < 3; q++) mc[p][q] = dot3_gemm(m[p][0], m[p][1], m[p][2], cov[0][q], cov[1][q], cov[2][q]);
#pragma unroll
                for (int p = 0; p < 2; p++)
#pragma unroll
                    for (int q = 0; q < 2; q++) sg[p][q] = dot3_gemm(mc[p][0], mc[p][1], mc[p][2], m[q][0], m[q][1], m[q][2]);
                double sa = (sg[0][0] + sg[0][0]) / 2.0;
                double sb = (sg[0][1] + sg[1][0]) / 2.0;
                double sc = (sg[1][1] + sg[1][1]) / 2.0;
                sa += 0.3;  // COV_DILATION, src/tilesplat/projection.py:14
                sc += 0.3;
                {  // _clamp_eigenvalues(sigma, 0.5), src/tilesplat/projection.py:45-65
                    const double mid = (sa + sc) / 2.0;
                    const double half = py_hypot((sa - sc) / 2.0, sb);
                    const double lo = mid - half, hi = mid + half;
                    if (!(lo >= 0.5)) {
                        const double lo_c = lo > 0.5 ? lo : 0.5, hi_c = hi > 0.5 ? hi : 0.5;
                        if (half == 0.0) {
                            sa = lo_c;
                            sb = 0.0;
                            sc = lo_c;
                        } else {
                            double v0, v1;
                            if (fabs(sb) > 1e-300) {
                                v0 = sb;
                                v1 = hi - sa;
                            } else if (sa >= sc) {
                                v0 = 1.0;
                                v1 = 0.0;
                            } else {
                                v0 = 0.0;
                                v1 = 1.0;
                            }
                            const double nrm = sqrt(fma(v1, v1, v0 * v0));
                            v0 = v0 / nrm;
                            v1 = v1 / nrm;
                            const double u0 = -v1, u1 = v0;
                            sa = hi_c * (v0 * v0) + lo_c * (u0 * u0);
                            sb = hi_c * (v0 * v1) + lo_c * (u0 * u1);
                            sc = hi_c * (v1 * v1) + lo_c * (u1 * u1);
                        }
                    }
                }
                const double mid = (sa + sc) / 2.0;
                const double lam_max = mid + py_hypot((sa - sc) / 2.0, sb);
                const int32_t rad = (int32_t)ceil(3.0 * sqrt(lam_max));
                const double det = sa * sc - sb * sb;
                if (!(det > 0.0)) {  // invert_cov2 raises -> project returns None (projection.py:104-107)
                    dropped = true;
                } else {
                    const double s11 = sc / det, s12 = -sb / det, s22 = sa / det;
                    if (a.debug) a.radius[i] = rad;  // (after the pdl_wait above)
                    if (a.debug) {
                        a.dbg_conic[3 * i] = s11;
                        a.dbg_conic[3 * i + 1] = s12;
                        a.dbg_conic[3 * i + 2] = s22;
                        a.dbg_depth[i] = tz;
                        a.dbg_mean2d[2 * i] = mx;
                        a.dbg_mean2d[2 * i + 1] = my;
                    }
                    // covered_tiles (src/tilesplat/tiling.py:34-43), clipped to the grid.  The rectangle is
                    // band-agnostic (binning clips it to a tile-row band), so one K1 serves every band choice.
                    double fx0 = floor((mx - rad) / TILE), fx1 = floor((mx + rad) / TILE);
                    double fy0 = floor((my - rad) / TILE), fy1 = floor((my + rad) / TILE);
                    if (a.coverage != TCGS_COVER_SQUARE) {
                        // opt-in, not the reference's coverage: keep only tiles the
                        // alpha >= 1/255 ellipse q <= 2 ln(255 o) can reach -- its bounding box, with margins
                        // above every rounding of K7's exponent -- inside the reference's square (the exact
                        // mode then keeps only the tiles the ellipse touches, in binning).  Splats it drops have no live fragment, so
                        // the image is unchanged; N and f_cull shrink.
                        const double Qc = 2.0 * (log(ld(opac, l)) + 5.541263545158426) + COVER_Q_MARGIN;
                        if (Qc > 0.0) {
                            const double ex = sqrt(Qc * sa) + COVER_PX_MARGIN, ey = sqrt(Qc * sc) + COVER_PX_MARGIN;
                            fx0 = fmax(fx0, floor((mx - ex) / TILE));
                            fx1 = fmin(fx1, floor((mx + ex) / TILE));
                            fy0 = fmax(fy0, floor((my - ey) / TILE));
                            fy1 = fmin(fy1, floor((my + ey) / TILE));
                        } else {
                            fx1 = fx0 - 1.0;  // opacity < 1/255: no fragment anywhere can pass EarlyCull
                        }
                    }
                    fx0 = fmax(fx0, 0.0);
                    fy0 = fmax(fy0, 0.0);
                    fx1 = fmin(fx1, (double)(a.tiles_x - 1));
                    fy1 = fmin(fy1, (double)(a.tiles_y - 1));
                    if (fx0 <= fx1 && fy0 <= fy1) {
                        const int x0 = (int)fx0, x1 = (int)fx1, y0 = (int)fy0, y1 = (int)fy1;
                        touched = (uint32_t)((x1 - x0 + 1) * (y1 - y0 + 1));
                        rect = make_short4((short)x0, (short)y0, (short)x1, (short)y1);
                        key = (unsigned long long)__double_as_longlong(tz);  // tz > 0: bit order == value order
                        Rec rc;
                        rc.mx = (float)mx;
                        rc.mx_lo = (float)(mx - (double)rc.mx);
                        rc.my = (float)my;
                        rc.my_lo = (float)(my - (double)rc.my);
                        rc.s11 = (float)s11;
                        rc.s12 = (float)s12;
                        rc.s22 = (float)s22;
                        const double o = ld(opac, l);
                        rc.ln_o = logf((float)o);
                        rc.opacity = (float)o;
                        float col[3] = {0.0f, 0.0f, 0.0f};
                        wait_bar(1);  // features staged (usually long done: they streamed in during the projection)
                        if (a.defer_colour) {
                            // colour_kernel fills it after the band partition
                        } else if (a.sh_degree < 0) {
                            col[0] = (float)ld(feats, 3 * l);
                            col[1] = (float)ld(feats, 3 * l + 1);
                            col[2] = (float)ld(feats, 3 * l + 2);
                        } else {
                            const int K = (a.sh_degree + 1) * (a.sh_degree + 1);
                            const double dx = m0 - a.campos[0], dy = m1 - a.campos[1], dz = m2 - a.campos[2];
                            const double nn = sqrt(dx * dx + dy * dy + dz * dz);
                            sh_color(feats + (size_t)l * K * 3, a.sh_degree, dx / nn, dy / nn, dz / nn, col);
                        }
                        rc.r = col[0];
                        rc.g = col[1];
                        rc.b = col[2];
                        pdl_wait();
                        a.rec[i] = rc;
                    }
                }
            }
            pdl_wait();
            a.rect[i] = rect;
            a.keys[i] = key;
        }
        // warp-aggregated counters
        pdl_wait();
        const unsigned full = 0xffffffffu;
        const unsigned n_drop = __popc(__ballot_sync(full, dropped));
        const unsigned n_vis = __popc(__ballot_sync(full, touched > 0));
        unsigned long long kmin = touched > 0 ? key : ~0ull, kmax = touched > 0 ? key : 0ull;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long omin = __shfl_xor_sync(full, kmin, o), omax = __shfl_xor_sync(full, kmax, o);
            kmin = omin < kmin ? omin : kmin;
            kmax = omax > kmax ? omax : kmax;
        }
        if ((threadIdx.x & 31) == 0) {
            if (n_drop) atomicAdd(&a.ctr->dropped, (unsigned long long)n_drop);
            if (n_vis) {
                atomicAdd(&a.ctr->n_visible, (unsigned long long)n_vis);
                atomicMin(&a.ctr->key_min, kmin);
                atomicMax(&a.ctr->key_max, kmax);
            }
        }
    }  // views
    wait_bar(1);  // no CTA may retire with a bulk copy into its shared memory still in flight
}


template <typename T, int NV>
cudaError_t launch_k1(const PreViews<NV> &pv, const tcgs_scene &scene, int F, int nt, cudaStream_t st) {
    size_t smem = 0;
    for (int per : {3, 3, 4, 1, F}) smem += ((size_t)per * nt * sizeof(T) + 15) / 16 * 16;
    static size_t configured_dev[TCGS_MAX_DEVICES] = {};
    size_t &configured = configured_dev[current_device()];
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(preprocess_kernel<T, NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    const unsigned blocks = (unsigned)((scene.P + nt - 1) / nt);
    return launch_k(preprocess_kernel<T, NV>, blocks, nt, smem, st, pv, (const T *)scene.means,
                    (const T *)scene.scales, (const T *)scene.rotations, (const T *)scene.opacities,
                    (const T *)scene.features);
}

PreArgs view_args(const tcgs_scene &scene, const tcgs_camera &cam, const Band &band, int debug, int coverage,
                  void *ws, const Layout &L) {
    PreArgs a;
    a.cam = cam;
    const double *V = cam.view;
    // camera centre -R^T t (row-major view)
    for (int k = 0; k < 3; k++) a.campos[k] = -(V[0 * 4 + k] * V[3] + V[1 * 4 + k] * V[7] + V[2 * 4 + k] * V[11]);
    a.P = scene.P;
    a.sh_degree = scene.sh_degree;
    a.tiles_x = band.tiles_x;
    a.tiles_y = band.tiles_y;
    a.band_y0 = band.y0;
    a.band_y1 = band.y1;
    a.debug = debug;
    a.coverage = coverage;
    a.defer_colour = 0;
    a.rec = at<Rec>(ws, L.rec);
    a.rect = at<short4>(ws, L.rect);
    a.keys = at<unsigned long long>(ws, L.key_src);
    a.radius = at<int32_t>(ws, L.radius);
    a.dbg_conic = at<double>(ws, L.dbg_conic);
    a.dbg_depth = at<double>(ws, L.dbg_depth);
    a.dbg_mean2d = at<double>(ws, L.dbg_mean2d);
    a.ctr = at<DevCounters>(ws, L.counters);
    return a;
}

template <int NV>
cudaError_t launch_views(const PreViews<NV> &pv, const tcgs_scene &scene, cudaStream_t st) {
    if (scene.P <= 0) return cudaSuccess;
    const int F = pv.v[0].defer_colour ? 0 : (scene.sh_degree < 0 ? 3 : 3 * (scene.sh_degree + 1) * (scene.sh_degree + 1));
    if (scene.dtype == TCGS_F64) return launch_k1<double, NV>(pv, scene, F, 128, st);
    return launch_k1<float, NV>(pv, scene, F, TCGS_K1_THREADS, st);
}

// Deferred colour (tile bands): the SH colour of every Gaussian whose tile rectangle meets the rank's tile rows
// [band_y0, band_y1), straight from global memory -- one 192-B SH3 read per such Gaussian instead of the
// CTA-wide staging of all of them -- with exactly K1's arithmetic (same function, same translation unit).
struct ColourArgs {
    double campos[3];
    int64_t P;
    int sh_degree, band_y0, band_y1;
    const short4 *rect;
    Rec *rec;
};

template <typename T>
__global__ void __launch_bounds__(256) colour_kernel(ColourArgs c, const T *__restrict__ g_means,
                                                     const T *__restrict__ g_feats) {
    pdl_wait();
    pdl_launch();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= c.P) return;
    const short4 r = c.rect[i];
    if (r.x > r.z || r.w < c.band_y0 || r.y >= c.band_y1) return;  // no tile, or none in the band
    float col[3];
    if (c.sh_degree < 0) {
        col[0] = (float)g_feats[3 * i];
        col[1] = (float)g_feats[3 * i + 1];
        col[2] = (float)g_feats[3 * i + 2];
    } else {
        const int K = (c.sh_degree + 1) * (c.sh_degree + 1);
        const double m0 = g_means[3 * i], m1 = g_means[3 * i + 1], m2 = g_means[3 * i + 2];
        const double dx = m0 - c.campos[0], dy = m1 - c.campos[1], dz = m2 - c.campos[2];
        const double nn = sqrt(dx * dx + dy * dy + dz * dz);
        sh_color(g_feats + (size_t)i * K * 3, c.sh_degree, dx / nn, dy / nn, dz / nn, col);
    }
    Rec &rr = c.rec[i];
    rr.r = col[0];
    rr.g = col[1];
    rr.b = col[2];
}

}  // namespace

cudaError_t launch_colour(const tcgs_scene &scene, const tcgs_camera &cam, const Band &band, void *ws,
                          const Layout &L, cudaStream_t st) {
    if (scene.P <= 0) return cudaSuccess;
    const PreArgs a = view_args(scene, cam, band, 0, 0, ws, L);
    ColourArgs c;
    for (int k = 0; k < 3; k++) c.campos[k] = a.campos[k];
    c.P = scene.P;
    c.sh_degree = scene.sh_degree;
    c.band_y0 = band.y0;
    c.band_y1 = band.y1;
    c.rect = a.rect;
    c.rec = a.rec;
    const unsigned blocks = (unsigned)((scene.P + 255) / 256);
    if (scene.dtype == TCGS_F64)
        return launch_k(colour_kernel<double>, blocks, 256, 0, st, c, (const double *)scene.means,
                        (const double *)scene.features);
    return launch_k(colour_kernel<float>, blocks, 256, 0, st, c, (const float *)scene.means,
                    (const float *)scene.features);
}

cudaError_t launch_preprocess(const tcgs_scene &scene, const tcgs_camera &cam, const Band &band, int debug,
                              int coverage, int defer_colour, void *ws, const Layout &L, cudaStream_t st) {
    PreViews<1> pv;
    pv.v[0] = view_args(scene, cam, band, debug, coverage, ws, L);
    pv.v[0].defer_colour = defer_colour;
    pv.n = 1;
    return launch_views(pv, scene, st);
}

cudaError_t launch_preprocess_views(const tcgs_scene &scene, const tcgs_camera *cams, const Band *bands, int n_views,
                                    int debug, int coverage, int defer_colour, void *const *ws, const Layout *L,
                                    cudaStream_t st) {
    PreViews<TCGS_MAX_VIEWS_PER_PASS> pv;
    for (int v = 0; v < n_views; v++) {
        pv.v[v] = view_args(scene, cams[v], bands[v], debug, coverage, ws[v], L[v]);
        pv.v[v].defer_colour = defer_colour;
    }
    pv.n = n_views;
    return launch_views(pv, scene, st);
}

}  // namespace tcgs
