// render.cu -- K7: tensor-core alpha (Frag2Mat + G2L + EarlyCull) and conditional
// blending for 16x16 tiles (sm_100a: tcgen05.mma, TMEM, mbarrier pipelines).
//
// Replaces the tile loop of tilesplat.raster.render and blend_tile
// (/root/reference/pkg/src/tilesplat/raster.py:110-146,177-193) with the
// Frag2Mat evaluator (src/tilesplat/tensor_path.py:25-163):
//
//   beta[p, j] = U[p, :] . V[j, :]       (256 pixels x 32 Gaussians per batch)
//
// U holds each pixel's tile-local monomials [1, ux, uy, ux^2, ux*uy, uy^2]
// (G2L: ux, uy in [-8, 7] about the tile centre, src/tilesplat/tensor_path.py:
// 21-22,92-100) -- exact in fp16 and the same for every tile, so it is built
// once per CTA.  V holds each Gaussian's coefficients (gaussian_vector,
// tensor_path.py:25-40) pre-scaled by log2(e) and split into fp16 hi + lo
// parts so the K = 16 of tcgen05.mma.kind::f16 carries ~22 significant bits
// (TCGS_ALPHA_TC_K8 keeps the paper's length-8 fp16 vector for ablation).
//
// CTA = 8 consumer warps (one pixel per thread; warp w owns an 8x4 pixel block
// = TMEM lanes 32(w%4).. of pixel half w/4) + 2 producer warps; 3 CTAs per SM.
//   producers: walk the CTA's static tile stream (blockIdx.x, +gridDim.x, ...) in
//     32-entry chunks, alternating chunks and handing the compaction state over
//     with a token mbarrier; gather each entry's projected record, drop Gaussians
//     whose EarlyCull test fails at every pixel of the tile (exact box minimum of
//     the quadratic form -- culls the reference would count, and they are
//     counted), compact the live ones 32 at a time into a shared-memory stage
//     (fp16 hi/lo V rows, colours, dead-before counts; unused rows of a partial
//     stage get beta = -65504), and issue two M=128 x N=32 x K=16 MMAs per stage
//     into a TMEM accumulator buffer (commit -> mbarrier);
//   consumers: tcgen05.ld their 32 betas; per column, a pixel passes EarlyCull
//     iff beta' >= thr (thr = -log2 255 while live, +inf once done) and a warp
//     vote skips columns no pixel passes (uniform branch, 3 instructions); in a
//     taken column: alpha = ex2(beta'), the termination test before compositing
//     (T - alpha T < 1e-4, src/tilesplat/raster.py:136-145), C += alpha T c,
//     T -= alpha T.  A warp whose pixels have all terminated stops working; when
//     all 8 have, the producers retire the tile.
// Stages (4) and TMEM buffers (2) are ring buffers: a consumer waits on one mbarrier per stage (mma_done: the
// producer's arrival with the stage rows + the MMA commit) and releases the stage with one arrival (released,
// which also frees the TMEM buffer NB stages later), so gathers, MMAs and blending overlap.
#include "tcgs_internal.cuh"

namespace tcgs {

namespace {

constexpr float LOG2E = 1.4426950408889634f;
constexpr float CUT_LOG2 = -7.994353436858858f;  // -log2(255): beta' < CUT culls (tensor_path.py:79-81)
constexpr float LN255 = 5.541263545158426f;
constexpr float TERM_T = 0.0001f;                // src/tilesplat/raster.py:16
// also caps residency at K7_CTAS_PER_SM CTAs/SM (TMEM: K7_CTAS_PER_SM x K7_TMEM_COLS <= 512 columns)
constexpr int K7_SMEM_BYTES = (K7_CTAS_PER_SM >= 4 ? 54 : 72) * 1024;
constexpr int S = K7_STAGES;
constexpr int NB = K7_TMEM_BUFS;

struct RenderArgs {
    const Rec *rec;
    const uint32_t *ids0;
    const uint32_t *ids1;
    const uint32_t *ids_override;
    const uint2 *ranges;
    DevCounters *ctr;
    int tiles_x, band_y0, n_tiles, width, height;
    float *rgb;
    float *T;
    int32_t *n_contrib;
    const uint32_t *cid, *cdb, *ccount;  // compacted live lists (binning wrote them when ctr->compact)
    float *dump_beta;      // debug (FL_DUMP): beta' of every evaluated (list entry, pixel), [N][256]
    uint8_t *dump_class;   // debug (FL_DUMP): 1 cull, 2 blend, 3 terminate; 0 = not evaluated, [N][256]
};

// K7 variants (template flags): FL_ECOFF = EarlyCull off -- alpha = 2^beta' for every active fragment and the
// cull on alpha < 1/255 afterwards (the reference's alpha_reference order, src/tilesplat/raster.py:86-94 /
// tensor_path.py:155-160), no dead-Gaussian box test in the producer; FL_DUMP = debug dump of beta' and the
// per-fragment classification (the a19 tolerance oracle, tests/test_gpu_beta.py).
#ifndef TCGS_K7_EX2EARLY
#define TCGS_K7_EX2EARLY 0
#endif
constexpr bool EX2EARLY = TCGS_K7_EX2EARLY != 0;
#ifndef TCGS_K7_RECBUF
#define TCGS_K7_RECBUF 1  // producers prefetch the next chunk's records into shared memory (cp.async, no registers)
#endif
constexpr bool K7_RECBUF = TCGS_K7_RECBUF != 0;
#ifndef TCGS_K7_LOOKAHEAD
#define TCGS_K7_LOOKAHEAD 1  // producer chunks of cursor / list ids prefetched ahead of the one being gathered
#endif
// ring slots: 2 = records one owned chunk ahead; 3 (with TCGS_K7_LOOKAHEAD=2) = two chunks ahead
constexpr int K7_RECDEPTH = (K7_RECBUF && TCGS_K7_LOOKAHEAD >= 2) ? 3 : 2;
constexpr int FL_ECOFF = 1;
constexpr int FL_DUMP = 2;
constexpr float ALPHA_CUT = 1.0f / 255.0f;  // src/tilesplat/raster.py:15

// A pixel that terminates at stage column j gets the pass threshold term_code(j) = 2^100 (1 + j/64): no beta can
// reach it (|beta| <= 16 * 65504^2 for finite fp16 operands), so one FSEL both retires the pixel and records j.
constexpr float TERM_CODE0 = 1.2676506002282294e30f;  // 2^100
__device__ __forceinline__ constexpr float term_code(int j) { return TERM_CODE0 * (1.0f + (float)j / 64.0f); }
__device__ __forceinline__ int term_col(float code) { return (int)((code * 7.888609052210118e-31f - 1.0f) * 64.0f); }

struct StageMeta {
    int tile;        // -1: no more tiles
    int seq;         // CTA-local tile sequence number
    int n_live;      // live Gaussians in this stage (<= K7_BATCH)
    int last;        // last stage of the tile's list
    uint32_t dead_total;  // (last stage) dead Gaussians in the whole list
    uint32_t n_total;     // list length of the tile
    int pad[2];
};

template <bool GL>  // GL: the global-coordinate ablation's per-stage A operands
struct __align__(1024) K7SmemT {
    __half U[2][128 * 16];              // A operands: pixel halves, K-major no-swizzle core matrices
    __half V[S][K7_BATCH * 16];         // B operands, one per stage
    float4 vf[S][K7_BATCH][2];          // FFMA mode: fp32 coefficients
    float4 col[S][K7_BATCH];            // colours
    uint32_t dead_before[S][K7_BATCH];  // dead Gaussians before each live one (list order)
    uint32_t pos[S][K7_BATCH];          // FL_DUMP: tile-list index of each live row
    __half Ug[GL ? S : 1][2][128 * 16];  // TC_K8_GLOBAL: per-stage A operands (global pixel coordinates)
    StageMeta meta[S];
    // full: stage data ready (FFMA mode; with tensor cores mma_done[b] also carries the producer's arrival, so
    // consumers wait on one barrier); released: every consumer warp is done with a stage (its shared-memory
    // rows, and -- NB stages later -- its TMEM buffer)
    unsigned long long full[S], released[S], mma_done[NB], tok[K7_PRODUCERS];
    uint32_t tmem_base;
    int retire[8];
    int c_fill, c_k, c_open;  // compaction state: touched only by the producer holding the token
    unsigned long long tslot[16];  // dynamic tile stream: (seq << 32) | tile, shared by the producers
    uint32_t c_dead;
    unsigned long long red[K7_CONSUMER_WARPS][4];
    Rec rbuf[K7_RECBUF ? K7_PRODUCERS : 1][K7_RECDEPTH][32];  // TCGS_K7_RECBUF: producer record ring (cp.async)
};

// Element offset (in halves) of (row, k) in a K-major, no-swizzle UMMA operand of 16 K-columns:
// 8x8 core matrices (8 rows x 16 B); the two K chunks sit LBO = 128 B apart, 8-row groups SBO = 256 B apart.
__device__ __forceinline__ int kmaj_off(int row, int k) {
    return (row >> 3) * 128 + (k >> 3) * 64 + (row & 7) * 8 + (k & 7);
}

__device__ __forceinline__ uint64_t umma_desc(const void *smem) {
    const uint32_t a = smem_u32(smem);
    return (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
           (1ull << 46);  // version 1 (sm_100), base offset 0, SWIZZLE_NONE
}

// kind::f16 instruction descriptor: D f32, A/B f16, K-major both, N = K7_BATCH, M = 128.
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(K7_BATCH >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void mbar_init(unsigned long long *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
#ifndef TCGS_K7_WAIT
#define TCGS_K7_WAIT 0
#endif
#ifdef TCGS_K7_TIMING  // experiment builds: cycles spent waiting, per barrier kind (tcgs_k7_timing reads them)
__device__ unsigned long long g_k7_wait[8];
#define K7_TWAIT(kind, call)                                        \
    do {                                                            \
        const long long t0_ = clock64();                            \
        call;                                                       \
        if ((threadIdx.x & 31) == 0) atomicAdd(&g_k7_wait[kind], (unsigned long long)(clock64() - t0_)); \
    } while (0)
#else
#define K7_TWAIT(kind, call) call
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
#if TCGS_K7_WAIT == 0
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680u)  // suspend-time hint: sleep until the phase flips instead of spinning
        : "memory");
#else
    // experiment: try_wait without a hint, then back off with nanosleep (TCGS_K7_WAIT ns) so a waiting warp
    // leaves its issue slots to the working ones
    uint32_t ok;
    for (;;) {
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n"
            "}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) break;
        __nanosleep(TCGS_K7_WAIT);
    }
#endif
}
__device__ __forceinline__ void mbar_arrive_n(unsigned long long *bar, uint32_t n) {
    asm volatile(
        "{\n"
        ".reg .b64 st;\n"
        "mbarrier.arrive.shared::cta.b64 st, [%0], %1;\n"
        "}\n" ::"r"(smem_u32(bar)), "r"(n)
        : "memory");
}
#ifndef TCGS_K7_PRODWAIT
#define TCGS_K7_PRODWAIT 0  // producer waits: 0 = suspend hint (as the consumers), N > 0 = try_wait + N ns backoff
#endif
// Producers run ahead of the consumers and mostly wait for a stage to be released: optionally back off with a
// plain nanosleep so the waiting warps leave issue slots to the consumers.
__device__ __forceinline__ void mbar_wait_prod(unsigned long long *bar, uint32_t parity) {
#if TCGS_K7_PRODWAIT == 0
    mbar_wait(bar, parity);
#else
    uint32_t ok;
    for (;;) {
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n"
            "}\n"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) break;
        __nanosleep(TCGS_K7_PRODWAIT);
    }
#endif
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
    asm volatile(
        "{\n"
        ".reg .b64 st;\n"
        "mbarrier.arrive.shared::cta.b64 st, [%0];\n"
        "}\n" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem, bool pred) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %2, 0;\n"
        "@p cp.async.cg.shared.global [%0], [%1], 16;\n"
        "}\n" ::"r"(smem_u32(smem)),
        "l"(gmem), "r"((int)pred)
        : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(0u));
}
__device__ __forceinline__ void mma_commit(unsigned long long *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
template <int G>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&v)[G]);
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t taddr, uint32_t (&v)[16]) {
    tmem_ld16(taddr, v);
}
template <>
__device__ __forceinline__ void tmem_ld<8>(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Gaussian coefficients for one tile (gaussian_vector, src/tilesplat/tensor_path.py:25-40) relative to the
// tile centre (G2L), scaled by log2 e.  Returns false ("dead") when EarlyCull fails at every point of the
// tile's pixel box [-8,7]^2: the minimum of the convex quadratic q(d - u) over the box is exact (interior
// minimiser or the clamped minimiser on one of the four edges), and the test keeps a 0.01 margin on
// beta, so every fragment of a dead Gaussian in this tile is a cull in exact arithmetic too.
// BOXCULL = false (EarlyCull off, global coordinates): every Gaussian of the list is live.
template <bool BOXCULL>
__device__ __forceinline__ bool gaussian_coeffs(const Rec &r, float ox, float oy, float v[6]) {
    // mean - centre in fp32: hi - centre is exact for frame coordinates (both on the hi value's grid),
    // then one rounding with the lo part -- the float64 difference to within an ulp of dx, with no FP64 op
    const float dx = __fadd_rn(__fsub_rn(r.mx, ox), r.mx_lo), dy = __fadd_rn(__fsub_rn(r.my, oy), r.my_lo);
    const float s11 = r.s11, s12 = r.s12, s22 = r.s22;
    const float q = s11 * dx * dx + 2.0f * s12 * dx * dy + s22 * dy * dy;
    const bool outside = !(dx >= -8.0f && dx <= 7.0f && dy >= -8.0f && dy <= 7.0f);
    if (BOXCULL && outside && s11 > 1e-30f && s22 > 1e-30f) {
        // (the minimiser only needs to be accurate to first order: q is flat there, and the test keeps a margin;
        // the normal-range guard above lets the reciprocal skip denormal handling)
        const float r11 = s12 * rcp_approx(s11), r22 = s12 * rcp_approx(s22);
        // The unconstrained minimiser d lies outside the box, so the box minimum lies on a face the segment
        // from any box point to d crosses: the face x = clamp(dx) if dx is outside [-8, 7], the face
        // y = clamp(dy) if dy is.  Evaluating the two clamped lines always is safe: a line through the box
        // interior only gives values >= the box minimum.
        float qmin;
        {  // line ux = clamp(dx)
            const float a = fminf(fmaxf(dx, -8.0f), 7.0f);
            const float ex = dx - a;
            const float uy = fminf(fmaxf(dy + r22 * ex, -8.0f), 7.0f);
            const float ey = dy - uy;
            qmin = s11 * ex * ex + 2.0f * s12 * ex * ey + s22 * ey * ey;
        }
        {  // line uy = clamp(dy)
            const float a = fminf(fmaxf(dy, -8.0f), 7.0f);
            const float ey = dy - a;
            const float ux = fminf(fmaxf(dx + r11 * ey, -8.0f), 7.0f);
            const float ex = dx - ux;
            qmin = fminf(qmin, s11 * ex * ex + 2.0f * s12 * ex * ey + s22 * ey * ey);
        }
        if (r.ln_o - 0.5f * qmin < -LN255 - 0.01f) return false;
    }
    v[0] = (r.ln_o - 0.5f * q) * LOG2E;
    v[1] = (s11 * dx + s12 * dy) * LOG2E;
    v[2] = (s12 * dx + s22 * dy) * LOG2E;
    v[3] = -0.5f * s11 * LOG2E;
    v[4] = -s12 * LOG2E;
    v[5] = -0.5f * s22 * LOG2E;
    return true;
}


__device__ __forceinline__ __half h16(float x) { return __float2half_rn(x); }
__device__ __forceinline__ float f32(__half x) { return __half2float(x); }

// One B-operand row (16 fp16, as two uint4) for MODE: hi/lo split (0) or the paper's K8 vector (1).
// U row: [1, 1, 1, ux, uy, ux^2, ux uy, uy^2, ux, uy, ux^2, ux uy, uy^2, 1, 0, 0]
#ifndef TCGS_K7_VROW2
#define TCGS_K7_VROW2 0
#endif
template <int MODE>
__device__ __forceinline__ void make_vrow(const float v[6], uint4 &lo8, uint4 &hi8) {
    __align__(16) __half e[16];
    if (MODE == TCGS_ALPHA_TC_K8 || MODE == TCGS_ALPHA_TC_K8_GLOBAL) {  // [v0/3, v0/3, v0/3, v1..v5] in fp16, the rest zero
        const __half third = h16(v[0] / 3.0f);
        e[0] = third;
        e[1] = third;
        e[2] = third;
#pragma unroll
        for (int i = 1; i <= 5; i++) e[2 + i] = h16(v[i]);
#pragma unroll
        for (int k = 8; k < 16; k++) e[k] = h16(0.0f);
    } else if (TCGS_K7_VROW2) {  // the same hi/lo vector with paired conversions (cvt.rn.f16x2.f32)
        const __half2 h12 = __floats2half2_rn(v[1], v[2]), h34 = __floats2half2_rn(v[3], v[4]);
        const __half2 h50 = __floats2half2_rn(v[5], v[0]);
        const float2 f12 = __half22float2(h12), f34 = __half22float2(h34), f50 = __half22float2(h50);
        const __half2 l12 = __floats2half2_rn(v[1] - f12.x, v[2] - f12.y);
        const __half2 l34 = __floats2half2_rn(v[3] - f34.x, v[4] - f34.y);
        const float r1 = v[0] - f50.y;
        const __half2 l5b = __floats2half2_rn(v[5] - f50.x, r1);  // (lo of v5, second piece of v0)
        const float r2 = r1 - __high2float(l5b);
        const __half c = h16(r2);
        const __half d = h16(r2 - f32(c));
        const __half2 w[8] = {__halves2half2(__high2half(h50), __high2half(l5b)), __halves2half2(c, __low2half(h12)),
                              __halves2half2(__high2half(h12), __low2half(h34)),
                              __halves2half2(__high2half(h34), __low2half(h50)), l12, l34,
                              __halves2half2(__low2half(l5b), d), __floats2half2_rn(0.0f, 0.0f)};
        lo8 = make_uint4(*reinterpret_cast<const uint32_t *>(&w[0]), *reinterpret_cast<const uint32_t *>(&w[1]),
                         *reinterpret_cast<const uint32_t *>(&w[2]), *reinterpret_cast<const uint32_t *>(&w[3]));
        hi8 = make_uint4(*reinterpret_cast<const uint32_t *>(&w[4]), *reinterpret_cast<const uint32_t *>(&w[5]),
                         *reinterpret_cast<const uint32_t *>(&w[6]), *reinterpret_cast<const uint32_t *>(&w[7]));
        return;
    } else {  // hi/lo: v0 = a + b + c + d (four fp16 pieces), v1..v5 = hi + lo
        const __half a = h16(v[0]);
        const float r1 = v[0] - f32(a);
        const __half b = h16(r1);
        const float r2 = r1 - f32(b);
        const __half c = h16(r2);
        const __half d = h16(r2 - f32(c));
        e[0] = a;
        e[1] = b;
        e[2] = c;
#pragma unroll
        for (int i = 1; i <= 5; i++) {
            const __half hi = h16(v[i]);
            e[2 + i] = hi;
            e[7 + i] = h16(v[i] - f32(hi));
        }
        e[13] = d;
        e[14] = h16(0.0f);
        e[15] = h16(0.0f);
    }
    lo8 = reinterpret_cast<const uint4 *>(e)[0];
    hi8 = reinterpret_cast<const uint4 *>(e)[1];
}

// ------------------------------------------------------------------------------------------ producers
// The CTA's tile stream starts at tile blockIdx.x and continues from a global queue (dynamic schedule) or with
// blockIdx.x + gridDim.x, ... (static schedule); each tile contributes
// max(1, ceil(n/32)) chunks of 32 list entries, and one "end" chunk closes the stream.  Producer warp p
// owns chunks p, p + NP, ...: it gathers and evaluates its chunk in parallel with the other producer,
// then waits for the compaction token, places its live rows into the current stage, emits full stages
// (issuing their MMAs) and passes the token on.
// The heavy build (TCGS_K7_COMPACT, a third compilation of this file) reads the compacted live lists when binning
// wrote them (ctr->compact); the other builds never see them (see producer_heavy in tcgs_internal.cuh).
#ifdef TCGS_K7_COMPACT
constexpr bool K7_COMPACT = true;
#else
constexpr bool K7_COMPACT = false;
#endif

struct Cursor {
    int tile, seq, c, chunks, n;
    int nfull;  // the tile's list length (n: the entries walked -- the live ones when the lists are compacted)
    uint32_t beg;
    float ox, oy;     // tile centre (16tx+8, 16ty+8), tensor_path.py:21-22
    bool prev_valid;  // the previous tile of the stream was a real one (its end chunk closes the stream)
};

constexpr uint32_t TSLOT_CLAIMED = 0xFFFFFFFFu;

// Tile of the CTA's seq-th stream position (seq >= 1), fetched from the global queue by whichever producer needs
// it first and shared through a tagged shared-memory slot: both producers walk the same stream.  Warp-uniform.
template <class SM>
__device__ __forceinline__ int seq_tile(SM &sm, const RenderArgs &a, int seq) {
    int t = 0;
    if ((threadIdx.x & 31) == 0) {
        unsigned long long *slot = &sm.tslot[seq & 15];
        const unsigned long long tag = (unsigned long long)(uint32_t)seq << 32;
        for (;;) {
            const unsigned long long v = *reinterpret_cast<volatile unsigned long long *>(slot);
            if ((uint32_t)(v >> 32) == (uint32_t)seq) {
                if ((uint32_t)v != TSLOT_CLAIMED) {
                    t = (int)(uint32_t)v;
                    break;
                }
                __nanosleep(32);  // the other producer is fetching it
                continue;
            }
            if (atomicCAS(slot, v, tag | TSLOT_CLAIMED) == v) {
                t = (int)gridDim.x + (int)atomicAdd(&a.ctr->tile_queue, 1u);
                atomicExch(slot, tag | (uint32_t)t);
                break;
            }
        }
    }
    return __shfl_sync(0xffffffffu, t, 0);
}

__device__ __forceinline__ void cursor_tile(Cursor &k, const RenderArgs &a) {
    k.c = 0;
    if (k.tile < a.n_tiles) {
        const int tx = k.tile % a.tiles_x, ty = a.band_y0 + k.tile / a.tiles_x;
        k.ox = (float)(tx * TILE + 8);
        k.oy = (float)(ty * TILE + 8);
        const uint2 rg = a.ranges[k.tile];
        k.beg = rg.x;
        k.nfull = (int)(rg.y - rg.x);
        k.n = (K7_COMPACT && a.ctr->compact) ? (int)a.ccount[k.tile] : k.nfull;  // compacted: the live entries
        k.chunks = k.n > 0 ? (k.n + 31) / 32 : 1;
    } else {
        k.beg = 0;
        k.n = k.nfull = 0;
        k.chunks = 1;
    }
}

// DYN (TCGS_SCHEDULE_DYNAMIC): tiles after the CTA's first come from a global queue, which balances the tail of
// a lone frame; static (tiles blockIdx.x, +gridDim.x, ...) leaves a staggered tail that other streams' kernels fill
// when several frames share the GPU.
template <bool DYN, class SM>
__device__ __forceinline__ void cursor_next(Cursor &k, const RenderArgs &a, SM &sm) {
    if (++k.c >= k.chunks) {
        k.prev_valid = k.tile < a.n_tiles;
        k.seq++;
        k.tile = DYN ? seq_tile(sm, a, k.seq) : k.tile + (int)gridDim.x;
        cursor_tile(k, a);
    }
}

// Global-coordinate A operand of one stage (TC_K8_GLOBAL, the paper's Frag2Mat-without-G2L ablation): pixel
// rows [1, 1, 1, x, y, x^2, xy, y^2, 0 ...] in fp16 (x^2 overflows for x >= 256, as tensor_path.py:92-100 with
// coords="global" does under the fp16 model), in the consumer's TMEM-lane order.
__device__ __forceinline__ void write_global_u(__half (*ug)[128 * 16], int tile, const RenderArgs &a, int lane) {
    const int tx = tile % a.tiles_x, ty = a.band_y0 + tile / a.tiles_x;
#pragma unroll 1
    for (int q = 0; q < 8; q++) {
        const int row = q * 32 + lane;  // 0..255: half row >> 7, TMEM lane row & 127
        const int h = row >> 7, r = row & 127;
        const int w = (r >> 5) + 4 * h;  // consumer warp owning the lane
        const float x = (float)(tx * TILE + 8 * (w & 1) + (lane & 7));
        const float y = (float)(ty * TILE + 4 * ((w >> 1) & 3) + (lane >> 3));
        __align__(16) __half e[16];
        e[0] = e[1] = e[2] = __float2half_rn(1.0f);
        e[3] = __float2half_rn(x);
        e[4] = __float2half_rn(y);
        e[5] = __float2half_rn(x * x);
        e[6] = __float2half_rn(x * y);
        e[7] = __float2half_rn(y * y);
#pragma unroll
        for (int k = 8; k < 16; k++) e[k] = __float2half_rn(0.0f);
        *reinterpret_cast<uint4 *>(ug[h] + kmaj_off(r, 0)) = reinterpret_cast<const uint4 *>(e)[0];
        *reinterpret_cast<uint4 *>(ug[h] + kmaj_off(r, 8)) = reinterpret_cast<const uint4 *>(e)[1];
    }
}

template <int MODE, bool DYN, int FL>
__device__ void producer(K7SmemT<MODE == TCGS_ALPHA_TC_K8_GLOBAL> &sm, const RenderArgs &a, const uint32_t *ids, uint32_t tmem, int p) {
    constexpr bool TC = MODE != TCGS_ALPHA_FFMA;
    constexpr bool GLOBAL = MODE == TCGS_ALPHA_TC_K8_GLOBAL;
    constexpr bool BOXCULL = !(FL & FL_ECOFF) && !GLOBAL;
    constexpr bool DUMP = (FL & FL_DUMP) != 0;
    constexpr int NP = K7_PRODUCERS;
    const int lane = threadIdx.x & 31;
    const unsigned FULL = 0xffffffffu, lt = lanemask_lt();
    const bool cmp = K7_COMPACT && a.ctr->compact != 0;  // walking the compacted live lists
    Cursor cur;
    cur.tile = blockIdx.x;
    cur.seq = 0;
    cur.prev_valid = true;
    cursor_tile(cur, a);
    for (int i = 0; i < p; i++) cursor_next<DYN>(cur, a, sm);
    Cursor nxt = cur;
    for (int i = 0; i < NP; i++) cursor_next<DYN>(nxt, a, sm);
    auto list_id = [&](const Cursor &k) -> uint32_t {
        const int i = k.c * 32 + lane;
        return i < k.n ? ids[k.beg + i] : 0u;
    };
    // gather pipeline: the records of the chunk being evaluated, and the ids of the next owned chunk.  With
    // K7_RECBUF the next chunk's records travel by cp.async into this warp's shared-memory ring (slot m & 1)
    // instead of registers, and are read back (LDS) when the chunk is evaluated.
    Rec rc;
    auto gather = [&](const Cursor &k, uint32_t id, int slot, Rec &r) {
        const bool v = k.c * 32 + lane < k.n;
        if (K7_RECBUF) {
            const Rec *src = a.rec + id;
            Rec *dst = &sm.rbuf[K7_RECBUF ? p : 0][slot][lane];
#pragma unroll
            for (int q = 0; q < 3; q++) cp_async16(reinterpret_cast<uint4 *>(dst) + q,
                                                   reinterpret_cast<const uint4 *>(src) + q, v);
            cp_async_commit();
        } else if (v) {
            r = a.rec[id];
        }
    };
    gather(cur, list_id(cur), 0, rc);
#if TCGS_K7_LOOKAHEAD >= 2
    if (K7_RECDEPTH == 3) {  // the chunk after this one too (the loop issues two chunks ahead)
        Rec r1;
        gather(nxt, list_id(nxt), 1, r1);
    }
#endif
    uint32_t id_nxt = list_id(nxt);
#if TCGS_K7_LOOKAHEAD >= 2
    // one more owned chunk of cursor and ids in flight: the tile-queue fetch and the range / id loads of a tile
    // transition get two producer iterations of latency budget
    Cursor nxa = nxt;
    for (int i = 0; i < NP; i++) cursor_next<DYN>(nxa, a, sm);
    uint32_t id_nxa = list_id(nxa);
#endif

    for (int m = 0;; m++) {
        const bool end = cur.tile >= a.n_tiles;
        // past the stream: the first chunk after the last real tile carries the terminator, every other returns
        if (end && !(cur.prev_valid && cur.c == 0)) return;
        // prefetch the next owned chunk's records; its successor's ids
#if TCGS_K7_LOOKAHEAD >= 2
        Cursor nx3 = nxa;
        for (int i = 0; i < NP; i++) cursor_next<DYN>(nx3, a, sm);
        const uint32_t id_nx3 = list_id(nx3);
        const Cursor nx2 = nxa;
        const uint32_t id_nx2 = id_nxa;
        Rec rn;
        if (K7_RECDEPTH == 3) gather(nxa, id_nxa, (m + 2) % 3, rn);
        else gather(nxt, id_nxt, (m + 1) & 1, rn);
#else
        Cursor nx2 = nxt;
        for (int i = 0; i < NP; i++) cursor_next<DYN>(nx2, a, sm);
        Rec rn;
        gather(nxt, id_nxt, (m + 1) & 1, rn);
        const uint32_t id_nx2 = list_id(nx2);
#endif
        if (K7_RECBUF) {  // this chunk's records (issued one or two groups before the one just issued)
            cp_async_wait<K7_RECDEPTH - 1>();
            rc = sm.rbuf[K7_RECBUF ? p : 0][m % K7_RECDEPTH][lane];
        }

        // evaluate this chunk (registers only)
#ifdef TCGS_K7_SLOWPROD  // sensitivity experiment: extra dependent work per producer chunk
        {
            float z = (float)lane;
#pragma unroll
            for (int q = 0; q < TCGS_K7_SLOWPROD; q++) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(z));
            if (z == 12345.0f) sm.c_dead = 0;
        }
#endif
        const bool valid = cur.c * 32 + lane < cur.n;
        // compacted lists: the marked (dead) entries of the full list before this live one -- culls if reached
        const uint32_t dpre = (K7_COMPACT && cmp && valid) ? a.cdb[cur.beg + cur.c * 32 + lane] : 0u;
        float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        bool live = false;
        // tile_center (tensor_path.py:21-22); the global-coordinate ablation keeps the origin at (0, 0)
        if (valid) live = gaussian_coeffs<BOXCULL>(rc, GLOBAL ? 0.0f : cur.ox, GLOBAL ? 0.0f : cur.oy, v);
        if (DUMP && valid && !live) {  // dead on the whole tile (box test): class 4 at every pixel
            uint4 *row = reinterpret_cast<uint4 *>(a.dump_class + (size_t)(cur.beg + cur.c * 32 + lane) * 256);
            const uint4 four = make_uint4(0x04040404u, 0x04040404u, 0x04040404u, 0x04040404u);
#pragma unroll 1
            for (int q = 0; q < 16; q++) row[q] = four;
        }
        uint4 vlo = make_uint4(0, 0, 0, 0), vhi = make_uint4(0, 0, 0, 0);
        if (TC && live) make_vrow<MODE>(v, vlo, vhi);
        const float4 col = make_float4(rc.r, rc.g, rc.b, 0.f);

        // wait for the compaction token
        if (!(p == 0 && m == 0)) K7_TWAIT(0, mbar_wait(&sm.tok[p], p == 0 ? ((m - 1) & 1) : (m & 1)));
#ifdef TCGS_K7_TIMING
        const long long t_tok = clock64();
#endif
        int k = sm.c_k;
        bool open = sm.c_open != 0;
        auto acquire = [&]() {
            if (!open) {
                K7_TWAIT(1, mbar_wait_prod(&sm.released[k % S], ((k / S) & 1) ^ 1));
                open = true;
            }
        };
        auto emit = [&](int tile, int sq, int n_live, int last, uint32_t dead_total, uint32_t n_total) {
            acquire();
            const int st = k % S;
            // unused columns of a partial stage: a row whose beta is -65504 at every pixel, so consumers need
            // no per-column validity test (it can never pass EarlyCull)
            for (int row = n_live + lane; tile >= 0 && row < K7_BATCH; row += 32) {
                if (TC) {
                    const uint4 lo = make_uint4(0xFBFFu, 0u, 0u, 0u);  // fp16 -65504 in K-column 0 (U = 1)
                    *reinterpret_cast<uint4 *>(sm.V[st] + kmaj_off(row, 0)) = lo;
                    *reinterpret_cast<uint4 *>(sm.V[st] + kmaj_off(row, 8)) = make_uint4(0u, 0u, 0u, 0u);
                } else {
                    sm.vf[st][row][0] = make_float4(-65504.0f, 0.f, 0.f, 0.f);
                    sm.vf[st][row][1] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
            if (GLOBAL && tile >= 0) write_global_u(sm.Ug[st], tile, a, lane);
            if (TC) fence_async_smem();
            __syncwarp();
            if (lane == 0) {
                StageMeta mt;
                mt.tile = tile;
                mt.seq = sq;
                mt.n_live = n_live;
                mt.last = last;
                mt.dead_total = dead_total;
                mt.n_total = n_total;
                sm.meta[st] = mt;
                if (!TC) {
                    mbar_arrive(&sm.full[st]);
                } else {
                    // TMEM buffer b was last read by the consumers of stage k - NB
                    const int b = k % NB;
                    if (k >= NB) K7_TWAIT(2, mbar_wait_prod(&sm.released[(k - NB) % S], ((k - NB) / S) & 1));
                    if (tile >= 0) {
                        mbar_arrive(&sm.mma_done[b]);  // the stage's rows and meta (release); the commit is the 2nd
                        tc_fence_after();
                        const uint64_t bdesc = umma_desc(sm.V[st]);
#pragma unroll
                        for (int h = 0; h < 2; h++)
                            mma_f16(tmem + b * (2 * K7_BATCH) + h * K7_BATCH,
                                    umma_desc(GLOBAL ? sm.Ug[st][h] : sm.U[h]), bdesc, IDESC);
                        mma_commit(&sm.mma_done[b]);
                    } else {
                        mbar_arrive_n(&sm.mma_done[b], 2);  // end of stream: no MMA
                    }
                }
            }
            __syncwarp();
            k++;
            open = false;
        };
        if (end) {
            emit(-1, cur.seq, 0, 1, 0u, 0u);
            return;
        }
        const int sq = cur.seq;
        if (cur.c == 0) {  // first chunk of a tile: reset its retirement counter and running counts
            if (lane == 0) *((volatile int *)&sm.retire[sq & 7]) = 0;
            sm.c_fill = 0;
            sm.c_dead = 0;
        }
        __syncwarp();
        const bool retired = cur.c > 0 && *((volatile int *)&sm.retire[sq & 7]) >= K7_CONSUMER_WARPS;
        if (!retired) {
            int fill = sm.c_fill;
            uint32_t dead = sm.c_dead;
            const unsigned lm = __ballot_sync(FULL, live), dm = __ballot_sync(FULL, valid && !live);
            const int slot = fill + __popc(lm & lt);
            const uint32_t my_dead = dead + __popc(dm & lt) + dpre;
            const int nl = __popc(lm);
            auto put = [&](int row) {
                const int st = k % S;
                if (TC) {
                    *reinterpret_cast<uint4 *>(sm.V[st] + kmaj_off(row, 0)) = vlo;
                    *reinterpret_cast<uint4 *>(sm.V[st] + kmaj_off(row, 8)) = vhi;
                } else {
                    sm.vf[st][row][0] = make_float4(v[0], v[1], v[2], v[3]);
                    sm.vf[st][row][1] = make_float4(v[4], v[5], 0.f, 0.f);
                }
                sm.col[st][row] = col;
                sm.dead_before[st][row] = my_dead;
                if (DUMP) sm.pos[st][row] = cur.beg + (uint32_t)(cur.c * 32 + lane);
            };
            if (nl > 0) acquire();
            if (live && slot < K7_BATCH) put(slot);
            if (fill + nl >= K7_BATCH) {
                emit(cur.tile, sq, K7_BATCH, 0, 0u, (uint32_t)cur.nfull);
                fill = fill + nl - K7_BATCH;
                if (fill > 0) {
                    acquire();
                    if (live && slot >= K7_BATCH) put(slot - K7_BATCH);
                }
            } else {
                fill += nl;
            }
            dead += __popc(dm);
            if (cur.c == cur.chunks - 1) {
                emit(cur.tile, sq, fill, 1, dead + (uint32_t)(cur.nfull - cur.n), (uint32_t)cur.nfull);
                fill = 0;
            }
            __syncwarp();
            if (lane == 0) {
                sm.c_fill = fill;
                sm.c_dead = dead;
            }
        }
        __syncwarp();
        if (lane == 0) {
            sm.c_k = k;
            sm.c_open = open ? 1 : 0;
            mbar_arrive(&sm.tok[(p + 1) % NP]);  // release: the compaction state travels with the token
#ifdef TCGS_K7_TIMING
            atomicAdd(&g_k7_wait[7], (unsigned long long)(clock64() - t_tok));
#endif
        }
        __syncwarp();
        cur = nxt;
        nxt = nx2;
        if (!K7_RECBUF) rc = rn;
        id_nxt = id_nx2;
#if TCGS_K7_LOOKAHEAD >= 2
        nxa = nx3;
        id_nxa = id_nx3;
#endif
    }
}

// ------------------------------------------------------------------------------------------ kernel
template <int MODE, bool DYN, int FL>
__global__ void __launch_bounds__(K7_THREADS, K7_CTAS_PER_SM) render_kernel(RenderArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    using K7Smem = K7SmemT<MODE == TCGS_ALPHA_TC_K8_GLOBAL>;
    K7Smem &sm = *reinterpret_cast<K7Smem *>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr bool TC = MODE != TCGS_ALPHA_FFMA;
    constexpr bool EC = !(FL & FL_ECOFF);       // EarlyCull: the cull decided on beta' before any ex2
    constexpr bool DUMP = (FL & FL_DUMP) != 0;
    constexpr bool GLOBAL = MODE == TCGS_ALPHA_TC_K8_GLOBAL;
    constexpr float INF = __builtin_huge_valf();
    const unsigned FULL = 0xffffffffu;

    // pixels owned by a consumer thread.  NPIX = 1: warp w covers an 8x4 block, TMEM lanes 32(w%4).. of
    // pixel half w/4.  NPIX = 2: warp w covers an 8x8 block as horizontal pixel pairs; pixel h of a thread
    // is row 32w + lane of pixel half h, so one thread reads both halves of its TMEM lane.
    constexpr int NPIX = K7_PIX;
    int lx[NPIX], ly[NPIX], hf[NPIX];
#pragma unroll
    for (int h = 0; h < NPIX; h++) {
        if (NPIX == 1) {
            lx[h] = 8 * (warp & 1) + (lane & 7);
            ly[h] = 4 * ((warp >> 1) & 3) + (lane >> 3);
            hf[h] = (warp >> 2) & 1;
        } else {
            lx[h] = 8 * (warp & 1) + 2 * (lane & 3) + h;
            ly[h] = 8 * ((warp >> 1) & 1) + (lane >> 2);
            hf[h] = h;
        }
    }
    const int urow = 32 * (warp & 3) + lane;  // TMEM lane == U row within a half

    if (warp < K7_CONSUMER_WARPS && TC) {
#pragma unroll
        for (int h = 0; h < NPIX; h++) {
            const float ux = (float)(lx[h] - 8), uy = (float)(ly[h] - 8);
            const float u[16] = {1.f, 1.f, 1.f, ux, uy, ux * ux, ux * uy, uy * uy, ux, uy, ux * ux, ux * uy, uy * uy, 1.f, 0.f, 0.f};
#pragma unroll
            for (int k = 0; k < 16; k++) sm.U[hf[h]][kmaj_off(urow, k)] = __float2half_rn(u[k]);
        }
        fence_async_smem();
    }
    if (tid == 0) {
        for (int s = 0; s < S; s++) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.released[s], K7_CONSUMER_WARPS);
        }
        for (int b = 0; b < NB; b++) mbar_init(&sm.mma_done[b], 2);  // producer arrive + MMA commit
        for (int q = 0; q < K7_PRODUCERS; q++) mbar_init(&sm.tok[q], 1);
        sm.c_fill = 0;
        sm.c_k = 0;
        sm.c_open = 0;
        sm.c_dead = 0;
        for (int q = 0; q < 16; q++) sm.tslot[q] = ~0ull;  // no stream position fetched yet
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (TC && warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                     "r"(K7_TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (TC) tc_fence_before();
    __syncthreads();
    if (TC) tc_fence_after();
    // PDL: the set-up above (A operand, barriers, TMEM) overlapped the previous kernel; the lists, records and
    // counters it reads below are written by the kernels before it
    pdl_wait();
    pdl_launch();
#ifdef TCGS_K7_TIMING
    const long long t_start = clock64();
#endif
    const uint32_t tmem = TC ? sm.tmem_base : 0u;
    const uint32_t *ids = a.ids_override ? a.ids_override
                                         : ((K7_COMPACT && a.ctr->compact) ? a.cid : (a.ctr->tile_cur ? a.ids1 : a.ids0));

    // per-thread K8 sums in 32 bits (a thread's pixels see at most a few hundred tiles of bounded lists); widened
    // to 64 bits in the CTA reduction
    uint32_t s_blend = 0, s_cull = 0, s_term = 0, s_pairs = 0;
    if (warp >= K7_CONSUMER_WARPS) {
        producer<MODE, DYN, FL>(sm, a, ids, tmem, warp - K7_CONSUMER_WARPS);
    } else {
        int cur_seq = -1, cur_tile = -1;
        bool done[NPIX], term[NPIX];
        float T[NPIX], c0[NPIX], c1[NPIX], c2[NPIX];
        uint32_t cull[NPIX];    // EarlyCull culls of dead (box-culled) Gaussians the pixel reached
        uint32_t reached[NPIX];  // live list entries the pixel reached (culls = reached - blends + cull)
        float fcnt[NPIX];  // blends of this pixel (exact in fp32; kept on the FMA pipe)
        bool warp_done = true;
        uint32_t n_total = 0;
#pragma unroll
        for (int h = 0; h < NPIX; h++) {
            term[h] = false;
            done[h] = true;
            T[h] = 1.0f;
            c0[h] = c1[h] = c2[h] = fcnt[h] = 0.0f;
            cull[h] = reached[h] = 0;
        }
#ifdef TCGS_K7_PROFILE  // experiment builds only: per-warp work (stages entered, relevant columns) replaces T / n_contrib
        int prof_rel = 0, prof_st = 0;
#endif
        // pixel h of this thread in tile t (recomputed where needed instead of held in registers)
        auto pix = [&](int t, int h, int &x, int &y) {
            x = (t % a.tiles_x) * TILE + lx[h];
            y = (a.band_y0 + t / a.tiles_x) * TILE + ly[h];
            return x < a.width && y < a.height;
        };
        auto flush = [&]() {
#pragma unroll
            for (int h = 0; h < NPIX; h++) {
                int px, py;
                const bool inside = pix(cur_tile, h, px, py);
#ifdef TCGS_K7_PROFILE
                T[h] = (float)prof_st;
                fcnt[h] = (float)prof_rel;
#endif
                if (inside) {
                    const int64_t p = (int64_t)py * a.width + px;
                    a.rgb[3 * p] = c0[h];
                    a.rgb[3 * p + 1] = c1[h];
                    a.rgb[3 * p + 2] = c2[h];
                    a.T[p] = T[h];
                    a.n_contrib[p] = (int32_t)fcnt[h];
                    s_pairs += n_total;
                }
                s_blend += (uint32_t)fcnt[h];
                s_cull += cull[h] + reached[h] - (uint32_t)fcnt[h];
                s_term += term[h] ? 1u : 0u;
            }
#ifdef TCGS_K7_PROFILE
            prof_rel = prof_st = 0;
#endif
        };
        static_assert(NB >= 2 && S % NB == 0, "K7 stage / TMEM rings");
        for (int k = 0;; k++) {
            const int st = k % S, b = k % NB;
            // tensor cores: mma_done[b] completes on the producer's arrival (stage rows, meta) AND the MMA commit
            if (TC) {
                K7_TWAIT(4, mbar_wait(&sm.mma_done[b], (k / NB) & 1));
                tc_fence_after();
            } else {
                K7_TWAIT(3, mbar_wait(&sm.full[st], (k / S) & 1));
            }
            const StageMeta m = sm.meta[st];
            if (m.seq != cur_seq || m.tile < 0) {
                if (cur_seq >= 0) flush();
                if (m.tile < 0) break;
                cur_seq = m.seq;
                cur_tile = m.tile;
                const int tx = cur_tile % a.tiles_x, ty = a.band_y0 + cur_tile / a.tiles_x;
                bool all_done = true;
#pragma unroll
                for (int h = 0; h < NPIX; h++) {
                    done[h] = !(tx * TILE + lx[h] < a.width && ty * TILE + ly[h] < a.height);
                    all_done = all_done && done[h];
                    term[h] = false;
                    T[h] = 1.0f;
                    c0[h] = c1[h] = c2[h] = 0.0f;
                    cull[h] = reached[h] = 0;
                    fcnt[h] = 0.0f;
                }
                n_total = m.n_total;
                warp_done = __all_sync(FULL, all_done);
                if (warp_done && lane == 0) atomicAdd(&sm.retire[cur_seq & 7], 1);
            }
            if (!warp_done) {
#ifdef TCGS_K7_PROFILE
                prof_st++;
#endif
                const int nl = m.n_live;
                float thr[NPIX];
                uint32_t tb[NPIX];
#pragma unroll
                for (int h = 0; h < NPIX; h++) {
                    if (!done[h]) reached[h] += (uint32_t)nl;  // (a pixel terminating here gives back the rest)
                    // pass threshold: the EarlyCull cut of beta' (EC) or the 1/255 cut of alpha (EarlyCull off)
                    // while the pixel is live, +inf once it has terminated (a float, so the test stays one FSETP
                    // and the update a predicated move)
                    thr[h] = done[h] ? INF : (EC ? CUT_LOG2 : ALPHA_CUT);
                    tb[h] = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + b * (2 * K7_BATCH) + hf[h] * K7_BATCH;
                }
                // one column of the stage: a pixel passes EarlyCull iff beta >= thr (thr = the cut while live,
                // +inf once done); a warp vote skips the column when no pixel of the warp passes (uniform branch)
                auto column = [&](const uint32_t (&rb)[NPIX], const uint32_t (&ex)[NPIX], int col) {
                    bool p[NPIX], any = false;
                    float alv[NPIX];
#pragma unroll
                    for (int h = 0; h < NPIX; h++) {
                        const float bt = __uint_as_float(rb[h]);
                        if (EC) {
                            p[h] = bt >= thr[h];  // (columns >= n_live hold beta = -65504: never pass)
                            // fp16 global coordinates can overflow: a non-finite beta is a cull (tensor_path.py:113)
                            if (GLOBAL) p[h] = p[h] && bt < INF;
                            if (EX2EARLY) alv[h] = __uint_as_float(ex[h]);  // exponentials issued per TMEM group
                        } else {  // EarlyCull off: the exponential of every active fragment, then the alpha cut
                            alv[h] = ex2_approx(bt);
                            p[h] = alv[h] >= thr[h];
                        }
                        any = any || p[h];
                    }
                    if (DUMP) {
                        const uint32_t e = sm.pos[st][col < nl ? col : 0];
#pragma unroll
                        for (int h = 0; h < NPIX; h++) {
                            int dx_, dy_;
                            if (col < nl && pix(cur_tile, h, dx_, dy_)) {
                                const size_t o = (size_t)e * 256 + (size_t)(ly[h] * TILE + lx[h]);
                                a.dump_beta[o] = __uint_as_float(rb[h]);
                                if (thr[h] < TERM_CODE0) {  // reached: classify as the blend below does
                                    const float al = ex2_approx(__uint_as_float(rb[h]));
                                    a.dump_class[o] = !p[h] ? 1 : (fmaf(-al, T[h], T[h]) < TERM_T ? 3 : 2);
                                }
                            }
                        }
                    }
                    if (__any_sync(FULL, any)) {
#ifdef TCGS_K7_PROFILE
                        prof_rel++;
#endif
                        const float4 cc = sm.col[st][col];
#pragma unroll
                        for (int h = 0; h < NPIX; h++) {
                            // alpha = 2^beta' for a passing lane, exactly 0 otherwise (ex2(-inf) = +0), so a
                            // non-passing lane's update below is the identity: T - 0 T = T >= 1e-4 never
                            // terminates, C + 0 c = C.  (No min(alpha, 1): alpha > 1 only by rounding, and then
                            // T - alpha T < 1e-4 terminates exactly as alpha = 1 would.)
                            const float al = (EC && !EX2EARLY) ? ex2_approx(p[h] ? __uint_as_float(rb[h]) : -INF)
                                                                : (p[h] ? alv[h] : 0.0f);
                            const float tn = fmaf(-al, T[h], T[h]);
                            if (p[h]) fcnt[h] += 1.0f;  // passes; the terminating one is taken back per stage
                            const bool tm = tn < TERM_T;  // termination precedes compositing
                            // a terminated pixel never passes again, and its threshold records the column
                            asm("{\n.reg .pred q;\nsetp.lt.f32 q, %1, %2;\n@q mov.f32 %0, %3;\n}"
                                : "+f"(thr[h]) : "f"(tn), "f"(TERM_T), "f"(term_code(col)));
                            if (!tm) {
                                const float w = al * T[h];
                                c0[h] = fmaf(w, cc.x, c0[h]);
                                c1[h] = fmaf(w, cc.y, c1[h]);
                                c2[h] = fmaf(w, cc.z, c2[h]);
                                T[h] = tn;
                            }
                        }
                    }
                };
#ifndef TCGS_K7_GROUP  // 8-column groups at 48 registers (4 CTAs/SM: 444 -> 440 us at C2), 16 at 56 (equal)
#define TCGS_K7_GROUP (TCGS_K7_CTAS >= 4 ? 8 : 16)
#endif
                constexpr int G = NPIX == 1 ? TCGS_K7_GROUP : 8;  // columns per TMEM load group (G x NPIX betas)
#pragma unroll
                for (int hc = 0; hc < K7_BATCH / G; hc++) {
                    uint32_t r[NPIX][G];
                    if (TC) {
#pragma unroll
                        for (int h = 0; h < NPIX; h++) tmem_ld<G>(tb[h] + G * hc, r[h]);
                        tmem_wait_ld();
#pragma unroll
                        for (int h = 0; h < NPIX; h++)
#pragma unroll
                            for (int j = 0; j < G; j++) asm volatile("" : "+r"(r[h][j]));
                    } else {
#pragma unroll
                        for (int h = 0; h < NPIX; h++) {
                            const float ux = (float)(lx[h] - 8), uy = (float)(ly[h] - 8);
#pragma unroll
                            for (int j = 0; j < G; j++) {
                                const float4 p0 = sm.vf[st][G * hc + j][0], p1 = sm.vf[st][G * hc + j][1];
                                r[h][j] = __float_as_uint(p0.x + p0.y * ux + p0.z * uy + p0.w * ux * ux + p1.x * ux * uy +
                                                          p1.y * uy * uy);
                            }
                        }
                    }
                    // TCGS_K7_EX2EARLY: the group's exponentials issued back to back ahead of the column votes, so
                    // their latency leaves the blend chain (costs an ex2 on the columns no pixel passes)
                    uint32_t e2[NPIX][EX2EARLY ? G : 1];
                    if (EX2EARLY) {
#pragma unroll
                        for (int h = 0; h < NPIX; h++)
#pragma unroll
                            for (int j = 0; j < G; j++)
                                asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=r"(e2[h][j]) : "f"(__uint_as_float(r[h][j])));
                    }
#pragma unroll
                    for (int j = 0; j < G; j++) {
                        uint32_t rj[NPIX], ej[NPIX];
#pragma unroll
                        for (int h = 0; h < NPIX; h++) {
                            rj[h] = r[h][j];
                            ej[h] = e2[h][EX2EARLY ? j : 0];
                        }
                        column(rj, ej, G * hc + j);
                    }
                }
#ifdef TCGS_K7_SLOWCONS  // sensitivity experiment: extra dependent work per consumer warp-stage
                {
                    float z = (float)lane;
#pragma unroll
                    for (int q = 0; q < TCGS_K7_SLOWCONS; q++) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(z));
                    if (z == 12345.0f) cull[0] += 1;
                }
#endif
                // terminated in this stage: thr holds term_code(column) (done lanes entered with +inf).  Rare (a
                // pixel terminates once per tile), so the bookkeeping sits behind one warp vote.
                bool tstage[NPIX], tany = false;
#pragma unroll
                for (int h = 0; h < NPIX; h++) {
                    tstage[h] = thr[h] >= TERM_CODE0 && thr[h] != INF;
                    tany = tany || tstage[h];
                }
                if (__any_sync(FULL, tany)) {
                    bool all_done = true;
#pragma unroll
                    for (int h = 0; h < NPIX; h++) {
                        if (tstage[h]) {
                            const int jt = term_col(thr[h]);
                            fcnt[h] -= 1.0f;  // the terminating pass was counted
                            // reached: the live columns before the terminating one, plus the dead Gaussians
                            // of the list before it (all culls)
                            reached[h] -= (uint32_t)(nl - jt);
                            cull[h] += sm.dead_before[st][jt];
                            term[h] = true;
                            done[h] = true;
                        }
                        all_done = all_done && done[h];
                    }
                    if (__all_sync(FULL, all_done)) {
                        warp_done = true;
                        if (lane == 0) atomicAdd(&sm.retire[cur_seq & 7], 1);
                    }
                }
            }
            if (m.last) {
#pragma unroll
                for (int h = 0; h < NPIX; h++)
                    if (!done[h]) cull[h] += m.dead_total;  // list exhausted: every dead Gaussian was a cull
            }
            if (TC) tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.released[st]);
        }
    }

#ifdef TCGS_K7_TIMING
    if (lane == 0) atomicAdd(&g_k7_wait[warp >= K7_CONSUMER_WARPS ? 5 : 6], (unsigned long long)(clock64() - t_start));
#endif
    // the outputs may be another GPU's frame mapped over NVLink (tile-band peer output): make this thread's
    // pixel stores visible system-wide before the CTA retires
    if (warp < K7_CONSUMER_WARPS) __threadfence_system();

    // K8: fragment statistics, one atomic per CTA and counter
    unsigned long long w_blend = s_blend, w_cull = s_cull, w_term = s_term, w_pairs = s_pairs;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        w_blend += __shfl_xor_sync(FULL, w_blend, o);
        w_cull += __shfl_xor_sync(FULL, w_cull, o);
        w_term += __shfl_xor_sync(FULL, w_term, o);
        w_pairs += __shfl_xor_sync(FULL, w_pairs, o);
    }
    if (lane == 0 && warp < K7_CONSUMER_WARPS) {
        sm.red[warp][0] = w_blend;
        sm.red[warp][1] = w_cull;
        sm.red[warp][2] = w_term;
        sm.red[warp][3] = w_pairs;
    }
    if (TC) tc_fence_before();
    __syncthreads();
    if (tid < 4) {
        unsigned long long t = 0;
        for (int w = 0; w < K7_CONSUMER_WARPS; w++) t += sm.red[w][tid];
        unsigned long long *dst = tid == 0 ? &a.ctr->f_blend
                                  : tid == 1 ? &a.ctr->f_cull
                                  : tid == 2 ? &a.ctr->pixels_terminated
                                             : &a.ctr->pairs;
        if (t) atomicAdd(dst, t);
    }
    if (TC && warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(K7_TMEM_COLS));
    }
}

__global__ void k7_reset(DevCounters *ctr) {
    pdl_wait();
    pdl_launch();
    if (threadIdx.x < 4) (&ctr->f_blend)[threadIdx.x] = 0ull;
    if (threadIdx.x == 0) ctr->tile_queue = 0u;
}

// dynamic shared memory of a K7 variant: K7_SMEM_BYTES (which also caps residency at K7_CTAS_PER_SM), or more for
// the global-coordinate ablation's per-stage A operands (lower occupancy is fine for an ablation)
template <int MODE>
constexpr int k7_smem() {
    constexpr int need = (int)sizeof(K7SmemT<MODE == TCGS_ALPHA_TC_K8_GLOBAL>) + 1024;
    return need > K7_SMEM_BYTES ? need : K7_SMEM_BYTES;
}

template <int MODE, bool DYN, int FL>
cudaError_t launch_mode(const RenderArgs &a, int num_sms, cudaStream_t st) {
    static bool configured_dev[TCGS_MAX_DEVICES] = {};
    bool &configured = configured_dev[current_device()];
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(render_kernel<MODE, DYN, FL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             k7_smem<MODE>());
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int grid = num_sms * K7_CTAS_PER_SM;
    return launch_k(render_kernel<MODE, DYN, FL>, grid, K7_THREADS, (size_t)k7_smem<MODE>(), st, a);
}

// EarlyCull on/off for the lone-frame (dynamic) and frames-in-flight (static) schedules; the debug dump runs
// with the static schedule.
template <int MODE>
cudaError_t launch_variant(const RenderArgs &a, bool dyn, bool early_cull, bool dump, int sms, cudaStream_t st) {
    if (dump) return early_cull ? launch_mode<MODE, false, FL_DUMP>(a, sms, st)
                                : launch_mode<MODE, false, FL_DUMP | FL_ECOFF>(a, sms, st);
    if (early_cull) return dyn ? launch_mode<MODE, true, 0>(a, sms, st) : launch_mode<MODE, false, 0>(a, sms, st);
    return dyn ? launch_mode<MODE, true, FL_ECOFF>(a, sms, st) : launch_mode<MODE, false, FL_ECOFF>(a, sms, st);
}

}  // namespace

// This file is compiled three times (paper_2505_24796_b200/build.py): launch_render_k7 with the default residency
// (4 CTAs per SM, 2 producer warps); launch_render_k7_few with 3 CTAs x 4 producer warps, the better trade when a
// frame has fewer tiles than resident CTAs (C1's 256 tiles: 94 -> 66 us); launch_render_k7_heavy, the default
// residency walking the compacted live lists of producer-heavy frames (C5).
#ifndef TCGS_K7_ENTRY
#define TCGS_K7_ENTRY launch_render_k7
#endif
cudaError_t TCGS_K7_ENTRY(int alpha_mode, int early_cull, float *dump_beta, uint8_t *dump_class,
                          const tcgs_camera &cam, const Band &band, const uint32_t *ids_override,
                          void *ws, const Layout &L, float *rgb, float *T, int32_t *n_contrib, cudaStream_t st) {
    static_assert(sizeof(K7SmemT<false>) + 1024 <= K7_SMEM_BYTES, "K7 shared memory");
    RenderArgs a;
    a.rec = at<Rec>(ws, L.rec);
    a.ids0 = at<uint32_t>(ws, L.tval[0]);
    a.ids1 = at<uint32_t>(ws, L.tval[1]);
    a.ids_override = ids_override;
    a.ranges = at<uint2>(ws, L.ranges);
    a.cid = at<uint32_t>(ws, L.cid);
    a.cdb = at<uint32_t>(ws, L.cdb);
    a.ccount = at<uint32_t>(ws, L.ccount);
    a.ctr = at<DevCounters>(ws, L.counters);
    a.tiles_x = band.tiles_x;
    a.band_y0 = band.y0;
    a.n_tiles = band.n_tiles();
    a.width = cam.width;
    a.height = cam.height;
    a.rgb = rgb;
    a.T = T;
    a.n_contrib = n_contrib;
    a.dump_beta = dump_beta;
    a.dump_class = dump_class;
    const bool dump = dump_beta != nullptr && dump_class != nullptr;
    // per-launch counters: the tile queue and the fragment statistics (f_blend, f_cull, terminated, pairs)
    cudaError_t e = launch_k(k7_reset, 1, 32, 0, st, a.ctr);
    if (e != cudaSuccess) return e;
    const bool dyn = band.schedule == TCGS_SCHEDULE_DYNAMIC;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const bool ec = early_cull != 0;
    switch (alpha_mode) {
        case TCGS_ALPHA_TC_HILO: return launch_variant<TCGS_ALPHA_TC_HILO>(a, dyn, ec, dump, sms, st);
        case TCGS_ALPHA_TC_K8: return launch_variant<TCGS_ALPHA_TC_K8>(a, dyn, ec, dump, sms, st);
        case TCGS_ALPHA_FFMA: return launch_variant<TCGS_ALPHA_FFMA>(a, dyn, ec, dump, sms, st);
        case TCGS_ALPHA_TC_K8_GLOBAL:  // ablation only: EarlyCull on, static schedule
            return dump ? launch_mode<TCGS_ALPHA_TC_K8_GLOBAL, false, FL_DUMP>(a, sms, st)
                        : launch_mode<TCGS_ALPHA_TC_K8_GLOBAL, false, 0>(a, sms, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace tcgs

#if defined(TCGS_K7_TIMING) && !defined(TCGS_K7_SECOND_BUILD)
// experiment builds only (not in include/tcgs.h): read and clear the K7 wait counters -- cycles summed over warps:
// [0] producer token, [1] producer empty stage, [2] producer TMEM buffer, [3] consumer full stage,
// [4] consumer MMA done, [5] producer total, [6] consumer total
extern "C" int tcgs_k7_timing(unsigned long long *out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, tcgs::g_k7_wait, sizeof(unsigned long long) * 8);
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(tcgs::g_k7_wait, z, sizeof(z));
    return 0;
}
#endif
