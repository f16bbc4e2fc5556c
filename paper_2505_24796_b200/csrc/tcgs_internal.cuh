// tcgs_internal.cuh -- shared definitions of libtcgs.so (sm_100a only).
#pragma once

#include <cuda_fp16.h>
#include <math.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <utility>

#include "tcgs.h"

namespace tcgs {

constexpr int TILE = 16;              // src/tilesplat/tiling.py:11
constexpr int RADIX_BITS = 8;
constexpr int RADIX = 1 << RADIX_BITS;
constexpr int OS_THREADS = 256;       // onesweep radix pass: 8 warps per CTA
constexpr int OS_WARPS = OS_THREADS / 32;
#ifndef TCGS_DEPTH_IPT
#define TCGS_DEPTH_IPT 8
#endif
constexpr int DEPTH_IPT = TCGS_DEPTH_IPT;  // items per thread: depth sort (u32 prefix keys), 2048-item tiles
#ifndef TCGS_TILEKEY_IPT
#define TCGS_TILEKEY_IPT 16
#endif
constexpr int TILEKEY_IPT = TCGS_TILEKEY_IPT;  // items per thread: tile-key sort, 4096-item tiles
constexpr int MAX_PASSES = 8;         // depth key: <= 64 bits
constexpr int TILE_MAX_PASSES = 4;    // tile key: <= 32 bits
#ifndef TCGS_DUP_ITEMS
#define TCGS_DUP_ITEMS 1024
#endif
constexpr int DUP_ITEMS = TCGS_DUP_ITEMS;  // Gaussians per duplicate-with-keys CTA (at most; see bin_tiles)
constexpr int DUP_MIN_CTAS = 4 * 148;     // K3/K4 CTAs below which a CTA takes fewer Gaussians
constexpr int DUP_THREADS = 256;

#ifndef TCGS_K7_PIX
#define TCGS_K7_PIX 1
#endif
constexpr int K7_PIX = TCGS_K7_PIX;              // pixels per consumer thread (1 or 2)
constexpr int K7_CONSUMER_WARPS = 8 / K7_PIX;  // 256 pixels of a 16x16 tile
#ifndef TCGS_K7_PRODUCERS
// measured (r2aa): 4 CTAs/SM x 2 producers (48 registers) against 3 CTAs/SM x 4 producers (56 registers): C2 K7
// 475 -> 445 us, C5 2.37 -> 2.45 ms; 4 CTAs x 3 producers (40 registers, spills): 504 us / 2.82 ms
#define TCGS_K7_PRODUCERS 2
#endif
constexpr int K7_PRODUCERS = TCGS_K7_PRODUCERS;  // producer warps (alternate 32-entry chunks, token-ordered compaction)
constexpr int K7_THREADS = 32 * (K7_CONSUMER_WARPS + K7_PRODUCERS);
#ifndef TCGS_K7_BATCH
#define TCGS_K7_BATCH 32
#endif
#ifndef TCGS_K7_TMEM_BUFS
#define TCGS_K7_TMEM_BUFS 2
#endif
constexpr int K7_BATCH = TCGS_K7_BATCH;  // live Gaussians per tcgen05 batch (MMA N): 32 or 64
#ifndef TCGS_K7_STAGES
#define TCGS_K7_STAGES 4
#endif
constexpr int K7_STAGES = TCGS_K7_STAGES;  // shared-memory B-operand stages
constexpr int K7_TMEM_BUFS = TCGS_K7_TMEM_BUFS;  // TMEM accumulator buffers (1: released after the last load)
constexpr int K7_TMEM_COLS = K7_TMEM_BUFS * 2 * K7_BATCH;  // buffers x pixel halves x N
#ifndef TCGS_K7_CTAS
#define TCGS_K7_CTAS 4  // resident K7 CTAs per SM: TMEM 4 x 128 columns = 512, 48 registers at 320 threads
#endif
constexpr int K7_CTAS_PER_SM = TCGS_K7_CTAS;

// Long tile lists of mostly dead entries (C5: 6M Gaussians at 1080p, 74 % of the entries are Gaussians whose
// alpha >= 1/255 ellipse misses the tile) bind K7's producers, which gather, box-test and compact every entry.
// For such frames K4 marks those entries (LIST_DEAD) and a pass after the tile sort writes each tile's live
// entries with the number of dead entries before each (the cull accounting of a termination), so K7 walks only
// the live ones.  The tile lists themselves are unchanged (tcgs_copy_lists strips the marks).
constexpr uint32_t LIST_DEAD = 0x80000000u;
constexpr int64_t COMPACT_MIN_PER_TILE = 400;  // Gaussians per frame tile from which binning compacts
inline bool producer_heavy(int64_t P, int tiles_x, int tiles_y) {
    return P > COMPACT_MIN_PER_TILE * (int64_t)tiles_x * (int64_t)tiles_y;
}

// Per-Gaussian record consumed by the blend kernel (48 B, three 16 B loads).
struct __align__(16) Rec {
    float mx, mx_lo, my, my_lo;  // float64 mean2d (src/tilesplat/projection.py:80-82) as fp32 hi + lo pairs
    float s11, s12, s22, ln_o; // conic (rounded from float64) and log opacity
    float r, g, b, opacity;    // colour (SH evaluated) and opacity
};

// ---- opt-in tile coverage.  A fragment can pass EarlyCull only inside the ellipse
// q(d) = s11 dx^2 + 2 s12 dx dy + s22 dy^2 <= Q = 2 ln(255 o) (d = pixel - mean).  The tests below keep every
// tile that ellipse, grown by margins far above K7's exponent rounding, touches -- so only splats with no
// live fragment are dropped and the image is unchanged.  The row-span parameters come from the render
// record's fp32 conic and log-opacity (what K7 evaluates), with the one cancellation-prone quantity (the
// determinant) in float64, so needle-thin ellipses keep their exact extent; rows are evaluated in fp32
// without cancellation.
constexpr double COVER_Q_MARGIN = 0.2;   // in q (0.1 in beta = ln alpha)
constexpr float COVER_PX_MARGIN = 0.5f;  // pixels, on every side

struct __align__(16) CoverRec {
    float mx, my;  // mean (pixels)
    float b_a;     // s12 / s11: the centre of a row's x-interval is -b_a * dy
    float det_a;   // det / s11^2: the half-width is sqrt(det_a (ry^2 - dy^2))
    float ry;      // |dy| extent of the ellipse: sqrt(Q s11 / det)
    float dys;     // dy of the rightmost point (the leftmost one is at -dys)
    float pad;
    int mode;      // 0: ellipse; 1: degenerate record, keep the reference's square; 2: no live fragment
};

__host__ __device__ inline CoverRec make_cover(const Rec &r) {
    CoverRec c;
    c.mx = (float)((double)r.mx + (double)r.mx_lo);
    c.my = (float)((double)r.my + (double)r.my_lo);
    c.b_a = c.det_a = c.ry = c.dys = c.pad = 0.0f;
    const float a = r.s11, b = r.s12, cc = r.s22;
    const float Q = 2.0f * (r.ln_o + 5.541263545158426f) + (float)COVER_Q_MARGIN;
    // the determinant in float64 (exact products of the fp32 entries): it is the one cancellation-prone
    // quantity; everything derived from it below keeps fp32 relative precision
    const float det = (float)((double)a * (double)cc - (double)b * (double)b);
    if (!(Q > 0.0f)) {
        c.mode = 2;
    } else if (!(a > 0.0f && cc > 0.0f && det > 0.0f) || !isfinite(det)) {
        c.mode = 1;
    } else {
        c.mode = 0;
        const float inv_a = 1.0f / a;
        c.b_a = b * inv_a;
        c.det_a = det * inv_a * inv_a;
        c.ry = sqrtf(Q * a / det);
        c.dys = -b * sqrtf(Q / (cc * det));
    }
    return c;
}

// Tiles [lo, hi] of tile row ty (within [x0, x1]) that the ellipse touches; false if none.  The x-interval of
// the ellipse over the row's pixel strip is [min of the left boundary, max of the right boundary]: the right
// boundary -b_a dy + hw(dy) is concave in dy, so its maximum over the strip is at the rightmost point's dy
// clamped into the strip (and symmetrically on the left).  hw = sqrt(det_a (ry - |dy|)(ry + |dy|)).
// one MUFU instruction, identical in every translation unit (relative error ~2^-22, far inside the margins)
__device__ __forceinline__ float sqrt_approx(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// (explicitly rounded operations: K1 and binning are compiled with different FMA contraction, and both must
// see the same spans)
__device__ __forceinline__ bool cover_row(const CoverRec &c, int ty, int x0, int x1, int &lo, int &hi) {
    lo = x0;
    hi = x1;
    if (c.mode) return c.mode == 1;
    const float ylo = fmaxf(__fsub_rn(__fsub_rn(16.0f * ty, c.my), COVER_PX_MARGIN), -c.ry);
    const float yhi = fminf(__fadd_rn(__fsub_rn(__fadd_rn(16.0f * ty, 15.0f), c.my), COVER_PX_MARGIN), c.ry);
    if (ylo > yhi) return false;
    const float yr = fminf(fmaxf(c.dys, ylo), yhi), yl = fminf(fmaxf(-c.dys, ylo), yhi);
    const float ar = fabsf(yr), al = fabsf(yl);
    const float hr = sqrt_approx(fmaxf(__fmul_rn(__fmul_rn(c.det_a, __fsub_rn(c.ry, ar)), __fadd_rn(c.ry, ar)), 0.0f));
    const float hl = sqrt_approx(fmaxf(__fmul_rn(__fmul_rn(c.det_a, __fsub_rn(c.ry, al)), __fadd_rn(c.ry, al)), 0.0f));
    const float xr = __fadd_rn(__fmul_rn(-c.b_a, yr), hr);
    const float xl = __fsub_rn(__fmul_rn(-c.b_a, yl), hl);
    const float fl = floorf(__fmul_rn(__fsub_rn(__fadd_rn(c.mx, xl), COVER_PX_MARGIN), 1.0f / 16.0f));
    const float fh = floorf(__fmul_rn(__fadd_rn(__fadd_rn(c.mx, xr), COVER_PX_MARGIN), 1.0f / 16.0f));
    lo = fl > (float)x0 ? (int)fl : x0;
    hi = fh < (float)x1 ? (int)fh : x1;
    return lo <= hi;
}

// Device-side counters and sort bookkeeping (zeroed at the start of each frame).
struct DevCounters {
    unsigned long long dropped, n_visible, n_splats, overflow;
    unsigned long long f_blend, f_cull, pixels_terminated, pairs;
    unsigned long long key_min, key_max, key_range;
    unsigned int tile_queue;
    int depth_cur, tile_cur;
    int depth_shift;           // K2: prefix shift of the depth key (0: the prefix sort is exact)
    unsigned int n_long_runs;  // K2 fix-up: runs of equal prefixes longer than a thread handles
    int debug_written;         // K1 ran with opts.debug (tcgs_copy_projection's float64 buffers are valid)
    int compact;               // binning also wrote the compacted live lists (cid / cdb / ccount) for K7
};

// Per-sort bookkeeping of the onesweep LSD radix sort (all decided on the device).
struct SortState {
    unsigned int ghist[MAX_PASSES][RADIX];  // digit counts, then exclusive global bases
    int pass_do[MAX_PASSES];                // 0: the pass is the identity (one digit value or above the key range)
    int pass_in[MAX_PASSES];                // ping-pong buffer the pass reads
    int final_buf;
    int done_ctas;  // depth_fix_hist: CTAs finished (the last one plans the passes)
    int pad[2];
    unsigned int tile_ctr[MAX_PASSES];  // onesweep passes: next radix tile to claim (launch order = look-back order)
    unsigned int drange[MAX_PASSES][2];  // depth passes: (255 - min digit, max digit), for the pass plan
};

// Onesweep look-back tables (one u64 per (radix tile, digit) and pass): epoch (32) | flag (2) | count (30).  The
// epoch of the current binning makes the previous frames' entries invalid without clearing the table; the header
// holds the epoch and a magic word whose absence (a fresh workspace) makes bin_init clear the tables once.
struct OsHeader {
    unsigned int magic, epoch;
};
constexpr unsigned int OS_MAGIC = 0x7c65a1e3u;

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

inline int64_t div_up(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct Layout {
    size_t counters, sort_state[2], rec, tmask, rect, key_src, key64[2], long_runs, fix_scratch, idx[2], radius, dbg_conic, dbg_depth, dbg_mean2d;
    size_t blocksum, lb_depth, lb_tile, lb_bytes, os_hdr, tkey[2], tval[2], ranges, total;
    size_t cid, cdb, ccount;  // compacted live lists: ids, dead entries before each, live entries per tile
    size_t zero_begin, zero_bytes;  // sort state, cleared at the start of every binning
    static Layout make(int64_t P, int W, int H, int64_t cap) {
        Layout L;
        size_t o = 0;
        size_t Pn = (size_t)(P > 0 ? P : 1), cn = (size_t)(cap > 0 ? cap : 1);
        size_t nt = (size_t)((W + TILE - 1) / TILE) * (size_t)((H + TILE - 1) / TILE);
        auto take = [&](size_t bytes) { size_t r = o; o = align_up(o + bytes, 256); return r; };
        L.counters = take(sizeof(DevCounters));
        L.zero_begin = o;
        L.sort_state[0] = take(sizeof(SortState));
        L.sort_state[1] = take(sizeof(SortState));
        L.zero_bytes = o - L.zero_begin;
        // per-pass [digit][tile] count tables of the radix passes (u64 entries: the onesweep look-back)
        L.os_hdr = take(sizeof(OsHeader));
        L.lb_depth = take(sizeof(uint64_t) * RADIX * MAX_PASSES * (size_t)div_up((int64_t)Pn, OS_THREADS * DEPTH_IPT));
        L.lb_tile = take(sizeof(uint64_t) * RADIX * TILE_MAX_PASSES * (size_t)div_up((int64_t)cn, OS_THREADS * TILEKEY_IPT));
        L.lb_bytes = o - L.lb_depth;
        L.rec = take(sizeof(Rec) * Pn);
        L.tmask = take(sizeof(uint64_t) * Pn);  // exact coverage: tile masks in depth order (K3 -> K4)
        L.rect = take(sizeof(short4) * Pn);
        L.key_src = take(sizeof(uint64_t) * Pn);
        L.key64[0] = take(sizeof(uint64_t) * Pn);
        L.key64[1] = take(sizeof(uint64_t) * Pn);
        L.idx[0] = take(sizeof(uint32_t) * Pn);
        L.idx[1] = take(sizeof(uint32_t) * Pn);
        L.radius = take(sizeof(int32_t) * Pn);
        L.long_runs = take(sizeof(uint32_t) * 4096);
        L.fix_scratch = take((sizeof(unsigned long long) + sizeof(uint32_t)) * 2 * Pn);  // pow2-padded run <= 2P
        L.dbg_conic = take(sizeof(double) * 3 * Pn);
        L.dbg_depth = take(sizeof(double) * Pn);
        L.dbg_mean2d = take(sizeof(double) * 2 * Pn);
        L.blocksum = take(sizeof(unsigned long long) * (size_t)div_up((int64_t)Pn, 32));  // >= 32 Gaussians per K3/K4 CTA
        L.tkey[0] = take(sizeof(uint32_t) * cn);
        L.tkey[1] = take(sizeof(uint32_t) * cn);
        L.tval[0] = take(sizeof(uint32_t) * cn);
        L.tval[1] = take(sizeof(uint32_t) * cn);
        L.ranges = take(sizeof(uint2) * (nt ? nt : 1));
        L.cid = take(sizeof(uint32_t) * cn);
        L.cdb = take(sizeof(uint32_t) * cn);
        L.ccount = take(sizeof(uint32_t) * (nt ? nt : 1));
        L.total = o;
        return L;
    }
};

template <typename T>
inline T *at(void *ws, size_t off) { return reinterpret_cast<T *>(static_cast<char *>(ws) + off); }
template <typename T>
inline const T *at(const void *ws, size_t off) { return reinterpret_cast<const T *>(static_cast<const char *>(ws) + off); }

struct Band {
    int tiles_x, tiles_y, y0, y1;  // tile rows [y0, y1)
    int coverage;                  // enum tcgs_coverage
    int schedule;                  // enum tcgs_schedule (K7 tile assignment)
    int n_tiles() const { return tiles_x * (y1 - y0); }
};

inline Band make_band(const tcgs_camera &cam, const tcgs_opts *o) {
    Band b;
    b.tiles_x = (cam.width + TILE - 1) / TILE;
    b.tiles_y = (cam.height + TILE - 1) / TILE;
    b.y0 = 0;
    b.y1 = b.tiles_y;
    b.coverage = o ? o->coverage : TCGS_COVER_SQUARE;
    b.schedule = o ? o->schedule : TCGS_SCHEDULE_DYNAMIC;
    if (o && o->tile_row_end > 0) {
        b.y0 = o->tile_row_begin < 0 ? 0 : o->tile_row_begin;
        b.y1 = o->tile_row_end > b.tiles_y ? b.tiles_y : o->tile_row_end;
    }
    return b;
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_preprocess(const tcgs_scene &scene, const tcgs_camera &cam, const Band &band, int debug,
                              int coverage, int defer_colour, void *ws, const Layout &L, cudaStream_t st);
cudaError_t launch_colour(const tcgs_scene &scene, const tcgs_camera &cam, const Band &band, void *ws,
                          const Layout &L, cudaStream_t st);
cudaError_t launch_preprocess_views(const tcgs_scene &scene, const tcgs_camera *cams, const Band *bands, int n_views,
                                    int debug, int coverage, int defer_colour, void *const *ws, const Layout *L,
                                    cudaStream_t st);
cudaError_t launch_bin(int64_t P, const Band &band, void *ws, const Layout &L, int64_t cap, cudaStream_t st,
                       bool compact = false);
cudaError_t launch_render_k7(int alpha_mode, int early_cull, float *dump_beta, uint8_t *dump_class,
                             const tcgs_camera &cam, const Band &band, const uint32_t *ids_override,
                             void *ws, const Layout &L, float *rgb, float *T, int32_t *n_contrib, cudaStream_t st);
cudaError_t launch_render_k7_few(int alpha_mode, int early_cull, float *dump_beta, uint8_t *dump_class,
                                 const tcgs_camera &cam, const Band &band, const uint32_t *ids_override,
                                 void *ws, const Layout &L, float *rgb, float *T, int32_t *n_contrib, cudaStream_t st);
cudaError_t launch_render_k7_heavy(int alpha_mode, int early_cull, float *dump_beta, uint8_t *dump_class,
                                   const tcgs_camera &cam, const Band &band, const uint32_t *ids_override,
                                   void *ws, const Layout &L, float *rgb, float *T, int32_t *n_contrib, cudaStream_t st);
// K7 build: producer-heavy frames (> COMPACT_MIN_PER_TILE Gaussians per frame tile: binning compacted their lists)
// -> the heavy build; fewer tiles than 4 resident CTAs per SM can take (C1) -> the 3-CTA x 4-producer build;
// otherwise the default.  TCGS_K7_BUILD=few|many in the environment forces one of the latter two (tests).
inline cudaError_t launch_render(int64_t P, int alpha_mode, int early_cull, float *dump_beta, uint8_t *dump_class,
                                 const tcgs_camera &cam, const Band &band, const uint32_t *ids_override,
                                 void *ws, const Layout &L, float *rgb, float *T, int32_t *n_contrib, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nt = band.n_tiles();
    static const char *force = getenv("TCGS_K7_BUILD");
    if (producer_heavy(P, band.tiles_x, band.tiles_y) && !ids_override)
        return launch_render_k7_heavy(alpha_mode, early_cull, dump_beta, dump_class, cam, band, ids_override, ws, L,
                                      rgb, T, n_contrib, st);
    const bool few = force && force[0] ? force[0] == 'f' : nt < 4 * sms;
    auto f = few ? launch_render_k7_few : launch_render_k7;
    return f(alpha_mode, early_cull, dump_beta, dump_class, cam, band, ids_override, ws, L, rgb, T, n_contrib, st);
}
cudaError_t launch_pack_lists(int64_t P, const double *mean2d, const double *conic, const double *opacity,
                              const float *colors, const int64_t *offsets, const Band &band, void *ws,
                              const Layout &L, cudaStream_t st);
cudaError_t launch_row_counts(int64_t P, const Band &band, const void *ws, const Layout &L, int64_t *out,
                              cudaStream_t st);
int tile_key_bits(const Band &band);
cudaError_t launch_strip_marks(const uint32_t *src, uint32_t *dst, int64_t n, cudaStream_t st);
// Host-side count of kernels this library has launched (tcgs_launch_count): the bench's gpu_launches.
void note_launch();

// Function attributes (max dynamic smem, carveout) are per device: launchers cache "already set" per device.
constexpr int TCGS_MAX_DEVICES = 64;
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d < 0 ? 0 : (d >= TCGS_MAX_DEVICES ? TCGS_MAX_DEVICES - 1 : d);
}

// ---------------------------------------------------------------- programmatic dependent launch (PDL)
// Every kernel of a frame is launched with programmatic stream serialisation: the next kernel's CTAs are
// scheduled as soon as every CTA of the current one has reached pdl_launch(), so its launch latency and its
// prologue overlap the current kernel's tail.  Each kernel calls pdl_wait() before it touches memory an earlier
// kernel of the stream writes (griddepcontrol.wait returns once the preceding grid has completed and its
// writes are visible; it returns at once for an ordinary launch).  Work before pdl_wait() may only read memory
// no libtcgs kernel writes (the caller's scene arrays).  TCGS_PDL=0 in the environment turns the attribute off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

bool pdl_enabled();
// Set by each entry point from its options: frames in flight on several streams (static K7 schedule) launch
// without PDL -- early-launched dependents would occupy SM slots the other streams' kernels fill better.
extern thread_local bool g_pdl_frame;
inline void pdl_for(const tcgs_opts *o) { g_pdl_frame = !(o && o->schedule == TCGS_SCHEDULE_STATIC); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                            Args &&...args) {
    note_launch();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (pdl_enabled() && g_pdl_frame) ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Exact coverage of a rectangle of at most 64 tiles as a row-major bit mask (bit (ty - y0) w + (tx - x0)):
// K3 builds it once (in depth order) so that K4 expands with popcounts, no float work.  Larger rectangles
// return 0 and K3/K4 walk their rows with cover_row.
constexpr int COVER_MASK_TILES = 64;
__device__ __forceinline__ unsigned long long cover_mask(const CoverRec &c, int x0, int y0, int x1, int y1) {
    const int w = x1 - x0 + 1;
    if (w * (y1 - y0 + 1) > COVER_MASK_TILES) return 0ull;
    unsigned long long m = 0ull;
    for (int ty = y0; ty <= y1; ty++) {
        int lo, hi;
        if (cover_row(c, ty, x0, x1, lo, hi)) {
            const int b0 = (ty - y0) * w + (lo - x0), n = hi - lo + 1;
            m |= (n >= 64 ? ~0ull : ((1ull << n) - 1ull)) << b0;
        }
    }
    return m;
}
// Rows [r0, r1] of a w-wide mask, shifted down so that row r0 becomes row 0.
__device__ __forceinline__ unsigned long long mask_rows(unsigned long long m, int w, int r0, int r1) {
    const int b0 = r0 * w, n = (r1 - r0 + 1) * w;
    m >>= b0;
    return n >= 64 ? m : (m & ((1ull << n) - 1ull));
}

__device__ __forceinline__ float rcp_approx(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

}  // namespace tcgs
