/*
 * tcgs.h -- C ABI of libtcgs.so, the B200 (sm_100a) TC-GS forward renderer.
 *
 * Drop-in boundary for the reference's render entry point
 *     tilesplat.render(scene, cam, backend) -> (ImageBuffer, FragmentStats)
 *     (/root/reference/pkg/src/tilesplat/raster.py:161-201)
 * whose stages are
 *     project_scene  (src/tilesplat/projection.py:119-134)   -> tcgs_preprocess
 *     build_tiles    (src/tilesplat/tiling.py:46-59)          -> tcgs_bin
 *     per-tile backend.tile_evaluator + blend_tile
 *                    (src/tilesplat/raster.py:102-146,
 *                     src/tilesplat/tensor_path.py:117-194)   -> tcgs_blend
 * and whose per-fragment plugin protocol (evaluator.fragment(j, active),
 * src/tilesplat/raster.py:86-94) is NOT crossed: the whole tile loop runs on
 * the GPU.  tcgs_blend_lists replays caller-given projected records and tile
 * lists through the same blend kernel (debug / KAT entry).
 *
 * Conventions
 *   - every pointer argument marked (device) is CUDA device memory owned by the
 *     caller; the library allocates nothing on the hot path and keeps no
 *     global mutable state except a thread-local last-error string;
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered
 *     and asynchronous except tcgs_read_stats (synchronises `stream`);
 *   - return value 0 = success, negative = error code (tcgs_error_string).
 */
#ifndef TCGS_H_
#define TCGS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCGS_TILE_SIZE 16 /* src/tilesplat/tiling.py:11 */

enum tcgs_status {
    TCGS_OK = 0,
    TCGS_ERR_INVALID_ARG = -1, /* wrapper raises ValueError (src/tilesplat/raster.py:157) */
    TCGS_ERR_CUDA = -2,        /* wrapper raises RuntimeError */
    TCGS_ERR_CAPACITY = -3,    /* splat count exceeded max_splats; tcgs_read_stats reports the need */
    TCGS_ERR_DEVICE = -4,      /* not an sm_100 device */
    TCGS_ERR_WORKSPACE = -5    /* workspace smaller than tcgs_workspace_size() */
};

/* Alpha-evaluation modes: compile-time instantiations of the same blend kernel. */
enum tcgs_alpha_mode {
    TCGS_ALPHA_TC_HILO = 0, /* tcgen05 fp16 K=16: hi/lo split Gaussian vector (default) */
    TCGS_ALPHA_TC_K8 = 1,   /* tcgen05 fp16, the paper's length-8 vector (src/tilesplat/tensor_path.py:25-40) */
    TCGS_ALPHA_FFMA = 2,    /* CUDA-core FP32 quadratic form, no tensor cores (ablation baseline) */
    TCGS_ALPHA_TC_K8_GLOBAL = 3 /* the paper's fp16 length-8 vector in GLOBAL pixel coordinates (no G2L):
                                   tensor_path.py:92-100 with coords="global"; precision ablation only
                                   (x^2 overflows fp16 beyond x = 255) */
};

enum tcgs_dtype { TCGS_F32 = 0, TCGS_F64 = 1 };

/* World-space Gaussians, SoA (src/tilesplat/scene.py:24-47).  All arrays (device). */
typedef struct tcgs_scene {
    int64_t P;
    int32_t sh_degree;     /* -1: `features` holds RGB in [0,1] [P,3] (Gaussian3D.color);
                              0..3: SH coefficients [P,(d+1)^2,3] (3DGS convention) */
    int32_t dtype;         /* enum tcgs_dtype, for every array below */
    const void *means;     /* [P,3] */
    const void *scales;    /* [P,3], activated (> 0) */
    const void *rotations; /* [P,4] unit quaternion (w, x, y, z) */
    const void *opacities; /* [P] in (0, 1] */
    const void *features;  /* [P,3] or [P,(d+1)^2,3] */
} tcgs_scene;

/* Pinhole camera (src/tilesplat/scene.py:50-68). */
typedef struct tcgs_camera {
    double view[16]; /* world -> camera, row-major 4x4; +z forward, +y down */
    double fx, fy, cx, cy;
    double near_plane; /* cull when z <= near (src/tilesplat/projection.py:77) */
    int32_t width, height;
} tcgs_camera;

typedef struct tcgs_opts {
    int32_t tile_row_begin; /* render tile rows [begin, end); end <= 0 means all rows */
    int32_t tile_row_end;
    int32_t alpha_mode;     /* enum tcgs_alpha_mode */
    int32_t early_cull;     /* 1 = EarlyCull: the cull is decided on the exponent before any ex2 and exp_calls
                               = blends + terminations (tensor_path.py:148-154); 0 = EarlyCull off: alpha =
                               exp(beta) for every active fragment, cull on alpha < 1/255 afterwards, exp_calls
                               = every active fragment (raster.py:86-94, tensor_path.py:155-160) */
    int32_t debug;          /* 1: K1 also stores the radius and float64 conic/depth for tcgs_copy_projection */
    int32_t coverage;       /* enum tcgs_coverage (K1's tile rectangle) */
    int32_t defer_colour;   /* 1: tcgs_preprocess computes geometry only; tcgs_colour adds the colours later */
    int32_t schedule;       /* enum tcgs_schedule (how tcgs_blend hands tiles to CTAs) */
    int32_t timing;         /* 1: time each stage with CUDA events on `stream`; the next tcgs_read_stats of this
                               workspace reports them in ms_preprocess / ms_sort / ms_blend
                               (FragmentStats.stage_ms, src/tilesplat/raster.py:196-200) */
    int32_t reserved;
    /* Debug dump (the beta tolerance oracle; NULL = off).  When both are set, tcgs_blend / tcgs_blend_lists /
     * tcgs_render record, for every (tile-list entry e, tile pixel i = 16 row + col) the blend kernel evaluates,
     * dump_beta[e*256 + i] = the exponent in log2 units (beta * log2 e, the value K7 compares and exponentiates)
     * and dump_class[e*256 + i] = 1 cull / 2 blend / 3 terminate / 4 dead: the producer's box test found the
     * Gaussian below the EarlyCull cut on the whole tile (a cull wherever the pixel is still live) / 0 not
     * evaluated (out of the image, or after the pixel terminated).  Both [N][256] (device); the caller
     * initialises them. */
    float *dump_beta;
    uint8_t *dump_class;
} tcgs_opts;

/* K7 tile assignment.  DYNAMIC (default): after its first tile a CTA takes the next from a global queue --
 * the best latency for a frame that has the GPU to itself.  STATIC: CTA b takes tiles b, b + grid, ... -- its
 * staggered tail lets other streams' kernels in, the better choice with several frames in flight. */
enum tcgs_schedule { TCGS_SCHEDULE_DYNAMIC = 0, TCGS_SCHEDULE_STATIC = 1 };

/* Tiles a Gaussian is binned to.  SQUARE is the reference's covered_tiles (src/tilesplat/tiling.py:34-43:
 * the 3-sigma square; parity).  The opt-in modes keep only tiles of that square the
 * alpha >= 1/255 ellipse (grown by a margin) can reach: ELLIPSE_BOX its bounding box, ELLIPSE every tile it
 * intersects (FlashGS-style exact coverage, per tile row).  The splats they drop have no fragment that can
 * pass EarlyCull, so the image is the same while N, f_cull and f_skip shrink.  Pass the same mode to
 * tcgs_preprocess and tcgs_bin. */
enum tcgs_coverage { TCGS_COVER_SQUARE = 0, TCGS_COVER_ELLIPSE_BOX = 1, TCGS_COVER_ELLIPSE = 2 };

/* FragmentStats (src/tilesplat/raster.py:19-49) plus extras. */
typedef struct tcgs_stats {
    int64_t n_splats;          /* N = total tile-list entries (band) */
    int64_t dropped;           /* near-culled Gaussians */
    int64_t f_blend, f_cull, f_skip, exp_calls, pixels_terminated;
    int64_t n_visible;         /* Gaussians touching at least one tile of the band */
    int64_t max_splats_needed; /* == n_splats; > max_splats on TCGS_ERR_CAPACITY */
    float ms_preprocess, ms_sort, ms_blend; /* stage device times of the frame when it ran with opts->timing = 1
                                               (FragmentStats.stage_ms preprocess / sorting / blending), else 0 */
    float reserved;
} tcgs_stats;

/* Bytes of device workspace for P Gaussians, a width x height frame and at most max_splats splats. */
size_t tcgs_workspace_size(int64_t P, int32_t width, int32_t height, int64_t max_splats);

/* K1: EWA projection in float64 + SH colour + tile rectangle per Gaussian
 * (replaces project/project_scene, src/tilesplat/projection.py:68-134). */
int tcgs_preprocess(const tcgs_scene *scene, const tcgs_camera *cam, const tcgs_opts *opts, void *ws,
                    size_t ws_bytes, int64_t max_splats, void *stream);

/* Deferred colour for tile bands: after tcgs_preprocess with opts->defer_colour = 1 (geometry
 * only: no SH read) and the band partition, evaluates the SH colour of every Gaussian whose tile rectangle meets
 * opts' tile-row band -- reading SH coefficients only for those -- with K1's arithmetic, so the frame is the
 * same as with tcgs_preprocess's own colours. */
int tcgs_colour(const tcgs_scene *scene, const tcgs_camera *cam, const tcgs_opts *opts, void *ws, size_t ws_bytes,
                int64_t max_splats, void *stream);

/* K1 for up to TCGS_MAX_VIEWS_PER_PASS cameras of one scene in one pass: each Gaussian's inputs (236 B at
 * SH3) are read once for all of them.  View v's outputs go to workspace ws[v] (each of
 * ws_bytes bytes) exactly as tcgs_preprocess(scene, &cams[v], opts, ws[v], ...) writes them, so tcgs_bin /
 * tcgs_blend then run per view (on any streams ordered after this one).  No reference counterpart: the
 * reference projects per camera (src/tilesplat/projection.py:119-134). */
#define TCGS_MAX_VIEWS_PER_PASS 8
int tcgs_preprocess_views(const tcgs_scene *scene, const tcgs_camera *cams, int32_t n_views, const tcgs_opts *opts,
                          void *const *ws, size_t ws_bytes, int64_t max_splats, void *stream);

/* K2-K6: depth-rank sort, duplicate-with-keys, tile radix sort, tile ranges
 * (replaces build_tiles, src/tilesplat/tiling.py:46-59). */
int tcgs_bin(int64_t P, const tcgs_camera *cam, const tcgs_opts *opts, void *ws, size_t ws_bytes,
             int64_t max_splats, void *stream);

/* K7: tensor-core alpha + conditional blend per tile (replaces the tile loop of
 * render + blend_tile, src/tilesplat/raster.py:110-146,177-193).
 * Outputs (device, full frame, rows outside the band untouched):
 *   rgb [H,W,3] f32, T [H,W] f32 (final transmittance), n_contrib [H,W] i32. */
int tcgs_blend(int64_t P, const tcgs_camera *cam, const tcgs_opts *opts, void *ws, size_t ws_bytes,
               int64_t max_splats, float *rgb, float *T, int32_t *n_contrib, void *stream);

/* K1 + K2-K6 + K7 in one call. */
int tcgs_render(const tcgs_scene *scene, const tcgs_camera *cam, const tcgs_opts *opts, void *ws,
                size_t ws_bytes, int64_t max_splats, float *rgb, float *T, int32_t *n_contrib, void *stream);

/* Synchronises `stream` and reads the frame's FragmentStats. Returns TCGS_ERR_CAPACITY if the
 * frame overflowed max_splats (stats->max_splats_needed then says how many are needed). */
int tcgs_read_stats(const void *ws, int64_t P, const tcgs_opts *opts, tcgs_stats *stats, void *stream);

/* Pipelined frames (no host synchronisation): tcgs_snapshot_stats enqueues a copy of the frame's
 * counters (tcgs_counters_bytes() bytes, at offset 0 of the workspace) to `dst` (pinned host or device
 * memory) on `stream`; once that copy has completed, tcgs_decode_stats turns the snapshot into the
 * same tcgs_stats tcgs_read_stats returns (including TCGS_ERR_CAPACITY). */
size_t tcgs_counters_bytes(void);
int tcgs_snapshot_stats(const void *ws, void *dst, void *stream);
int tcgs_decode_stats(const void *snapshot, const tcgs_opts *opts, tcgs_stats *stats);

/* Tile-band frames written straight into rank 0's frame over NVLink peer memory (multi-GPU; replaces
 * the band gather).  Rank 0 allocates the frame with tcgs_frame_alloc and exports it with
 * tcgs_ipc_get_handle; every other rank maps it with tcgs_ipc_open and passes the mapped pointers as the
 * rgb / T / n_contrib outputs of tcgs_blend, so K7 stores its band's pixels directly into rank 0's HBM. */
#define TCGS_IPC_HANDLE_BYTES 64
int tcgs_frame_alloc(size_t bytes, void **ptr);
int tcgs_frame_free(void *ptr);
int tcgs_ipc_get_handle(void *ptr, void *handle /* TCGS_IPC_HANDLE_BYTES */);
int tcgs_ipc_open(const void *handle, void **ptr);
int tcgs_ipc_close(void *ptr);

/* Debug/KAT entry: blend caller-given projected records through K7.
 *   mean2d [P,2] f64, conic [P,3] f64 (s11,s12,s22), opacity [P] f64, rgb [P,3] f32 (device);
 *   tile lists as CSR: offsets [n_tiles+1] i64, ids [N] i32 (device), row-major tiles. */
int tcgs_blend_lists(int64_t P, const double *mean2d, const double *conic, const double *opacity,
                     const float *colors, const int64_t *offsets, const int32_t *ids, const tcgs_camera *cam,
                     const tcgs_opts *opts, void *ws, size_t ws_bytes, float *rgb, float *T, int32_t *n_contrib,
                     void *stream);

/* Debug: copy the binned splat lists (tile-major Gaussian ids) and per-tile [start,end) ranges
 * out of the workspace (device -> device). ranges has (band tiles) entries of 2 x i32. */
int tcgs_copy_lists(const void *ws, int64_t P, const tcgs_camera *cam, const tcgs_opts *opts,
                    int64_t max_splats, int32_t *ids_out, int32_t *ranges_out, void *stream);

/* Debug: copy per-Gaussian projection results (device -> device): visible u8 [P], mean2d [P,2] f64,
 * conic [P,3] f64, depth [P] f64, radius [P] i32, rgb [P,3] f32.  Needs the frame's tcgs_preprocess to have run
 * with opts->debug = 1 (the float64 buffers are written only then); TCGS_ERR_INVALID_ARG otherwise.
 * Synchronises `stream`. */
int tcgs_copy_projection(const void *ws, int64_t P, const tcgs_camera *cam, int64_t max_splats,
                         uint8_t *visible, double *mean2d, double *conic, double *depth, int32_t *radius,
                         float *rgb, void *stream);

/* Tile-band partition input (multi-GPU, no reference equivalent: the reference renders one frame on one
 * CPU thread, src/tilesplat/raster.py:177-193).  After tcgs_preprocess, writes the number of splats of
 * every tile row of the whole frame into row_counts [tiles_y] i64 (device).  K1 is band-agnostic, so the
 * same preprocess serves any band passed to tcgs_bin / tcgs_blend afterwards. */
int tcgs_tile_row_counts(const void *ws, int64_t P, const tcgs_camera *cam, int64_t max_splats, int64_t *row_counts,
                         void *stream);

/* 0 if the current device is sm_100 (B200); TCGS_ERR_DEVICE otherwise.  Every entry point that launches work
 * runs this check (cached per device) and returns TCGS_ERR_DEVICE on another GPU. */
int tcgs_device_check(void);

/* Number of kernels libtcgs.so has launched so far in this process (all streams, all devices). */
unsigned long long tcgs_launch_count(void);

const char *tcgs_error_string(int code);
const char *tcgs_last_error(void);
int tcgs_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TCGS_H_ */
