// abi.cu -- the extern "C" boundary of libtcgs.so (include/tcgs.h).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <mutex>
#include <unordered_map>

#include "tcgs_internal.cuh"

using namespace tcgs;

static std::atomic<unsigned long long> g_launches{0};
void tcgs::note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

thread_local bool tcgs::g_pdl_frame = true;

bool tcgs::pdl_enabled() {
    static const bool on = [] {
        const char *v = getenv("TCGS_PDL");
        return !(v && v[0] == '0');
    }();
    return on;
}

extern "C" int tcgs_device_check(void);

namespace {

thread_local char g_last_error[512] = "";

int fail(int code, const char *msg) {
    snprintf(g_last_error, sizeof(g_last_error), "%s", msg);
    return code;
}

int cuda_fail(cudaError_t e, const char *where) {
    snprintf(g_last_error, sizeof(g_last_error), "%s: %s", where, cudaGetErrorString(e));
    return TCGS_ERR_CUDA;
}

// (PDL: the dependent K1 may be scheduled before this kernel's wait -- it computes from the caller's scene and
// waits itself before writing the workspace, which orders it after this kernel and, through it, after the
// previous frame's K7)
__global__ void init_counters(DevCounters *c, int debug) {
    pdl_launch();
    pdl_wait();
    DevCounters z;
    memset(&z, 0, sizeof(z));
    z.key_min = ~0ull;
    z.debug_written = debug;
    *c = z;
}

struct CounterSet {
    DevCounters *c[TCGS_MAX_VIEWS_PER_PASS];
};
__global__ void init_counters_views(const __grid_constant__ CounterSet s, int n, int debug) {
    pdl_launch();
    pdl_wait();
    if ((int)threadIdx.x < n) {
        DevCounters z;
        memset(&z, 0, sizeof(z));
        z.key_min = ~0ull;
        z.debug_written = debug;
        *s.c[threadIdx.x] = z;
    }
}

// sm_100 check, cached per device (every launching entry point runs it)
int device_ok() {
    static std::atomic<int> cache[TCGS_MAX_DEVICES];  // 0 unknown, 1 ok, -1 not sm_100
    const int d = current_device();
    int v = cache[d].load(std::memory_order_relaxed);
    if (v == 0) {
        v = tcgs_device_check() == TCGS_OK ? 1 : -1;
        cache[d].store(v, std::memory_order_relaxed);
    }
    if (v < 0) return fail(TCGS_ERR_DEVICE, "libtcgs.so is built for sm_100a (B200); the current device is not sm_100");
    return TCGS_OK;
}

// ---- stage timing (opts->timing): CUDA events per workspace, read back by tcgs_read_stats
enum { ST_PRE = 0, ST_SORT = 1, ST_BLEND = 2 };
struct StageTimer {
    cudaEvent_t ev[3][2] = {};
    bool recorded[3] = {false, false, false};
};
std::mutex g_timer_mu;
std::unordered_map<const void *, StageTimer> g_timers;

void time_mark(const tcgs_opts *opts, const void *ws, int stage, int end, cudaStream_t st) {
    if (!opts || !opts->timing) return;
    std::lock_guard<std::mutex> lk(g_timer_mu);
    StageTimer &t = g_timers[ws];
    cudaEvent_t &e = t.ev[stage][end];
    if (!e && cudaEventCreate(&e) != cudaSuccess) {
        e = nullptr;
        return;
    }
    cudaEventRecord(e, st);
    if (end) t.recorded[stage] = true;
}

// after the stream has been synchronised: the stage times recorded since the last read (0 if none)
void time_read(const void *ws, tcgs_stats *stats) {
    std::lock_guard<std::mutex> lk(g_timer_mu);
    auto it = g_timers.find(ws);
    if (it == g_timers.end()) return;
    float *dst[3] = {&stats->ms_preprocess, &stats->ms_sort, &stats->ms_blend};
    for (int s = 0; s < 3; s++) {
        if (!it->second.recorded[s]) continue;
        float ms = 0.0f;
        if (cudaEventElapsedTime(&ms, it->second.ev[s][0], it->second.ev[s][1]) == cudaSuccess) *dst[s] = ms;
        it->second.recorded[s] = false;
    }
}

int check_scene(const tcgs_scene *scene) {
    if (!scene) return fail(TCGS_ERR_INVALID_ARG, "null scene");
    if (scene->sh_degree < -1 || scene->sh_degree > 3) return fail(TCGS_ERR_INVALID_ARG, "sh_degree must be -1..3");
    if (scene->dtype != TCGS_F32 && scene->dtype != TCGS_F64) return fail(TCGS_ERR_INVALID_ARG, "dtype");
    if (scene->P > 0 && (!scene->means || !scene->scales || !scene->rotations || !scene->opacities || !scene->features))
        return fail(TCGS_ERR_INVALID_ARG, "null scene array");
    return TCGS_OK;
}

int check_common(const tcgs_camera *cam, const tcgs_opts *opts, void *ws, size_t ws_bytes, int64_t P,
                 int64_t max_splats, bool device = true) {
    if (!cam || !ws) return fail(TCGS_ERR_INVALID_ARG, "null camera or workspace");
    if (cam->width <= 0 || cam->height <= 0) return fail(TCGS_ERR_INVALID_ARG, "image dimensions must be positive");
    if (!(cam->fx > 0) || !(cam->fy > 0)) return fail(TCGS_ERR_INVALID_ARG, "focal lengths must be positive");
    if (!(cam->near_plane > 0)) return fail(TCGS_ERR_INVALID_ARG, "near clip must be positive");
    if (P < 0 || P >= (int64_t)1 << 32) return fail(TCGS_ERR_INVALID_ARG, "P out of range");
    if (max_splats < 1 || max_splats >= (int64_t)1 << 32) return fail(TCGS_ERR_INVALID_ARG, "max_splats out of range");
    const int tx = (cam->width + TILE - 1) / TILE, ty = (cam->height + TILE - 1) / TILE;
    if (tx > 32767 || ty > 32767) return fail(TCGS_ERR_INVALID_ARG, "image too large");
    if (opts) {
        if (opts->alpha_mode < 0 || opts->alpha_mode > TCGS_ALPHA_TC_K8_GLOBAL)
            return fail(TCGS_ERR_INVALID_ARG, "unknown alpha mode");
        if (opts->coverage < TCGS_COVER_SQUARE || opts->coverage > TCGS_COVER_ELLIPSE)
            return fail(TCGS_ERR_INVALID_ARG, "unknown coverage mode");
        if (opts->schedule != TCGS_SCHEDULE_DYNAMIC && opts->schedule != TCGS_SCHEDULE_STATIC)
            return fail(TCGS_ERR_INVALID_ARG, "unknown tile schedule");
        if (opts->tile_row_end > 0 && (opts->tile_row_begin < 0 || opts->tile_row_begin >= opts->tile_row_end ||
                                       opts->tile_row_end > ty))
            return fail(TCGS_ERR_INVALID_ARG, "invalid tile-row band");
        if ((opts->dump_beta == nullptr) != (opts->dump_class == nullptr))
            return fail(TCGS_ERR_INVALID_ARG, "dump_beta and dump_class must both be set or both be NULL");
    }
    if (ws_bytes < Layout::make(P, cam->width, cam->height, max_splats).total)
        return fail(TCGS_ERR_WORKSPACE, "workspace smaller than tcgs_workspace_size()");
    return device ? device_ok() : TCGS_OK;
}

}  // namespace

extern "C" {

int tcgs_version(void) { return 1; }

unsigned long long tcgs_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

const char *tcgs_last_error(void) { return g_last_error; }

const char *tcgs_error_string(int code) {
    switch (code) {
        case TCGS_OK: return "ok";
        case TCGS_ERR_INVALID_ARG: return "invalid argument";
        case TCGS_ERR_CUDA: return "CUDA error";
        case TCGS_ERR_CAPACITY: return "splat capacity exceeded";
        case TCGS_ERR_DEVICE: return "unsupported device (sm_100a required)";
        case TCGS_ERR_WORKSPACE: return "workspace too small";
        default: return "unknown error";
    }
}

int tcgs_device_check(void) {
    int dev = 0, major = 0, minor = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0) {
        snprintf(g_last_error, sizeof(g_last_error), "libtcgs.so is built for sm_100a; device is sm_%d%d", major, minor);
        return TCGS_ERR_DEVICE;
    }
    return TCGS_OK;
}

size_t tcgs_workspace_size(int64_t P, int32_t width, int32_t height, int64_t max_splats) {
    return Layout::make(P, width, height, max_splats).total;
}

int tcgs_preprocess(const tcgs_scene *scene, const tcgs_camera *cam, const tcgs_opts *opts, void *ws,
                    size_t ws_bytes, int64_t max_splats, void *stream) {
    pdl_for(opts);
    int rc = check_scene(scene);
    if (rc) return rc;
    rc = check_common(cam, opts, ws, ws_bytes, scene->P, max_splats);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const Layout L = Layout::make(scene->P, cam->width, cam->height, max_splats);
    time_mark(opts, ws, ST_PRE, 0, st);
    cudaError_t e = launch_k(init_counters, 1, 1, 0, st, at<DevCounters>(ws, L.counters), opts ? opts->debug : 0);
    if (e != cudaSuccess) return cuda_fail(e, "init_counters");
    e = launch_preprocess(*scene, *cam, make_band(*cam, opts), opts ? opts->debug : 0,
                                      opts ? opts->coverage : 0, opts ? opts->defer_colour : 0, ws, L, st);
    if (e != cudaSuccess) return cuda_fail(e, "preprocess");
    time_mark(opts, ws, ST_PRE, 1, st);
    return TCGS_OK;
}

int tcgs_colour(const tcgs_scene *scene, const tcgs_camera *cam, const tcgs_opts *opts, void *ws, size_t ws_bytes,
                int64_t max_splats, void *stream) {
    pdl_for(opts);
    int rc = check_scene(scene);
    if (rc) return rc;
    rc = check_common(cam, opts, ws, ws_bytes, scene->P, max_splats);
    if (rc) return rc;
    const Layout L = Layout::make(scene->P, cam->width, cam->height, max_splats);
    cudaError_t e = launch_colour(*scene, *cam, make_band(*cam, opts), ws, L, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "colour");
    return TCGS_OK;
}

int tcgs_preprocess_views(const tcgs_scene *scene, const tcgs_camera *cams, int32_t n_views, const tcgs_opts *opts,
                          void *const *ws, size_t ws_bytes, int64_t max_splats, void *stream) {
    pdl_for(opts);
    int rc = check_scene(scene);
    if (rc) return rc;
    if (!cams || !ws) return fail(TCGS_ERR_INVALID_ARG, "null cameras or workspaces");
    if (n_views < 1 || n_views > TCGS_MAX_VIEWS_PER_PASS)
        return fail(TCGS_ERR_INVALID_ARG, "n_views must be 1..TCGS_MAX_VIEWS_PER_PASS");
    Layout L[TCGS_MAX_VIEWS_PER_PASS];
    Band bands[TCGS_MAX_VIEWS_PER_PASS];
    CounterSet cs;
    for (int v = 0; v < n_views; v++) {
        rc = check_common(&cams[v], opts, ws[v], ws_bytes, scene->P, max_splats, false);
        if (rc) return rc;
        for (int u = 0; u < v; u++)
            if (ws[u] == ws[v]) return fail(TCGS_ERR_INVALID_ARG, "views need distinct workspaces");
        L[v] = Layout::make(scene->P, cams[v].width, cams[v].height, max_splats);
        bands[v] = make_band(cams[v], opts);
        cs.c[v] = at<DevCounters>(ws[v], L[v].counters);
    }
    if ((rc = device_ok())) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = launch_k(init_counters_views, 1, 32, 0, st, cs, n_views, opts ? opts->debug : 0);
    if (e != cudaSuccess) return cuda_fail(e, "init_counters_views");
    e = launch_preprocess_views(*scene, cams, bands, n_views, opts ? opts->debug : 0,
                                            opts ? opts->coverage : 0, opts ? opts->defer_colour : 0, ws, L, st);
    if (e != cudaSuccess) return cuda_fail(e, "preprocess_views");
    return TCGS_OK;
}

int tcgs_bin(int64_t P, const tcgs_camera *cam, const tcgs_opts *opts, void *ws, size_t ws_bytes,
             int64_t max_splats, void *stream) {
    pdl_for(opts);
    int rc = check_common(cam, opts, ws, ws_bytes, P, max_splats);
    if (rc) return rc;
    const Layout L = Layout::make(P, cam->width, cam->height, max_splats);
    time_mark(opts, ws, ST_SORT, 0, (cudaStream_t)stream);
    const Band band = make_band(*cam, opts);
    // compacted live lists cull whole (Gaussian, tile) entries before K7: part of EarlyCull (with it off, or in the
    // global-coordinate ablation, K7 evaluates every entry as the reference does); not with the debug dump
    const bool compact = producer_heavy(P, band.tiles_x, band.tiles_y) && !(opts && opts->dump_beta) &&
                         (!opts || (opts->early_cull && opts->alpha_mode != TCGS_ALPHA_TC_K8_GLOBAL));
    cudaError_t e = launch_bin(P, band, ws, L, max_splats, (cudaStream_t)stream, compact);
    if (e != cudaSuccess) return cuda_fail(e, "bin");
    time_mark(opts, ws, ST_SORT, 1, (cudaStream_t)stream);
    return TCGS_OK;
}

int tcgs_blend(int64_t P, const tcgs_camera *cam, const tcgs_opts *opts, void *ws, size_t ws_bytes,
               int64_t max_splats, float *rgb, float *T, int32_t *n_contrib, void *stream) {
    pdl_for(opts);
    int rc = check_common(cam, opts, ws, ws_bytes, P, max_splats);
    if (rc) return rc;
    if (!rgb || !T || !n_contrib) return fail(TCGS_ERR_INVALID_ARG, "null output");
    const Layout L = Layout::make(P, cam->width, cam->height, max_splats);
    time_mark(opts, ws, ST_BLEND, 0, (cudaStream_t)stream);
    cudaError_t e = launch_render(P, opts ? opts->alpha_mode : 0, opts ? opts->early_cull : 1,
                                  opts ? opts->dump_beta : nullptr, opts ? opts->dump_class : nullptr, *cam,
                                  make_band(*cam, opts), nullptr, ws, L, rgb, T, n_contrib, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "render");
    time_mark(opts, ws, ST_BLEND, 1, (cudaStream_t)stream);
    return TCGS_OK;
}

int tcgs_render(const tcgs_scene *scene, const tcgs_camera *cam, const tcgs_opts *opts, void *ws, size_t ws_bytes,
                int64_t max_splats, float *rgb, float *T, int32_t *n_contrib, void *stream) {
    int rc = tcgs_preprocess(scene, cam, opts, ws, ws_bytes, max_splats, stream);
    if (rc) return rc;
    rc = tcgs_bin(scene->P, cam, opts, ws, ws_bytes, max_splats, stream);
    if (rc) return rc;
    return tcgs_blend(scene->P, cam, opts, ws, ws_bytes, max_splats, rgb, T, n_contrib, stream);
}

namespace {
int decode_stats(const DevCounters &c, const tcgs_opts *opts, tcgs_stats *stats) {
    memset(stats, 0, sizeof(*stats));
    stats->n_splats = (int64_t)c.n_splats;
    stats->max_splats_needed = (int64_t)c.n_splats;
    stats->dropped = (int64_t)c.dropped;
    stats->n_visible = (int64_t)c.n_visible;
    stats->f_blend = (int64_t)c.f_blend;
    stats->f_cull = (int64_t)c.f_cull;
    stats->pixels_terminated = (int64_t)c.pixels_terminated;
    // every in-image (pixel, splat) pair is exactly one of blend / cull / skip (src/tilesplat/raster.py:124-145)
    stats->f_skip = (int64_t)c.pairs - stats->f_blend - stats->f_cull;
    const int early = opts ? opts->early_cull : 1;
    stats->exp_calls = early ? stats->f_blend + stats->pixels_terminated
                             : stats->f_blend + stats->f_cull + stats->pixels_terminated;
    if (c.overflow) return fail(TCGS_ERR_CAPACITY, "splat count exceeded max_splats");
    return TCGS_OK;
}
}  // namespace

int tcgs_read_stats(const void *ws, int64_t P, const tcgs_opts *opts, tcgs_stats *stats, void *stream) {
    if (!ws || !stats) return fail(TCGS_ERR_INVALID_ARG, "null workspace or stats");
    (void)P;
    DevCounters c;
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(&c, ws, sizeof(c), cudaMemcpyDeviceToHost, st);  // counters sit at offset 0
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "read_stats");
    const int rc = decode_stats(c, opts, stats);
    time_read(ws, stats);
    return rc;
}

size_t tcgs_counters_bytes(void) { return sizeof(DevCounters); }

int tcgs_frame_alloc(size_t bytes, void **ptr) {
    if (!ptr || bytes == 0) return fail(TCGS_ERR_INVALID_ARG, "null pointer or zero size");
    cudaError_t e = cudaMalloc(ptr, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "frame_alloc");
    return TCGS_OK;
}

int tcgs_frame_free(void *ptr) {
    cudaError_t e = cudaFree(ptr);
    if (e != cudaSuccess) return cuda_fail(e, "frame_free");
    return TCGS_OK;
}

int tcgs_ipc_get_handle(void *ptr, void *handle) {
    if (!ptr || !handle) return fail(TCGS_ERR_INVALID_ARG, "null pointer");
    static_assert(sizeof(cudaIpcMemHandle_t) == TCGS_IPC_HANDLE_BYTES, "IPC handle size");
    cudaError_t e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t *>(handle), ptr);
    if (e != cudaSuccess) return cuda_fail(e, "ipc_get_handle");
    return TCGS_OK;
}

int tcgs_ipc_open(const void *handle, void **ptr) {
    if (!ptr || !handle) return fail(TCGS_ERR_INVALID_ARG, "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "ipc_open");
    return TCGS_OK;
}

int tcgs_ipc_close(void *ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(ptr);
    if (e != cudaSuccess) return cuda_fail(e, "ipc_close");
    return TCGS_OK;
}

int tcgs_snapshot_stats(const void *ws, void *dst, void *stream) {
    if (!ws || !dst) return fail(TCGS_ERR_INVALID_ARG, "null workspace or destination");
    cudaError_t e = cudaMemcpyAsync(dst, ws, sizeof(DevCounters), cudaMemcpyDefault, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "snapshot_stats");
    return TCGS_OK;
}

int tcgs_decode_stats(const void *snapshot, const tcgs_opts *opts, tcgs_stats *stats) {
    if (!snapshot || !stats) return fail(TCGS_ERR_INVALID_ARG, "null snapshot or stats");
    DevCounters c;
    memcpy(&c, snapshot, sizeof(c));
    return decode_stats(c, opts, stats);
}

int tcgs_blend_lists(int64_t P, const double *mean2d, const double *conic, const double *opacity, const float *colors,
                     const int64_t *offsets, const int32_t *ids, const tcgs_camera *cam, const tcgs_opts *opts,
                     void *ws, size_t ws_bytes, float *rgb, float *T, int32_t *n_contrib, void *stream) {
    pdl_for(opts);
    int rc = check_common(cam, opts, ws, ws_bytes, P, 1);
    if (rc) return rc;
    if (P > 0 && (!mean2d || !conic || !opacity || !colors)) return fail(TCGS_ERR_INVALID_ARG, "null records");
    if (!offsets || !rgb || !T || !n_contrib) return fail(TCGS_ERR_INVALID_ARG, "null list/output");
    cudaStream_t st = (cudaStream_t)stream;
    const Layout L = Layout::make(P, cam->width, cam->height, 1);
    const Band band = make_band(*cam, opts);
    cudaError_t e = launch_k(init_counters, 1, 1, 0, st, at<DevCounters>(ws, L.counters), 0);
    if (e != cudaSuccess) return cuda_fail(e, "init_counters");
    e = launch_pack_lists(P, mean2d, conic, opacity, colors, offsets, band, ws, L, st);
    if (e != cudaSuccess) return cuda_fail(e, "pack_lists");
    e = launch_render(P, opts ? opts->alpha_mode : 0, opts ? opts->early_cull : 1, opts ? opts->dump_beta : nullptr,
                      opts ? opts->dump_class : nullptr, *cam, band, reinterpret_cast<const uint32_t *>(ids), ws, L,
                      rgb, T, n_contrib, st);
    if (e != cudaSuccess) return cuda_fail(e, "render");
    return TCGS_OK;
}

int tcgs_copy_lists(const void *ws, int64_t P, const tcgs_camera *cam, const tcgs_opts *opts, int64_t max_splats,
                    int32_t *ids_out, int32_t *ranges_out, void *stream) {
    if (!ws || !cam || !ids_out || !ranges_out) return fail(TCGS_ERR_INVALID_ARG, "null argument");
    if (int rc = device_ok()) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    const Layout L = Layout::make(P, cam->width, cam->height, max_splats);
    DevCounters c;
    cudaError_t e = cudaMemcpyAsync(&c, ws, sizeof(c), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "copy_lists");
    const int64_t n = (int64_t)c.n_splats < max_splats ? (int64_t)c.n_splats : max_splats;
    const uint32_t *src = at<uint32_t>(ws, c.tile_cur ? L.tval[1] : L.tval[0]);
    if (n > 0) e = launch_strip_marks(src, reinterpret_cast<uint32_t *>(ids_out), n, st);  // (K4's dead marks)
    const Band band = make_band(*cam, opts);
    if (e == cudaSuccess && band.n_tiles() > 0)
        e = cudaMemcpyAsync(ranges_out, at<uint2>(ws, L.ranges), sizeof(uint2) * (size_t)band.n_tiles(),
                            cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "copy_lists");
    return TCGS_OK;
}

int tcgs_tile_row_counts(const void *ws, int64_t P, const tcgs_camera *cam, int64_t max_splats, int64_t *row_counts,
                         void *stream) {
    if (!ws || !cam || !row_counts) return fail(TCGS_ERR_INVALID_ARG, "null argument");
    if (cam->width <= 0 || cam->height <= 0) return fail(TCGS_ERR_INVALID_ARG, "image dimensions must be positive");
    if (int rc = device_ok()) return rc;
    const Layout L = Layout::make(P, cam->width, cam->height, max_splats);
    cudaError_t e = launch_row_counts(P, make_band(*cam, nullptr), ws, L, row_counts, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "tile_row_counts");
    return TCGS_OK;
}

}  // extern "C"

namespace {
__global__ void copy_projection_kernel(int64_t P, const int32_t *radius, const Rec *rec, const double *dconic,
                                       const double *ddepth, const double *dmean2d, uint8_t *visible, double *mean2d, double *conic,
                                       double *depth, int32_t *rad_out, float *rgb) {
    pdl_wait();
    pdl_launch();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    const int32_t r = radius[i];
    visible[i] = r >= 0;
    rad_out[i] = r;
    conic[3 * i] = dconic[3 * i];
    conic[3 * i + 1] = dconic[3 * i + 1];
    conic[3 * i + 2] = dconic[3 * i + 2];
    depth[i] = ddepth[i];
    const Rec q = rec[i];  // colour is only defined for Gaussians that touch a tile
    mean2d[2 * i] = dmean2d[2 * i];
    mean2d[2 * i + 1] = dmean2d[2 * i + 1];
    rgb[3 * i] = q.r;
    rgb[3 * i + 1] = q.g;
    rgb[3 * i + 2] = q.b;
}
}  // namespace

extern "C" int tcgs_copy_projection(const void *ws, int64_t P, const tcgs_camera *cam, int64_t max_splats,
                                    uint8_t *visible, double *mean2d, double *conic, double *depth, int32_t *radius,
                                    float *rgb, void *stream) {
    if (!ws || !cam || !visible || !mean2d || !conic || !depth || !radius || !rgb)
        return fail(TCGS_ERR_INVALID_ARG, "null argument");
    if (int rc = device_ok()) return rc;
    if (P <= 0) return TCGS_OK;
    const Layout L = Layout::make(P, cam->width, cam->height, max_splats);
    cudaStream_t st = (cudaStream_t)stream;
    DevCounters c;
    cudaError_t e0 = cudaMemcpyAsync(&c, ws, sizeof(c), cudaMemcpyDeviceToHost, st);
    if (e0 == cudaSuccess) e0 = cudaStreamSynchronize(st);
    if (e0 != cudaSuccess) return cuda_fail(e0, "copy_projection");
    if (!c.debug_written)
        return fail(TCGS_ERR_INVALID_ARG, "tcgs_copy_projection needs the frame preprocessed with opts->debug = 1");
    cudaError_t e = launch_k(copy_projection_kernel, (unsigned)((P + 255) / 256), 256, 0, st,
        P, at<int32_t>(ws, L.radius), at<Rec>(ws, L.rec), at<double>(ws, L.dbg_conic), at<double>(ws, L.dbg_depth),
        at<double>(ws, L.dbg_mean2d), visible, mean2d, conic, depth, radius, rgb);
    if (e != cudaSuccess) return cuda_fail(e, "copy_projection");
    return TCGS_OK;
}
