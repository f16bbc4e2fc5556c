/* render_c.c -- a C caller of libtcgs.so through include/tcgs.h only (no Python, no torch): the binding a
 * non-Python host of the reference's render path would write.
 *
 *   make -C examples            (gcc; links libtcgs.so and libcudart)
 *   examples/render_c [P] [out.f32]
 *
 * Builds a deterministic scene (an LCG the test suite mirrors in numpy), renders one 256x192 frame with
 * tcgs_render, reads the FragmentStats with tcgs_read_stats, prints them and writes the RGB frame (float32,
 * [H, W, 3]) to out.f32.  tests/test_gpu_parity.py::test_c_example_matches_python renders the same scene
 * through the Python API and requires the two frames to be bit-identical. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "tcgs.h"

static uint32_t lcg_state = 12345u;
static float uni(void) { /* [0, 1): the top 24 bits of a 32-bit LCG */
    lcg_state = lcg_state * 1664525u + 1013904223u;
    return (float)(lcg_state >> 8) * (1.0f / 16777216.0f);
}

#define CHECK_CUDA(x)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) {                                                          \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
            return 2;                                                                     \
        }                                                                                 \
    } while (0)

static void *to_device(const void *h, size_t bytes) {
    void *d = NULL;
    if (cudaMalloc(&d, bytes) != cudaSuccess) return NULL;
    if (cudaMemcpy(d, h, bytes, cudaMemcpyHostToDevice) != cudaSuccess) return NULL;
    return d;
}

int main(int argc, char **argv) {
    const int64_t P = argc > 1 ? atoll(argv[1]) : 5000;
    const char *out = argc > 2 ? argv[2] : NULL;
    const int W = 256, H = 192;
    float *means = malloc(sizeof(float) * 3 * P), *scales = malloc(sizeof(float) * 3 * P);
    float *rots = malloc(sizeof(float) * 4 * P), *opac = malloc(sizeof(float) * P);
    float *rgb = malloc(sizeof(float) * 3 * P);
    for (int64_t i = 0; i < P; i++) {
        const float z = 3.0f + 6.0f * uni();
        means[3 * i + 0] = (2.0f * uni() - 1.0f) * z * 0.5f;
        means[3 * i + 1] = (2.0f * uni() - 1.0f) * z * 0.4f;
        means[3 * i + 2] = z;
        for (int k = 0; k < 3; k++) scales[3 * i + k] = 0.01f + 0.08f * uni();
        float q[4], n = 0.0f;
        for (int k = 0; k < 4; k++) {
            q[k] = uni() - 0.5f;
            n += q[k] * q[k];
        }
        n = sqrtf(n);
        for (int k = 0; k < 4; k++) rots[4 * i + k] = q[k] / n;
        opac[i] = 0.1f + 0.8f * uni();
        for (int k = 0; k < 3; k++) rgb[3 * i + k] = uni();
    }

    int rc = tcgs_device_check();
    if (rc) {
        fprintf(stderr, "tcgs_device_check: %s (%s)\n", tcgs_error_string(rc), tcgs_last_error());
        return 1;
    }
    tcgs_scene scene = {P, -1, TCGS_F32, to_device(means, sizeof(float) * 3 * P), to_device(scales, sizeof(float) * 3 * P),
                        to_device(rots, sizeof(float) * 4 * P), to_device(opac, sizeof(float) * P),
                        to_device(rgb, sizeof(float) * 3 * P)};
    if (!scene.means || !scene.scales || !scene.rotations || !scene.opacities || !scene.features) return 2;
    tcgs_camera cam = {{1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1}, 1.2 * W, 1.2 * W, W / 2.0, H / 2.0, 0.2, W, H};
    /* designated initialisers: fields added to tcgs_opts later default to 0 (the reference's behaviour) */
    tcgs_opts opts = {.alpha_mode = TCGS_ALPHA_TC_HILO, .early_cull = 1, .coverage = TCGS_COVER_SQUARE};

    const int64_t max_splats = 64 * P;
    const size_t ws_bytes = tcgs_workspace_size(P, W, H, max_splats);
    void *ws = NULL;
    float *d_rgb = NULL, *d_T = NULL;
    int32_t *d_cnt = NULL;
    CHECK_CUDA(cudaMalloc(&ws, ws_bytes));
    CHECK_CUDA(cudaMalloc((void **)&d_rgb, sizeof(float) * 3 * W * H));
    CHECK_CUDA(cudaMalloc((void **)&d_T, sizeof(float) * W * H));
    CHECK_CUDA(cudaMalloc((void **)&d_cnt, sizeof(int32_t) * W * H));

    rc = tcgs_render(&scene, &cam, &opts, ws, ws_bytes, max_splats, d_rgb, d_T, d_cnt, NULL);
    if (rc) {
        fprintf(stderr, "tcgs_render: %s (%s)\n", tcgs_error_string(rc), tcgs_last_error());
        return 1;
    }
    tcgs_stats st;
    rc = tcgs_read_stats(ws, P, &opts, &st, NULL); /* synchronises the stream */
    if (rc) {
        fprintf(stderr, "tcgs_read_stats: %s (%s)\n", tcgs_error_string(rc), tcgs_last_error());
        return 1;
    }
    printf("N=%lld f_blend=%lld f_cull=%lld f_skip=%lld exp_calls=%lld dropped=%lld pixels_terminated=%lld\n",
           (long long)st.n_splats, (long long)st.f_blend, (long long)st.f_cull, (long long)st.f_skip,
           (long long)st.exp_calls, (long long)st.dropped, (long long)st.pixels_terminated);
    if (out) {
        float *h = malloc(sizeof(float) * 3 * W * H);
        CHECK_CUDA(cudaMemcpy(h, d_rgb, sizeof(float) * 3 * W * H, cudaMemcpyDeviceToHost));
        FILE *f = fopen(out, "wb");
        if (!f || fwrite(h, sizeof(float), (size_t)3 * W * H, f) != (size_t)3 * W * H) return 3;
        fclose(f);
        free(h);
    }
    return 0;
}
