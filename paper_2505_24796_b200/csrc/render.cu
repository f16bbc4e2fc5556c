// render.cu -- K7: tensor-core alpha (Frag2Mat + G2L + EarlyCull) and conditional
// blending, one 16x16 tile per CTA iteration (sm_100a, tcgen05 + TMEM).
//
// Replaces the tile loop of tilesplat.raster.render and blend_tile
// (/root/reference/pkg/src/tilesplat/raster.py:110-146,177-193) with the
// Frag2Mat evaluator (src/tilesplat/tensor_path.py:25-163):
//
//   beta[p, j] = U[p, :] . V[j, :]       (256 pixels x 64 Gaussians per batch)
//
// U holds each pixel's tile-local monomials [1, ux, uy, ux^2, ux*uy, uy^2]
// (G2L: ux, uy in [-8, 7], tile centre origin, src/tilesplat/tensor_path.py:
// 21-22,92-100) -- exact in fp16 and identical for every tile, so it is built
// once per CTA in shared memory.  V holds each Gaussian's coefficients
// (gaussian_vector, tensor_path.py:25-40) pre-scaled by log2(e) and split
// into fp16 hi + lo parts so the K = 16 of tcgen05.mma.kind::f16 carries ~22
// significant bits (TCGS_ALPHA_TC_K8 keeps the paper's length-8 fp16 vector).
// Two MMAs (pixel halves, M = 128 each, N = 64, K = 16) accumulate in fp32 in
// TMEM; each thread (= one pixel = one TMEM lane) reads its 64 betas with
// tcgen05.ld and runs Algorithm 1: EarlyCull (beta < -log2 255 culls without
// an exponential), alpha = ex2(beta), termination test before compositing
// (T - alpha T < 1e-4), C += alpha T c, T -= alpha T.  The CTA retires the
// tile when every in-image pixel has terminated (__syncthreads_or).
//
// Pipeline: double-buffered V stages and TMEM accumulators -- the MMA of
// batch k+1 runs while the threads blend batch k.
#include "tcgs_internal.cuh"

namespace tcgs {

namespace {

constexpr float LOG2E = 1.4426950408889634f;
constexpr float CUT_LOG2 = -7.994353436858858f;  // -log2(255): beta' < CUT culls (tensor_path.py:79-81)
constexpr float TERM_T = 0.0001f;                // src/tilesplat/raster.py:16
constexpr int K7_SMEM_BYTES = 80 * 1024;         // also caps residency at 2 CTAs/SM (TMEM: 2 x 256 columns)

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
};

struct __align__(1024) K7Smem {
    __half U[2][128 * 16];           // A operands: pixel halves, K-major no-swizzle core matrices
    __half V[2][K7_BATCH * 16];      // B operands: one per stage
    float vf[2][K7_BATCH][8];        // FFMA mode coefficients
    float4 col[2][K7_BATCH];         // colours per stage
    unsigned long long bar[2];       // MMA-complete mbarriers, one per stage
    uint32_t tmem_base;
    int tile;
    unsigned long long red[K7_THREADS / 32][4];
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

// kind::f16 instruction descriptor: D f32, A/B f16, K-major both, N = 64, M = 128.
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(K7_BATCH >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);

__device__ __forceinline__ void mbar_init(unsigned long long *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
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

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
        "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Gaussian coefficients for one tile (gaussian_vector, src/tilesplat/tensor_path.py:25-40), relative to the
// tile centre (G2L), scaled by log2 e.  Returns false when no pixel of the tile can pass EarlyCull: then
// sqrt(q(mu - c)) - sqrt(lambda_max(conic)) * 8 sqrt(2) > sqrt(2 (ln o + ln 255)) holds with margin and every
// fragment of this Gaussian in the tile is culled in exact arithmetic (the reference would cull it too).
__device__ __forceinline__ bool gaussian_coeffs(const Rec &r, double ox, double oy, float v[6]) {
    const float dx = (float)(r.mx - ox), dy = (float)(r.my - oy);
    const float s11 = r.s11, s12 = r.s12, s22 = r.s22;
    const float q = s11 * dx * dx + 2.0f * s12 * dx * dy + s22 * dy * dy;
    const float hm = 0.5f * (s11 - s22);
    const float lam = 0.5f * (s11 + s22) + sqrtf(hm * hm + s12 * s12);
    const float gap = sqrtf(fmaxf(q, 0.0f)) - sqrtf(fmaxf(lam, 0.0f)) * 11.3137085f;
    const float need = 2.0f * (r.ln_o + 5.5412635451584258f) + 1.0f;  // 2 (ln o + ln 255) + margin
    if (gap > 0.0f && gap * gap > need) return false;
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

// Write one B-operand row (16 fp16) for MODE: hi/lo split (0) or the paper's K8 vector (1).
template <int MODE>
__device__ __forceinline__ void write_vrow(__half *V, int row, const float v[6], bool live) {
    __align__(16) __half e[16];
    if (!live) {
#pragma unroll
        for (int k = 0; k < 16; k++) e[k] = __float2half_rn(0.0f);
        e[0] = h16(-1000.0f);  // beta' = -1000: culled at every pixel
    } else if (MODE == TCGS_ALPHA_TC_HILO) {
        // v0 = a + b + c + d (four fp16 pieces), v1..v5 = hi + lo
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
    } else {  // TCGS_ALPHA_TC_K8: [v0/3, v0/3, v0/3, v1..v5] in fp16, the rest zero
        const __half third = h16(v[0] / 3.0f);
        e[0] = third;
        e[1] = third;
        e[2] = third;
#pragma unroll
        for (int i = 1; i <= 5; i++) e[2 + i] = h16(v[i]);
#pragma unroll
        for (int k = 8; k < 16; k++) e[k] = h16(0.0f);
    }
    const uint4 *src = reinterpret_cast<const uint4 *>(e);
    *reinterpret_cast<uint4 *>(V + kmaj_off(row, 0)) = src[0];
    *reinterpret_cast<uint4 *>(V + kmaj_off(row, 8)) = src[1];
}

template <int MODE>
__global__ void __launch_bounds__(K7_THREADS, K7_CTAS_PER_SM) render_kernel(RenderArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    K7Smem &sm = *reinterpret_cast<K7Smem *>(smem_raw);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr bool TC = MODE != TCGS_ALPHA_FFMA;

    // pixel owned by this thread: warp w covers an 8x4 block (compact footprints per warp)
    const int lx = 8 * (warp & 1) + (lane & 7);
    const int ly = 4 * (warp >> 1) + (lane >> 3);
    const float ux = (float)(lx - 8), uy = (float)(ly - 8);
    const int half = warp >> 2;               // which M=128 MMA (TMEM column block) holds this pixel
    const int urow = 32 * (warp & 3) + lane;  // TMEM lane == U row within the half

    if (TC) {
        // U: [1, 1, 1, ux, uy, ux^2, ux uy, uy^2, ux, uy, ux^2, ux uy, uy^2, 1, 0, 0]
        const float u[16] = {1.f, 1.f, 1.f, ux, uy, ux * ux, ux * uy, uy * uy, ux, uy, ux * ux, ux * uy, uy * uy, 1.f, 0.f, 0.f};
#pragma unroll
        for (int k = 0; k < 16; k++) sm.U[half][kmaj_off(urow, k)] = __float2half_rn(u[k]);
        if (tid == 0) {
            mbar_init(&sm.bar[0], 1);
            mbar_init(&sm.bar[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        if (warp == 0) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&sm.tmem_base)),
                         "r"(K7_TMEM_COLS));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
        fence_async_smem();
        tc_fence_before();
    }
    __syncthreads();
    if (TC) tc_fence_after();
    const uint32_t tmem = TC ? sm.tmem_base : 0u;
    uint32_t phase = 0;  // bit s: parity of the next completion of bar[s]

    unsigned long long s_blend = 0, s_cull = 0, s_term = 0, s_pairs = 0;
    const uint32_t *ids = a.ids_override ? a.ids_override : (a.ctr->tile_cur ? a.ids1 : a.ids0);

    for (;;) {
        if (tid == 0) sm.tile = (int)atomicAdd(&a.ctr->tile_queue, 1u);
        __syncthreads();
        const int tile = sm.tile;
        if (tile >= a.n_tiles) break;
        const uint2 rg = a.ranges[tile];
        const int n = (int)(rg.y - rg.x);
        const int tx = tile % a.tiles_x, ty = a.band_y0 + tile / a.tiles_x;
        const int px = tx * TILE + lx, py = ty * TILE + ly;
        const bool inside = px < a.width && py < a.height;
        const double ox = tx * TILE + 8.0, oy = ty * TILE + 8.0;  // tile_center (tensor_path.py:21-22)
        bool done = !inside;
        bool term = false;
        float T = 1.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f;
        uint32_t cnt = 0, cull = 0;
        const int nb = (n + K7_BATCH - 1) / K7_BATCH;

        auto build = [&](int kb, int s) {
            if (tid < K7_BATCH) {
                const int j = kb * K7_BATCH + tid;
                float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                bool live = false;
                float4 col = make_float4(0.f, 0.f, 0.f, 0.f);
                if (j < n) {
                    const Rec r = a.rec[ids[rg.x + j]];
                    live = gaussian_coeffs(r, ox, oy, v);
                    col = make_float4(r.r, r.g, r.b, 0.f);
                }
                sm.col[s][tid] = col;
                if (TC) {
                    write_vrow<MODE>(sm.V[s], tid, v, live);
                } else {
                    if (!live) {
                        v[0] = -1000.0f;
                        v[1] = v[2] = v[3] = v[4] = v[5] = 0.0f;
                    }
#pragma unroll
                    for (int i = 0; i < 6; i++) sm.vf[s][tid][i] = v[i];
                }
            }
        };
        auto issue = [&](int s) {
            if (TC && tid == 0) {
                tc_fence_after();
                const uint64_t bdesc = umma_desc(sm.V[s]);
#pragma unroll
                for (int h = 0; h < 2; h++) mma_f16(tmem + s * 128 + h * 64, umma_desc(sm.U[h]), bdesc, IDESC);
                mma_commit(&sm.bar[s]);
            }
        };
        auto wait_mma = [&](int s) {
            if (TC) {
                mbar_wait(&sm.bar[s], (phase >> s) & 1u);
                phase ^= 1u << s;
            }
        };

        if (nb > 0) {
            build(0, 0);
            if (TC) {
                fence_async_smem();
                tc_fence_before();
            }
            __syncthreads();
            issue(0);
            for (int kb = 0; kb < nb; kb++) {
                const int s = kb & 1;
                if (kb + 1 < nb) build(kb + 1, s ^ 1);
                if (TC) {
                    fence_async_smem();
                    tc_fence_before();
                }
                __syncthreads();
                if (kb + 1 < nb) issue(s ^ 1);
                wait_mma(s);
                const int jmax = min(K7_BATCH, n - kb * K7_BATCH);
                float beta[K7_BATCH];
                if (TC) {
                    tc_fence_after();
                    uint32_t r0[32], r1[32];
                    const uint32_t taddr = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + s * 128 + half * 64;
                    tmem_ld32(taddr, r0);
                    tmem_ld32(taddr + 32, r1);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; j++) {
                        asm volatile("" : "+r"(r0[j]));
                        asm volatile("" : "+r"(r1[j]));
                    }
#pragma unroll
                    for (int j = 0; j < 32; j++) {
                        beta[j] = __uint_as_float(r0[j]);
                        beta[32 + j] = __uint_as_float(r1[j]);
                    }
                }
#pragma unroll
                for (int j = 0; j < K7_BATCH; j++) {
                    if (!done && j < jmax) {
                        float b;
                        if (TC) {
                            b = beta[j];
                        } else {
                            const float *v = sm.vf[s][j];
                            b = v[0] + v[1] * ux + v[2] * uy + v[3] * ux * ux + v[4] * ux * uy + v[5] * uy * uy;
                        }
                        if (b >= CUT_LOG2) {
                            const float al = fminf(ex2_approx(b), 1.0f);
                            const float tn = fmaf(-al, T, T);
                            if (tn < TERM_T) {
                                done = true;
                                term = true;
                            } else {
                                const float w = al * T;
                                const float4 cc = sm.col[s][j];
                                c0 = fmaf(w, cc.x, c0);
                                c1 = fmaf(w, cc.y, c1);
                                c2 = fmaf(w, cc.z, c2);
                                T = tn;
                                cnt++;
                            }
                        } else {
                            cull++;
                        }
                    }
                }
                if (TC) tc_fence_before();
                const int alive = __syncthreads_or(!done);
                if (!alive) {
                    if (kb + 1 < nb) wait_mma(s ^ 1);  // drain the MMA already in flight
                    break;
                }
            }
        }
        if (inside) {
            const int64_t p = (int64_t)py * a.width + px;
            a.rgb[3 * p] = c0;
            a.rgb[3 * p + 1] = c1;
            a.rgb[3 * p + 2] = c2;
            a.T[p] = T;
            a.n_contrib[p] = (int32_t)cnt;
            s_pairs += (unsigned long long)n;
        }
        s_blend += cnt;
        s_cull += cull;
        s_term += term ? 1u : 0u;
        __syncthreads();
    }

    // K8: fragment statistics, one atomic per CTA and counter
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s_blend += __shfl_xor_sync(0xffffffffu, s_blend, o);
        s_cull += __shfl_xor_sync(0xffffffffu, s_cull, o);
        s_term += __shfl_xor_sync(0xffffffffu, s_term, o);
        s_pairs += __shfl_xor_sync(0xffffffffu, s_pairs, o);
    }
    if (lane == 0) {
        sm.red[warp][0] = s_blend;
        sm.red[warp][1] = s_cull;
        sm.red[warp][2] = s_term;
        sm.red[warp][3] = s_pairs;
    }
    if (TC) tc_fence_before();
    __syncthreads();
    if (tid < 4) {
        unsigned long long t = 0;
        for (int w = 0; w < K7_THREADS / 32; w++) t += sm.red[w][tid];
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

template <int MODE>
cudaError_t launch_mode(const RenderArgs &a, int num_sms, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(render_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, K7_SMEM_BYTES);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int grid = num_sms * K7_CTAS_PER_SM;
    render_kernel<MODE><<<grid, K7_THREADS, K7_SMEM_BYTES, st>>>(a);
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_render(int alpha_mode, const tcgs_camera &cam, const Band &band, const uint32_t *ids_override,
                          void *ws, const Layout &L, float *rgb, float *T, int32_t *n_contrib, cudaStream_t st) {
    static_assert(sizeof(K7Smem) <= K7_SMEM_BYTES, "K7 shared memory");
    RenderArgs a;
    a.rec = at<Rec>(ws, L.rec);
    a.ids0 = at<uint32_t>(ws, L.tval[0]);
    a.ids1 = at<uint32_t>(ws, L.tval[1]);
    a.ids_override = ids_override;
    a.ranges = at<uint2>(ws, L.ranges);
    a.ctr = at<DevCounters>(ws, L.counters);
    a.tiles_x = band.tiles_x;
    a.band_y0 = band.y0;
    a.n_tiles = band.n_tiles();
    a.width = cam.width;
    a.height = cam.height;
    a.rgb = rgb;
    a.T = T;
    a.n_contrib = n_contrib;
    // per-launch counters: the tile queue and the fragment statistics (f_blend, f_cull, terminated, pairs)
    cudaError_t e = cudaMemsetAsync(&a.ctr->f_blend, 0, 4 * sizeof(unsigned long long), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(&a.ctr->tile_queue, 0, sizeof(unsigned int), st);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    switch (alpha_mode) {
        case TCGS_ALPHA_TC_HILO: return launch_mode<TCGS_ALPHA_TC_HILO>(a, sms, st);
        case TCGS_ALPHA_TC_K8: return launch_mode<TCGS_ALPHA_TC_K8>(a, sms, st);
        case TCGS_ALPHA_FFMA: return launch_mode<TCGS_ALPHA_FFMA>(a, sms, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace tcgs
