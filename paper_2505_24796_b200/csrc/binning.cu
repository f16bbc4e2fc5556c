// binning.cu -- K2-K6: tile binning with the reference's exact order (sm_100a).
//
// Replaces tilesplat.tiling.build_tiles (/root/reference/pkg/src/tilesplat/
// tiling.py:46-59): every tile's list holds the Gaussians whose closed
// bounding square covers it, ascending by float64 depth, ties by index
// (Python's stable sort).  The order is the LSD radix order of the composite
// key (tile, depth, index), produced in two stages so the expensive depth
// digits are sorted on the P Gaussians rather than the N splats:
//
//   K2  depth-rank sort: stable LSD radix (8-bit digits) of the float64 depth
//       bits (minus the visible minimum) carrying the Gaussian index; passes
//       whose digit is constant are detected on the device and skipped;
//   K3  exclusive scan of the tile counts in depth order -> write offsets, N;
//   K4  duplicate-with-keys: emit (tile, id) for every covered tile, in depth
//       order, with a block-cooperative load-balanced expansion (coalesced
//       stores);
//   K5  stable LSD radix sort of the splats on the tile digits only;
//   K6  identify tile ranges [start, end).
//
// Every kernel runs on a fixed grid and reads its item count from device
// memory, so a frame needs no host synchronisation (graph-capturable).
#include "tcgs_internal.cuh"

namespace tcgs {

namespace {

__device__ __forceinline__ int64_t dev_count(const unsigned long long *n_dev, int64_t n_host, int64_t cap) {
    if (!n_dev) return n_host;
    const unsigned long long n = *n_dev;
    return (int64_t)(n < (unsigned long long)cap ? n : (unsigned long long)cap);
}

__device__ __forceinline__ void chunk_of(int64_t n, int nblocks, int b, int64_t &beg, int64_t &end) {
    int64_t c = (n + nblocks - 1) / nblocks;
    c = (c + 31) & ~31ll;
    beg = (int64_t)b * c;
    end = beg + c < n ? beg + c : n;
    if (beg > n) beg = n;
}

// K2 prologue: depth bits -> (bits - min over visible); Gaussians touching no tile get 0
// (they emit nothing, so their position in the depth order is irrelevant).
__global__ void depth_key_fix(unsigned long long *keys, int64_t P, DevCounters *ctr) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    const unsigned long long kmin = ctr->key_min;
    if (i == 0) ctr->key_range = ctr->n_visible ? ctr->key_max - kmin : 0ull;
    const unsigned long long k = keys[i];
    keys[i] = (k == ~0ull) ? 0ull : k - kmin;
}

template <typename KT>
__device__ __forceinline__ const KT *sel(const KT *a, const KT *b, int s) {
    return s ? b : a;
}

// ---------------------------------------------------------------- radix sort
// Upsweep: per-block digit histograms of the block's contiguous chunk.
template <typename KT>
__global__ void __launch_bounds__(SORT_THREADS) radix_upsweep(const KT *keys0, const KT *keys1, const int *cur,
                                                              const unsigned long long *n_dev, int64_t n_host,
                                                              int64_t cap, int shift, const unsigned long long *range,
                                                              uint32_t *hist) {
    __shared__ uint32_t wh[SORT_WARPS][RADIX];
    const int tid = threadIdx.x, warp = tid >> 5;
    const int64_t n = dev_count(n_dev, n_host, cap);
    int64_t beg, end;
    chunk_of(n, gridDim.x, blockIdx.x, beg, end);
    if (range && ((*range) >> shift) == 0) {  // every digit is 0: nothing to count
        for (int d = tid; d < RADIX; d += SORT_THREADS) hist[d * gridDim.x + blockIdx.x] = d == 0 ? (uint32_t)(end - beg) : 0u;
        return;
    }
    for (int d = tid; d < SORT_WARPS * RADIX; d += SORT_THREADS) (&wh[0][0])[d] = 0;
    __syncthreads();
    const KT *keys = sel(keys0, keys1, *cur);
    int64_t i = beg + tid;
    for (; i + 3 * SORT_THREADS < end; i += 4 * SORT_THREADS) {
        KT k[4];
#pragma unroll
        for (int u = 0; u < 4; u++) k[u] = keys[i + u * SORT_THREADS];
#pragma unroll
        for (int u = 0; u < 4; u++) atomicAdd(&wh[warp][(unsigned)(k[u] >> shift) & (RADIX - 1)], 1u);
    }
    for (; i < end; i += SORT_THREADS) atomicAdd(&wh[warp][(unsigned)(keys[i] >> shift) & (RADIX - 1)], 1u);
    __syncthreads();
    for (int d = tid; d < RADIX; d += SORT_THREADS) {
        uint32_t s = 0;
#pragma unroll
        for (int w = 0; w < SORT_WARPS; w++) s += wh[w][d];
        hist[d * gridDim.x + blockIdx.x] = s;
    }
}

// Scan: digit-major exclusive scan of the [RADIX][blocks] histogram table (stable order),
// plus the triviality test (one digit holds every item -> the pass is the identity).
__global__ void __launch_bounds__(1024) radix_scan(uint32_t *hist, int nblocks, const unsigned long long *n_dev,
                                                   int64_t n_host, int64_t cap, int *cur, DevCounters *ctr, int slot) {
    __shared__ uint32_t total[RADIX];
    __shared__ int trivial;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = dev_count(n_dev, n_host, cap);
    if (tid == 0) trivial = 0;
    __syncthreads();
    for (int d = warp; d < RADIX; d += 32) {
        uint32_t run = 0;
        for (int b0 = 0; b0 < nblocks; b0 += 32) {
            const int b = b0 + lane;
            const uint32_t v = b < nblocks ? hist[d * nblocks + b] : 0u;
            uint32_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (b < nblocks) hist[d * nblocks + b] = run + x - v;
            run += __shfl_sync(0xffffffffu, x, 31);
        }
        if (lane == 0) {
            total[d] = run;
            if ((int64_t)run == n) trivial = 1;
        }
    }
    __syncthreads();
    if (n == 0) trivial = 1;
    if (trivial) {
        if (tid == 0) {
            ctr->pass_in[slot] = *cur;
            ctr->pass_do[slot] = 0;
        }
        return;
    }
    if (warp == 0) {  // exclusive scan of the RADIX digit totals (8 per lane)
        uint32_t v[RADIX / 32], s = 0;
#pragma unroll
        for (int k = 0; k < RADIX / 32; k++) {
            v[k] = total[lane * (RADIX / 32) + k];
            s += v[k];
        }
        uint32_t x = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        uint32_t base = x - s;
#pragma unroll
        for (int k = 0; k < RADIX / 32; k++) {
            total[lane * (RADIX / 32) + k] = base;
            base += v[k];
        }
    }
    __syncthreads();
    for (int e = tid; e < RADIX * nblocks; e += blockDim.x) hist[e] += total[e / nblocks];
    if (tid == 0) {
        const int in = *cur;
        ctr->pass_in[slot] = in;
        ctr->pass_do[slot] = 1;
        *cur = in ^ 1;
    }
}

// Downsweep: stable block-local ranking (warp match_any multi-split) and scatter.
template <typename KT>
__global__ void __launch_bounds__(SORT_THREADS) radix_downsweep(KT *keys0, KT *keys1, uint32_t *vals0, uint32_t *vals1,
                                                                const unsigned long long *n_dev, int64_t n_host,
                                                                int64_t cap, int shift, const uint32_t *hist,
                                                                const DevCounters *ctr, int slot) {
    if (!ctr->pass_do[slot]) return;
    __shared__ uint32_t running[RADIX];
    __shared__ uint32_t tot[RADIX];
    __shared__ uint32_t wh[SORT_WARPS][RADIX];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int in = ctr->pass_in[slot];
    const KT *kin = in ? keys1 : keys0;
    KT *kout = in ? keys0 : keys1;
    const uint32_t *vin = in ? vals1 : vals0;
    uint32_t *vout = in ? vals0 : vals1;
    const int64_t n = dev_count(n_dev, n_host, cap);
    int64_t beg, end;
    chunk_of(n, gridDim.x, blockIdx.x, beg, end);
    for (int d = tid; d < RADIX; d += SORT_THREADS) running[d] = hist[d * gridDim.x + blockIdx.x];
    const unsigned lt = lanemask_lt();
    constexpr int SEG = 32 * SORT_IPT;
    for (int64_t tb = beg; tb < end; tb += SORT_THREADS * SORT_IPT) {
        for (int d = lane; d < RADIX; d += 32) wh[warp][d] = 0;
        __syncwarp();
        const int64_t seg = tb + (int64_t)warp * SEG;
        KT k[SORT_IPT];
        uint32_t rank[SORT_IPT];
        int dig[SORT_IPT];
#pragma unroll
        for (int it = 0; it < SORT_IPT; it++) {
            const int64_t idx = seg + it * 32 + lane;
            const bool valid = idx < end;
            k[it] = valid ? kin[idx] : (KT)0;
            dig[it] = valid ? (int)((k[it] >> shift) & (RADIX - 1)) : RADIX;
        }
#pragma unroll
        for (int it = 0; it < SORT_IPT; it++) {
            const int d = dig[it];
            const unsigned peers = __match_any_sync(0xffffffffu, d);
            const unsigned leader = __ffs(peers) - 1;
            uint32_t base = 0;
            if (d < RADIX) base = wh[warp][d];
            __syncwarp();
            if (d < RADIX && lane == (int)leader) wh[warp][d] = base + __popc(peers);
            __syncwarp();
            rank[it] = base + __popc(peers & lt);
        }
        __syncthreads();
        for (int d = tid; d < RADIX; d += SORT_THREADS) {
            uint32_t s = 0;
#pragma unroll
            for (int w = 0; w < SORT_WARPS; w++) {
                const uint32_t v = wh[w][d];
                wh[w][d] = s;
                s += v;
            }
            tot[d] = s;
        }
        __syncthreads();
#pragma unroll
        for (int it = 0; it < SORT_IPT; it++) {
            const int d = dig[it];
            if (d < RADIX) {
                const int64_t idx = seg + it * 32 + lane;
                const uint32_t pos = running[d] + wh[warp][d] + rank[it];
                kout[pos] = k[it];
                vout[pos] = vin[idx];
            }
        }
        __syncthreads();
        for (int d = tid; d < RADIX; d += SORT_THREADS) running[d] += tot[d];
        __syncthreads();
    }
}

template <typename KT>
void radix_sort(KT *k0, KT *k1, uint32_t *v0, uint32_t *v1, int *cur, const unsigned long long *n_dev, int64_t n_host,
                int64_t cap, int bits, int first_slot, const unsigned long long *range, uint32_t *hist,
                DevCounters *ctr, cudaStream_t st) {
    const int passes = (bits + RADIX_BITS - 1) / RADIX_BITS;
    for (int p = 0; p < passes; p++) {
        const int shift = p * RADIX_BITS;
        radix_upsweep<KT><<<SORT_BLOCKS, SORT_THREADS, 0, st>>>(k0, k1, cur, n_dev, n_host, cap, shift, range, hist);
        radix_scan<<<1, 1024, 0, st>>>(hist, SORT_BLOCKS, n_dev, n_host, cap, cur, ctr, first_slot + p);
        radix_downsweep<KT><<<SORT_BLOCKS, SORT_THREADS, 0, st>>>(k0, k1, v0, v1, n_dev, n_host, cap, shift, hist, ctr,
                                                                   first_slot + p);
    }
}

// ---------------------------------------------------------------- K3 / K4
// Per-block sums of the tile counts, taken in depth order.
__global__ void __launch_bounds__(SCAN_THREADS) count_upsweep(const uint32_t *idx0, const uint32_t *idx1,
                                                              const DevCounters *ctr, const uint32_t *touched,
                                                              int64_t P, unsigned long long *blocksum) {
    const uint32_t *order = ctr->depth_cur ? idx1 : idx0;
    int64_t beg, end;
    chunk_of(P, gridDim.x, blockIdx.x, beg, end);
    unsigned long long s = 0;
    for (int64_t i = beg + threadIdx.x; i < end; i += SCAN_THREADS) s += touched[order[i]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ unsigned long long ws[SCAN_THREADS / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < SCAN_THREADS / 32; w++) t += ws[w];
        blocksum[blockIdx.x] = t;
    }
}

__global__ void count_scan(unsigned long long *blocksum, int nblocks, DevCounters *ctr, int64_t cap) {
    if (threadIdx.x != 0) return;
    unsigned long long run = 0;
    for (int b = 0; b < nblocks; b++) {
        const unsigned long long v = blocksum[b];
        blocksum[b] = run;
        run += v;
    }
    ctr->n_splats = run;
    ctr->overflow = run > (unsigned long long)cap ? 1ull : 0ull;
    ctr->tile_cur = 0;
}

// K4: duplicate-with-keys.  Each block walks its chunk 256 Gaussians at a time, scans their
// counts, then expands the (Gaussian, covered tile) pairs cooperatively: consecutive threads
// write consecutive splats (binary search of the slot in the shared scan).
__global__ void __launch_bounds__(SCAN_THREADS) duplicate_keys(const uint32_t *idx0, const uint32_t *idx1,
                                                               const DevCounters *ctr, const uint32_t *touched,
                                                               const short4 *rect, int64_t P,
                                                               const unsigned long long *blockoff, int tiles_x,
                                                               int band_y0, int64_t cap, uint32_t *tkey,
                                                               uint32_t *tval) {
    __shared__ uint32_t incl[SCAN_THREADS];
    __shared__ uint32_t gid[SCAN_THREADS];
    __shared__ short4 rc[SCAN_THREADS];
    __shared__ uint32_t wsum[SCAN_THREADS / 32];
    const uint32_t *order = ctr->depth_cur ? idx1 : idx0;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int64_t beg, end;
    chunk_of(P, gridDim.x, blockIdx.x, beg, end);
    unsigned long long base = blockoff[blockIdx.x];
    for (int64_t tb = beg; tb < end; tb += SCAN_THREADS) {
        const int64_t i = tb + tid;
        uint32_t c = 0, g = 0;
        short4 r = make_short4(0, 0, -1, -1);
        if (i < end) {
            g = order[i];
            c = touched[g];
            if (c) r = rect[g];
        }
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        uint32_t wpre = 0, total = 0;
#pragma unroll
        for (int w = 0; w < SCAN_THREADS / 32; w++) {
            const uint32_t s = wsum[w];
            if (w < warp) wpre += s;
            total += s;
        }
        incl[tid] = wpre + x;
        gid[tid] = g;
        rc[tid] = r;
        __syncthreads();
        for (uint32_t s = tid; s < total; s += SCAN_THREADS) {
            int lo = 0, hi = SCAN_THREADS - 1;  // first item with incl > s
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (incl[mid] > s) hi = mid;
                else lo = mid + 1;
            }
            const uint32_t k = s - (lo ? incl[lo - 1] : 0u);
            const short4 q = rc[lo];
            const int w = q.z - q.x + 1;
            const int ty = q.y + (int)(k / w), tx = q.x + (int)(k % w);
            const unsigned long long pos = base + s;
            if (pos < (unsigned long long)cap) {
                tkey[pos] = (uint32_t)((ty - band_y0) * tiles_x + tx);
                tval[pos] = gid[lo];
            }
        }
        base += total;
        __syncthreads();
    }
}

// K6: tile ranges from the sorted keys.
__global__ void tile_ranges(const uint32_t *k0, const uint32_t *k1, const DevCounters *ctr, int64_t cap, uint2 *ranges) {
    const uint32_t *keys = ctr->tile_cur ? k1 : k0;
    const unsigned long long nn = ctr->n_splats;
    const int64_t n = (int64_t)(nn < (unsigned long long)cap ? nn : (unsigned long long)cap);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t t = keys[i];
        if (i == 0 || keys[i - 1] != t) ranges[t].x = (uint32_t)i;
        if (i == n - 1 || keys[i + 1] != t) ranges[t].y = (uint32_t)(i + 1);
    }
}

// Debug / KAT entry: pack caller-given projected records and CSR offsets.
__global__ void pack_records(int64_t P, const double *mean2d, const double *conic, const double *opacity,
                             const float *colors, Rec *rec) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    Rec r;
    r.mx = mean2d[2 * i];
    r.my = mean2d[2 * i + 1];
    r.s11 = (float)conic[3 * i];
    r.s12 = (float)conic[3 * i + 1];
    r.s22 = (float)conic[3 * i + 2];
    r.ln_o = (float)log(opacity[i]);
    r.opacity = (float)opacity[i];
    r.r = colors[3 * i];
    r.g = colors[3 * i + 1];
    r.b = colors[3 * i + 2];
    rec[i] = r;
}

__global__ void pack_ranges(const int64_t *offsets, int band_tile0, int n_tiles, uint2 *ranges) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    ranges[t] = make_uint2((uint32_t)offsets[band_tile0 + t], (uint32_t)offsets[band_tile0 + t + 1]);
}

}  // namespace

int tile_key_bits(const Band &band) {
    const int nt = band.n_tiles();
    int bits = 1;
    while ((1 << bits) < nt) bits++;
    return bits;
}

cudaError_t launch_bin(int64_t P, const Band &band, void *ws, const Layout &L, int64_t cap, cudaStream_t st) {
    DevCounters *ctr = at<DevCounters>(ws, L.counters);
    uint32_t *hist = at<uint32_t>(ws, L.hist);
    unsigned long long *k0 = at<unsigned long long>(ws, L.key64[0]);
    unsigned long long *k1 = at<unsigned long long>(ws, L.key64[1]);
    uint32_t *i0 = at<uint32_t>(ws, L.idx[0]);
    uint32_t *i1 = at<uint32_t>(ws, L.idx[1]);
    uint32_t *tk0 = at<uint32_t>(ws, L.tkey[0]);
    uint32_t *tk1 = at<uint32_t>(ws, L.tkey[1]);
    uint32_t *tv0 = at<uint32_t>(ws, L.tval[0]);
    uint32_t *tv1 = at<uint32_t>(ws, L.tval[1]);
    unsigned long long *blocksum = at<unsigned long long>(ws, L.blocksum);
    uint2 *ranges = at<uint2>(ws, L.ranges);
    cudaError_t e = cudaMemsetAsync(ranges, 0, sizeof(uint2) * (size_t)(band.n_tiles() ? band.n_tiles() : 1), st);
    if (e != cudaSuccess) return e;
    if (P > 0) {
        depth_key_fix<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(k0, P, ctr);
        // K2: key_range = max - min bounds every fixed key, so passes above its top bit are skipped
        radix_sort<unsigned long long>(k0, k1, i0, i1, &ctr->depth_cur, nullptr, P, P, 64, 0, &ctr->key_range, hist,
                                       ctr, st);
    }
    // K3
    count_upsweep<<<SCAN_BLOCKS, SCAN_THREADS, 0, st>>>(i0, i1, ctr, at<uint32_t>(ws, L.touched), P, blocksum);
    count_scan<<<1, 32, 0, st>>>(blocksum, SCAN_BLOCKS, ctr, cap);
    // K4
    duplicate_keys<<<SCAN_BLOCKS, SCAN_THREADS, 0, st>>>(i0, i1, ctr, at<uint32_t>(ws, L.touched),
                                                          at<short4>(ws, L.rect), P, blocksum, band.tiles_x, band.y0,
                                                          cap, tk0, tv0);
    // K5
    radix_sort<uint32_t>(tk0, tk1, tv0, tv1, &ctr->tile_cur, &ctr->n_splats, 0, cap, tile_key_bits(band),
                         TILE_PASS_SLOT, nullptr, hist, ctr, st);
    // K6
    tile_ranges<<<4 * 148, 256, 0, st>>>(tk0, tk1, ctr, cap, ranges);
    return cudaGetLastError();
}

cudaError_t launch_pack_lists(int64_t P, const double *mean2d, const double *conic, const double *opacity,
                              const float *colors, const int64_t *offsets, const Band &band, void *ws,
                              const Layout &L, cudaStream_t st) {
    if (P > 0)
        pack_records<<<(unsigned)((P + 255) / 256), 256, 0, st>>>(P, mean2d, conic, opacity, colors, at<Rec>(ws, L.rec));
    const int nt = band.n_tiles();
    if (nt > 0)
        pack_ranges<<<(nt + 255) / 256, 256, 0, st>>>(offsets, band.y0 * band.tiles_x, nt, at<uint2>(ws, L.ranges));
    return cudaGetLastError();
}

}  // namespace tcgs
