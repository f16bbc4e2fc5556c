// binning.cu -- K2-K6: tile binning with the reference's exact order (sm_100a).
//
// Replaces tilesplat.tiling.build_tiles (/root/reference/pkg/src/tilesplat/
// tiling.py:46-59): every tile's list holds the Gaussians whose closed
// bounding square covers it, ascending by float64 depth, ties by index
// (Python's stable sort).  That is the LSD radix order of the composite key
// (tile, depth, index), produced in two stages so that the wide depth digits
// are sorted on the P Gaussians rather than on the N splats:
//
//   K2  depth-rank sort: stable LSD radix (8-bit digits) of the float64 depth
//       bits minus the visible minimum, carrying the Gaussian index; passes
//       above the key range or with a single digit value are skipped on the
//       device (the digit histograms of all passes come from one read, fused
//       with the key rebase);
//   K3  exclusive scan of the tile counts in depth order -> write offsets, N;
//   K4  duplicate-with-keys: emit (tile, id) for every covered tile in depth
//       order with a CTA-cooperative, load-balanced expansion (coalesced
//       stores), histogramming the tile digits for K5 on the fly;
//   K5  stable LSD radix sort of the splats on the tile digits only (16-bit
//       keys when the band has <= 65536 tiles);
//   K6  tile ranges [start, end) from the sorted keys.
//
// Every radix pass is reduce-then-scan: per-tile digit histograms, a
// per-digit row scan over the tiles (which also yields the digit totals),
// and a downsweep with a ballot-based warp multi-split for the stable local
// rank and a shared-memory staged scatter so the global stores are coalesced
// runs.  For the depth key, the digit histograms of all passes come from one
// read fused with the key rebase, so passes above the key range or with a
// single digit value exit at entry.  All counts live on the device: a frame needs no
// host synchronisation (graph-capturable).
#include <algorithm>

#ifndef TCGS_DUP_SMALL
#define TCGS_DUP_SMALL 32  // K4: rectangles of more tiles than this are expanded by the whole warp
#endif
#ifndef TCGS_TILE_DIGITS_EVEN
#define TCGS_TILE_DIGITS_EVEN 0  // tile-key radix: 1 = equal digit widths per pass (measured: no gain over 8-bit)
#endif

#include "tcgs_internal.cuh"

#ifndef TCGS_ONESWEEP
#define TCGS_ONESWEEP 0  // 1: single-kernel passes with decoupled look-back (measured slower, r2f: 276 vs 251 us)
#endif

namespace tcgs {

namespace {

__device__ __forceinline__ int64_t dev_count(const unsigned long long *n_dev, int64_t n_host, int64_t cap) {
    if (!n_dev) return n_host;
    const unsigned long long n = *n_dev;
    return (int64_t)(n < (unsigned long long)cap ? n : (unsigned long long)cap);
}

__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t *warp_tmp, uint32_t *total) {
    // exclusive scan over the 256 threads of the CTA (blockDim.x == 256)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tmp[warp] = x;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; w++) {
        const uint32_t s = warp_tmp[w];
        pre += w < warp ? s : 0u;
        tot += s;
    }
    if (total) *total = tot;
    __syncthreads();
    return pre + x - v;
}

#ifndef TCGS_MATCH
#define TCGS_MATCH 0
#endif
// Lanes of the warp holding the same digit (invalid items: digit >= RADIX match only each other).  Nine ballots:
// MATCH.ANY has the higher throughput in isolation (B200: 1.9 vs 13.3 ns per warp-wide peer mask per SM,
// scripts/micro/match_vs_ballot.cu) but its latency sits on the downsweep's serial rank chain -- with it the
// binning took 297 instead of 251 us (r2g).  TCGS_MATCH=1 selects it.
template <int DB = RADIX_BITS>  // digit bits (<= RADIX_BITS); invalid items carry d = RADIX
__device__ __forceinline__ unsigned warp_peers(int d) {
    if (TCGS_MATCH) return __match_any_sync(0xffffffffu, d);
    unsigned peers = __ballot_sync(0xffffffffu, d < RADIX);
    if (d >= RADIX) peers = ~peers;
#pragma unroll
    for (int b = 0; b < DB; b++) {
        const bool bit = (d >> b) & 1;
        const unsigned m = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? m : ~m;
    }
    return peers;
}

// ---------------------------------------------------------------- K2 prologue
// The float64 depth bits minus the visible minimum span up to ~55 bits (depths 2..20: exponents 1..4).
// They are radix-sorted on a 24-bit prefix only (3 passes instead of 7): key = (bits - min) >> shift with
// shift chosen so every visible key is <= DEPTH_KEY_MAX - 1; Gaussians touching no tile get DEPTH_KEY_MAX
// and sort last (they emit nothing).  Equal prefixes whose full keys differ are put in float64 order by
// depth_fixup afterwards (stable: ties keep the index order, tiling.py:55-58).
constexpr uint32_t DEPTH_KEY_BITS = 24;
constexpr uint32_t DEPTH_KEY_MAX = (1u << DEPTH_KEY_BITS) - 1u;
constexpr int DEPTH_PASSES = 3;

__device__ __forceinline__ int depth_shift(unsigned long long range) {
    if (range < (unsigned long long)DEPTH_KEY_MAX) return 0;
    return (64 - __clzll((long long)range)) - (int)(DEPTH_KEY_BITS - 1);  // range >> shift < 2^23
}

__global__ void __launch_bounds__(256) depth_fix_hist(const unsigned long long *src, uint32_t *keys, uint32_t *idx,
                                                      int64_t P, DevCounters *ctr, SortState *ss, OsHeader *hdr,
                                                      uint32_t *table0, int64_t T0) {
    pdl_wait();
    pdl_launch();
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // a new look-back epoch for this binning's radix passes
        hdr->magic = OS_MAGIC;
        hdr->epoch = hdr->epoch + 1u;
    }
    // pass 0: the digit counts of this CTA's radix tile (that pass's upsweep table column); every pass: the digit
    // range, which plans the passes (a pass with a single digit value is the identity)
    __shared__ uint32_t h0[RADIX];
    __shared__ uint32_t rng[DEPTH_PASSES][2];  // (255 - min digit, max digit)
    h0[threadIdx.x] = 0;
    if (threadIdx.x < DEPTH_PASSES * 2) (&rng[0][0])[threadIdx.x] = 0;
    __syncthreads();
    const unsigned long long kmin = ctr->key_min;
    const unsigned long long range = ctr->n_visible ? ctr->key_max - kmin : 0ull;
    const int shift = depth_shift(range);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        ctr->key_range = DEPTH_KEY_MAX;  // the prefix keys span [0, DEPTH_KEY_MAX]
        ctr->depth_shift = shift;
    }
    // one CTA per radix tile of the first pass (OS_THREADS x DEPTH_IPT keys): its pass-0 digit counts are that
    // pass's upsweep table column, so the pass runs without an upsweep
    const int64_t t0 = (int64_t)blockIdx.x * (OS_THREADS * DEPTH_IPT);
    const int64_t t1 = t0 + OS_THREADS * DEPTH_IPT < P ? t0 + OS_THREADS * DEPTH_IPT : P;
    uint32_t dlo[DEPTH_PASSES], dhi[DEPTH_PASSES];
#pragma unroll
    for (int p = 0; p < DEPTH_PASSES; p++) {
        dlo[p] = RADIX - 1;
        dhi[p] = 0;
    }
    for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
        const unsigned long long k = src[i];  // K1's output stays intact: tcgs_bin can run again (other bands)
        const uint32_t key = (k == ~0ull) ? DEPTH_KEY_MAX : (uint32_t)((k - kmin) >> shift);
        keys[i] = key;
        idx[i] = (uint32_t)i;
        atomicAdd(&h0[key & (RADIX - 1)], 1u);
#pragma unroll
        for (int p = 0; p < DEPTH_PASSES; p++) {
            const uint32_t d = (key >> (RADIX_BITS * p)) & (RADIX - 1);
            dlo[p] = d < dlo[p] ? d : dlo[p];
            dhi[p] = d > dhi[p] ? d : dhi[p];
        }
    }
#pragma unroll
    for (int p = 0; p < DEPTH_PASSES; p++) {
        const uint32_t lo = __reduce_min_sync(0xffffffffu, dlo[p]), hi = __reduce_max_sync(0xffffffffu, dhi[p]);
        if ((threadIdx.x & 31) == 0 && t0 + (threadIdx.x & ~31) < t1) {  // (warps with keys)
            atomicMax(&rng[p][0], RADIX - 1 - lo);
            atomicMax(&rng[p][1], hi);
        }
    }
    __syncthreads();
    if (threadIdx.x < DEPTH_PASSES * 2) atomicMax(&(&ss->drange[0][0])[threadIdx.x], (&rng[0][0])[threadIdx.x]);
    if (TCGS_ONESWEEP) {  // single-kernel passes take their digit totals from here
        __syncthreads();
        for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
            const uint32_t key = keys[i];
#pragma unroll
            for (int p = 0; p < DEPTH_PASSES; p++)
                atomicAdd(&ss->ghist[p][(key >> (RADIX_BITS * p)) & (RADIX - 1)], 1u);
        }
    }
    static_assert(OS_THREADS == RADIX, "one digit per thread");
    if (table0) table0[(int64_t)threadIdx.x * T0 + blockIdx.x] = h0[threadIdx.x];
    // the last CTA to finish plans the passes (no separate planning launch): a pass whose digit is
    // the same for every key is the identity and is skipped
    __shared__ int last, trivial;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&ss->done_ctas, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    int cur = 0;
    for (int p = 0; p < DEPTH_PASSES; p++) {
        if (threadIdx.x == 0)
            trivial = (P == 0 || RADIX - 1 - __ldcg(&ss->drange[p][0]) == __ldcg(&ss->drange[p][1])) ? 1 : 0;
        __syncthreads();
        const int triv = trivial;
        if (threadIdx.x == 0) {
            ss->pass_in[p] = cur;
            ss->pass_do[p] = triv ? 0 : 1;
        }
        if (!triv) cur ^= 1;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        ss->final_buf = cur;
        ctr->depth_cur = cur;
    }
}

// ---------------------------------------------------------------- K2 fix-up
// After the prefix sort, a run of equal prefixes is in index order; put it in (float64 depth, index)
// order.  Runs of <= FIX_SHORT: one thread, insertion sort (stable).  Longer runs go to depth_fixup_long.
constexpr int FIX_SHORT = 32;
constexpr int FIX_SMEM = 4096;

__global__ void __launch_bounds__(256) depth_fixup(const uint32_t *k0, const uint32_t *k1, uint32_t *i0, uint32_t *i1,
                                                   const unsigned long long *src, int64_t P, DevCounters *ctr,
                                                   uint32_t *long_runs) {
    pdl_wait();
    pdl_launch();
    if (ctr->depth_shift == 0) return;  // the prefix is the whole key
    const uint32_t *key = ctr->depth_cur ? k1 : k0;
    uint32_t *idx = ctr->depth_cur ? i1 : i0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = key[i];
        if (k == DEPTH_KEY_MAX) continue;
        if (i > 0 && key[i - 1] == k) continue;
        if (i + 1 >= P || key[i + 1] != k) continue;
        int64_t e = i + 2;
        while (e < P && key[e] == k && e - i <= FIX_SHORT) e++;
        if (e - i > FIX_SHORT) {
            const unsigned slot = atomicAdd(&ctr->n_long_runs, 1u);
            if (slot < (unsigned)FIX_SMEM) long_runs[slot] = (uint32_t)i;
            continue;
        }
        const int n = (int)(e - i);
        uint32_t g[FIX_SHORT];
        unsigned long long f[FIX_SHORT];
        bool moved = false;
        for (int j = 0; j < n; j++) {
            const uint32_t gj = idx[i + j];
            const unsigned long long fj = src[gj];
            int m = j - 1;
            while (m >= 0 && f[m] > fj) {  // strict: equal depths keep the index order
                f[m + 1] = f[m];
                g[m + 1] = g[m];
                m--;
                moved = true;
            }
            f[m + 1] = fj;
            g[m + 1] = gj;
        }
        if (moved)
            for (int j = 0; j < n; j++) idx[i + j] = g[j];
    }
}

// Long runs (rare: > FIX_SHORT Gaussians whose float64 depths share the 24-bit prefix): one CTA per run,
// bitonic sort of (depth bits, index) pairs -- in shared memory up to FIX_SMEM elements, otherwise in place
// over the run with a global-memory scratch of the same length.
__device__ __forceinline__ bool pair_less(unsigned long long fa, uint32_t ga, unsigned long long fb, uint32_t gb) {
    return fa < fb || (fa == fb && ga < gb);
}

__global__ void __launch_bounds__(256) depth_fixup_long(const uint32_t *k0, const uint32_t *k1, uint32_t *i0,
                                                        uint32_t *i1, const unsigned long long *src, int64_t P,
                                                        DevCounters *ctr, const uint32_t *long_runs,
                                                        unsigned long long *gscratch) {
    pdl_wait();
    pdl_launch();
    __shared__ unsigned long long sf[FIX_SMEM];
    __shared__ uint32_t sg[FIX_SMEM];
    const unsigned nruns = ctr->n_long_runs;
    if (ctr->depth_shift == 0 || nruns == 0) return;
    const uint32_t *key = ctr->depth_cur ? k1 : k0;
    uint32_t *idx = ctr->depth_cur ? i1 : i0;
    for (unsigned r = blockIdx.x; r < nruns; r += gridDim.x) {
        int64_t s;
        if (nruns <= (unsigned)FIX_SMEM) {
            s = long_runs[r];
        } else {  // the list overflowed: recover run starts by scanning (r-th run start of the array)
            if (r > 0) break;
            s = -1;
        }
        // process either the listed run, or (overflow) every long run sequentially in this CTA
        for (int64_t i = (s >= 0 ? s : 0); i < P;) {
            const uint32_t k = key[i];
            int64_t e = i + 1;
            while (e < P && key[e] == k) e++;
            const int64_t n = e - i;
            const bool do_it = k != DEPTH_KEY_MAX && n > FIX_SHORT && (s >= 0 || (i == 0 || key[i - 1] != k));
            if (do_it) {
                int64_t n2 = 1;
                while (n2 < n) n2 <<= 1;
                const bool sm = n2 <= FIX_SMEM;
                unsigned long long *F = sm ? sf : gscratch;
                uint32_t *G = sm ? sg : reinterpret_cast<uint32_t *>(gscratch + 2 * P);
                for (int64_t j = threadIdx.x; j < n2; j += blockDim.x) {
                    const uint32_t gj = j < n ? idx[i + j] : 0xffffffffu;
                    F[j] = j < n ? src[gj] : ~0ull;
                    G[j] = gj;
                }
                __syncthreads();
                for (int64_t kk = 2; kk <= n2; kk <<= 1) {
                    for (int64_t jj = kk >> 1; jj > 0; jj >>= 1) {
                        for (int64_t t = threadIdx.x; t < n2; t += blockDim.x) {
                            const int64_t u = t ^ jj;
                            if (u > t) {
                                const bool up = (t & kk) == 0;
                                const bool lt = pair_less(F[u], G[u], F[t], G[t]);
                                if (up == lt) {
                                    const unsigned long long tf = F[t];
                                    F[t] = F[u];
                                    F[u] = tf;
                                    const uint32_t tg = G[t];
                                    G[t] = G[u];
                                    G[u] = tg;
                                }
                            }
                        }
                        __syncthreads();
                    }
                }
                for (int64_t j = threadIdx.x; j < n; j += blockDim.x) idx[i + j] = G[j];
                __syncthreads();
            }
            if (s >= 0) break;
            i = e;
        }
    }
}

// One stable LSD radix pass = three kernels with no inter-CTA chain:
//   radix_upsweep   per-tile digit histograms -> table[digit][tile]
//   radix_rowscan   one CTA per digit: exclusive scan of its row over the tiles, digit total
//   radix_downsweep stable local rank (ballot multi-split), global position =
//                   digit base (scan of the totals) + row prefix + local rank, scatter staged
//                   through shared memory
//                   so the stores are coalesced runs.
template <typename KT, int IPT, int DB>
__global__ void __launch_bounds__(OS_THREADS) radix_upsweep(const KT *k0, const KT *k1, const unsigned long long *n_dev,
                                                            int64_t n_host, int64_t cap, int pass, int shift,
                                                            const SortState *ss, uint32_t *table, int64_t T) {
    pdl_wait();
    pdl_launch();
    if (!ss->pass_do[pass]) return;
    constexpr int TILE_ITEMS = OS_THREADS * IPT;
    __shared__ uint32_t wh[OS_WARPS][RADIX];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = dev_count(n_dev, n_host, cap);
    const int64_t tile = blockIdx.x;
    if (tile * TILE_ITEMS >= n) return;
    for (int e = lane; e < RADIX; e += 32) wh[warp][e] = 0;
    __syncwarp();
    const KT *kin = ss->pass_in[pass] ? k1 : k0;
    const int64_t seg = tile * TILE_ITEMS + (int64_t)warp * 32 * IPT;
    KT k[IPT];
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        const int64_t idx = seg + it * 32 + lane;
        k[it] = idx < n ? kin[idx] : (KT)0;
    }
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        const int64_t idx = seg + it * 32 + lane;
        if (idx < n) atomicAdd(&wh[warp][(unsigned)(k[it] >> shift) & ((1u << DB) - 1u)], 1u);
    }
    __syncthreads();
    const int d = tid;
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < OS_WARPS; w++) t += wh[w][d];
    table[(int64_t)d * T + tile] = t;
}

template <int IPT>
__global__ void __launch_bounds__(256) radix_rowscan(const unsigned long long *n_dev, int64_t n_host, int64_t cap,
                                                     int pass, SortState *ss, uint32_t *table, int64_t T) {
    pdl_wait();
    pdl_launch();
    if (!ss->pass_do[pass]) return;
    constexpr int TILE_ITEMS = OS_THREADS * IPT;
    __shared__ uint32_t wt[8];
    const int64_t n = dev_count(n_dev, n_host, cap);
    const int64_t ntiles = (n + TILE_ITEMS - 1) / TILE_ITEMS;
    uint32_t *row = table + (int64_t)blockIdx.x * T;
    uint32_t carry = 0;
    for (int64_t c0 = 0; c0 < ntiles; c0 += 256 * 8) {
        uint32_t v[8], s = 0;
        const int64_t b = c0 + threadIdx.x * 8;
#pragma unroll
        for (int u = 0; u < 8; u++) {
            v[u] = b + u < ntiles ? row[b + u] : 0u;
            s += v[u];
        }
        uint32_t tot;
        uint32_t ex = carry + block_excl_scan256(s, wt, &tot);
#pragma unroll
        for (int u = 0; u < 8; u++) {
            if (b + u < ntiles) row[b + u] = ex;
            ex += v[u];
        }
        carry += tot;
    }
    if (threadIdx.x == 0) ss->ghist[pass][blockIdx.x] = carry;  // digit total
}

template <typename KT, int IPT, int DB>  // DB digit bits: digits >= 1 << DB stay empty
#ifndef TCGS_DOWNSWEEP_CTAS
#define TCGS_DOWNSWEEP_CTAS 3  // resident downsweep CTAs per SM the register allocation must allow
#endif
__global__ void __launch_bounds__(OS_THREADS, TCGS_DOWNSWEEP_CTAS) radix_downsweep(KT *k0, KT *k1, uint32_t *v0, uint32_t *v1,
                                                              const unsigned long long *n_dev, int64_t n_host,
                                                              int64_t cap, int pass, int shift, const SortState *ss,
                                                              const uint32_t *table, int64_t T) {
    pdl_wait();
    pdl_launch();
    if (!ss->pass_do[pass]) return;
    constexpr int TILE_ITEMS = OS_THREADS * IPT;
    extern __shared__ __align__(16) unsigned char os_smem[];
    KT *skey = reinterpret_cast<KT *>(os_smem);
    uint32_t *sval = reinterpret_cast<uint32_t *>(os_smem + sizeof(KT) * TILE_ITEMS);
    __shared__ uint32_t wh[OS_WARPS][RADIX];
    __shared__ uint32_t loc[RADIX], gofs[RADIX], wt[8];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = dev_count(n_dev, n_host, cap);
    const int64_t tile = blockIdx.x;
    if (tile * TILE_ITEMS >= n) return;
    for (int e = lane; e < RADIX; e += 32) wh[warp][e] = 0;
    const int in = ss->pass_in[pass];
    const KT *kin = in ? k1 : k0;
    KT *kout = in ? k0 : k1;
    const uint32_t *vin = in ? v1 : v0;
    uint32_t *vout = in ? v0 : v1;
    const int64_t base = tile * TILE_ITEMS;
    const int tile_n = (int)(n - base < TILE_ITEMS ? n - base : TILE_ITEMS);
    const int64_t seg = base + (int64_t)warp * 32 * IPT;
    const uint32_t dtot = ss->ghist[pass][tid];
    const uint32_t rowpre = table[(int64_t)tid * T + tile];

    KT k[IPT];
    uint32_t val[IPT];
    uint32_t dr[IPT];  // digit (bits 16..24, RADIX = invalid) | rank within the warp's digit (bits 0..15)
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        const int64_t idx = seg + it * 32 + lane;
        const bool valid = idx < n;
        k[it] = valid ? kin[idx] : (KT)0;
        val[it] = valid ? vin[idx] : 0u;
    }
    __syncwarp();
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        const bool valid = seg + it * 32 + lane < n;
        const int d = valid ? (int)((k[it] >> shift) & ((1u << DB) - 1u)) : RADIX;
        const unsigned peers = warp_peers<DB>(d);
        uint32_t b = 0;
        if (d < RADIX) b = wh[warp][d];
        __syncwarp();
        if (d < RADIX && lane == (int)(__ffs(peers) - 1)) wh[warp][d] = b + __popc(peers);
        __syncwarp();
        dr[it] = ((uint32_t)d << 16) | (b + __popc(peers & lt));
    }
    __syncthreads();
    const int d = tid;
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < OS_WARPS; w++) {
        const uint32_t v = wh[w][d];
        wh[w][d] = total;
        total += v;
    }
    const uint32_t lo = block_excl_scan256(total, wt, nullptr);  // (contains __syncthreads)
    const uint32_t dbase = block_excl_scan256(dtot, wt, nullptr);
    loc[d] = lo;
    gofs[d] = dbase + rowpre - lo;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        const uint32_t dd = dr[it] >> 16;
        if (dd < RADIX) {
            const uint32_t lp = loc[dd] + wh[warp][dd] + (dr[it] & 0xffffu);
            skey[lp] = k[it];
            sval[lp] = val[it];
        }
    }
    __syncthreads();
    for (int i = tid; i < tile_n; i += OS_THREADS) {
        const KT key = skey[i];
        const uint32_t pos = gofs[(unsigned)(key >> shift) & ((1u << DB) - 1u)] + (uint32_t)i;
        kout[pos] = key;
        vout[pos] = sval[i];
    }
}

// ---------------------------------------------------------------- onesweep pass (decoupled look-back)
// One kernel per stable LSD radix pass: a CTA claims the next radix tile (atomic counter: tiles are claimed in
// launch order, so every earlier tile is being processed and the look-back always progresses), ranks its items
// locally (ballot multi-split, as the downsweep), publishes its per-digit counts, looks back over the earlier
// tiles' published counts (inclusive prefixes stop the walk) to get its global offset per digit, and scatters
// through shared memory.  Digit totals come from one histogram computed before the pass (depth_fix_hist for
// the depth key, duplicate_keys for the tile key), so no separate upsweep / row-scan kernels run.
constexpr uint64_t OS_FLAG_AGG = 1ull << 30, OS_FLAG_INC = 2ull << 30, OS_COUNT = (1ull << 30) - 1;

__device__ __forceinline__ void os_store(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t os_load(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <typename KT, int IPT, int DB>
__global__ void __launch_bounds__(OS_THREADS, 3) radix_onesweep(KT *k0, KT *k1, uint32_t *v0, uint32_t *v1,
                                                              const unsigned long long *n_dev, int64_t n_host,
                                                              int64_t cap, int pass, int shift, SortState *ss,
                                                              uint64_t *look, const OsHeader *hdr) {
    pdl_wait();
    pdl_launch();
    if (!ss->pass_do[pass]) return;
    constexpr int TILE_ITEMS = OS_THREADS * IPT;
    extern __shared__ __align__(16) unsigned char os_smem[];
    KT *skey = reinterpret_cast<KT *>(os_smem);
    uint32_t *sval = reinterpret_cast<uint32_t *>(os_smem + sizeof(KT) * TILE_ITEMS);
    __shared__ uint32_t wh[OS_WARPS][RADIX];
    __shared__ uint32_t loc[RADIX], gofs[RADIX], wt[8];
    __shared__ int s_tile;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t n = dev_count(n_dev, n_host, cap);
    const int64_t ntiles = (n + TILE_ITEMS - 1) / TILE_ITEMS;
    if (tid == 0) s_tile = (int)atomicAdd(&ss->tile_ctr[pass], 1u);
    for (int e = lane; e < RADIX; e += 32) wh[warp][e] = 0;
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) return;
    const uint64_t epoch = (uint64_t)hdr->epoch << 32;
    const int in = ss->pass_in[pass];
    const KT *kin = in ? k1 : k0;
    KT *kout = in ? k0 : k1;
    const uint32_t *vin = in ? v1 : v0;
    uint32_t *vout = in ? v0 : v1;
    const int64_t base = tile * TILE_ITEMS;
    const int tile_n = (int)(n - base < TILE_ITEMS ? n - base : TILE_ITEMS);
    const int64_t seg = base + (int64_t)warp * 32 * IPT;
    const uint32_t dtot = ss->ghist[pass][tid];

    KT k[IPT];
    uint32_t val[IPT];
    uint32_t dr[IPT];  // digit (bits 16..24, RADIX = invalid) | rank within the warp's digit (bits 0..15)
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        const int64_t idx = seg + it * 32 + lane;
        const bool valid = idx < n;
        k[it] = valid ? kin[idx] : (KT)0;
        val[it] = valid ? vin[idx] : 0u;
    }
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        const bool valid = seg + it * 32 + lane < n;
        const int d = valid ? (int)((k[it] >> shift) & ((1u << DB) - 1u)) : RADIX;
        const unsigned peers = warp_peers<DB>(d);
        uint32_t b = 0;
        if (d < RADIX) b = wh[warp][d];
        __syncwarp();
        if (d < RADIX && lane == (int)(__ffs(peers) - 1)) wh[warp][d] = b + __popc(peers);
        __syncwarp();
        dr[it] = ((uint32_t)d << 16) | (b + __popc(peers & lt));
    }
    __syncthreads();
    const int d = tid;
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < OS_WARPS; w++) {
        const uint32_t v = wh[w][d];
        wh[w][d] = total;
        total += v;
    }
    // publish this tile's count of digit d, then look back for the exclusive prefix over the earlier tiles
    uint64_t *my = look + (size_t)tile * RADIX + d;
    if (tile == 0) {
        os_store(my, epoch | OS_FLAG_INC | total);
    } else {
        os_store(my, epoch | OS_FLAG_AGG | total);
    }
    uint32_t excl = 0;
    for (int64_t t = tile - 1; t >= 0;) {
        const uint64_t v = os_load(look + (size_t)t * RADIX + d);
        if ((v & ~(OS_COUNT | OS_FLAG_AGG | OS_FLAG_INC)) != epoch || (v & (OS_FLAG_AGG | OS_FLAG_INC)) == 0) continue;
        excl += (uint32_t)(v & OS_COUNT);
        if (v & OS_FLAG_INC) break;
        t--;
    }
    if (tile > 0) os_store(my, epoch | OS_FLAG_INC | (excl + total));
    const uint32_t lo = block_excl_scan256(total, wt, nullptr);  // (contains __syncthreads)
    const uint32_t dbase = block_excl_scan256(dtot, wt, nullptr);
    loc[d] = lo;
    gofs[d] = dbase + excl - lo;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < IPT; it++) {
        const uint32_t dd = dr[it] >> 16;
        if (dd < RADIX) {
            const uint32_t lp = loc[dd] + wh[warp][dd] + (dr[it] & 0xffffu);
            skey[lp] = k[it];
            sval[lp] = val[it];
        }
    }
    __syncthreads();
    for (int i = tid; i < tile_n; i += OS_THREADS) {
        const KT key = skey[i];
        const uint32_t pos = gofs[(unsigned)(key >> shift) & ((1u << DB) - 1u)] + (uint32_t)i;
        kout[pos] = key;
        vout[pos] = sval[i];
    }
}

template <typename KT, int IPT>
constexpr int downsweep_smem() {
    return (int)((sizeof(KT) + sizeof(uint32_t)) * OS_THREADS * IPT);
}

template <typename KT, int IPT, int DB>
cudaError_t launch_radix_pass_db(KT *k0, KT *k1, uint32_t *v0, uint32_t *v1, const unsigned long long *n_dev,
                                 int64_t n_host, int64_t cap, int pass, int shift, SortState *ss, uint32_t *table_all,
                                 cudaStream_t st, bool have_table = false) {
    static bool configured_dev[TCGS_MAX_DEVICES] = {};
    bool &configured = configured_dev[current_device()];
    constexpr int smem = downsweep_smem<KT, IPT>();
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(radix_downsweep<KT, IPT, DB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(radix_downsweep<KT, IPT, DB>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int64_t tiles = div_up(n_dev ? cap : n_host, OS_THREADS * IPT);
    const unsigned grid = (unsigned)(tiles > 0 ? tiles : 1);
    uint32_t *table = table_all + (int64_t)pass * RADIX * tiles;
    cudaError_t e = cudaSuccess;
    if (!have_table)  // (have_table: an earlier kernel already wrote this pass's per-tile digit counts)
        e = launch_k(radix_upsweep<KT, IPT, DB>, grid, OS_THREADS, 0, st, k0, k1, n_dev, n_host, cap, pass, shift,
                     (const SortState *)ss, table, tiles);
    if (e == cudaSuccess) e = launch_k(radix_rowscan<IPT>, RADIX, 256, 0, st, n_dev, n_host, cap, pass, ss, table, tiles);
    if (e == cudaSuccess)
        e = launch_k(radix_downsweep<KT, IPT, DB>, grid, OS_THREADS, (size_t)smem, st, k0, k1, v0, v1, n_dev, n_host,
                     cap, pass, shift, (const SortState *)ss, (const uint32_t *)table, tiles);
    return e;
}


template <typename KT, int IPT, int DB>
cudaError_t launch_onesweep_db(KT *k0, KT *k1, uint32_t *v0, uint32_t *v1, const unsigned long long *n_dev,
                               int64_t n_host, int64_t cap, int pass, int shift, SortState *ss, uint64_t *look_all,
                               const OsHeader *hdr, cudaStream_t st) {
    static bool configured_dev[TCGS_MAX_DEVICES] = {};
    bool &configured = configured_dev[current_device()];
    constexpr int smem = downsweep_smem<KT, IPT>();
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(radix_onesweep<KT, IPT, DB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(radix_onesweep<KT, IPT, DB>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int64_t tiles = div_up(n_dev ? cap : n_host, OS_THREADS * IPT);
    const unsigned grid = (unsigned)(tiles > 0 ? tiles : 1);
    uint64_t *look = look_all + (int64_t)pass * RADIX * tiles;
    return launch_k(radix_onesweep<KT, IPT, DB>, grid, OS_THREADS, (size_t)smem, st, k0, k1, v0, v1, n_dev, n_host, cap,
                    pass, shift, ss, look, hdr);
}

// One pass on digit bits [shift, shift + db) (db <= RADIX_BITS): fewer digit bits, fewer warp ballots.
template <typename KT, int IPT>
cudaError_t launch_radix_pass(KT *k0, KT *k1, uint32_t *v0, uint32_t *v1, const unsigned long long *n_dev,
                              int64_t n_host, int64_t cap, int pass, int shift, int db, SortState *ss,
                              uint32_t *table_all, const OsHeader *hdr, cudaStream_t st, bool have_table = false) {
    if (TCGS_ONESWEEP) {
        uint64_t *look = reinterpret_cast<uint64_t *>(table_all);
        switch (db) {
            case 5: return launch_onesweep_db<KT, IPT, 5>(k0, k1, v0, v1, n_dev, n_host, cap, pass, shift, ss, look, hdr, st);
            case 6: return launch_onesweep_db<KT, IPT, 6>(k0, k1, v0, v1, n_dev, n_host, cap, pass, shift, ss, look, hdr, st);
            case 7: return launch_onesweep_db<KT, IPT, 7>(k0, k1, v0, v1, n_dev, n_host, cap, pass, shift, ss, look, hdr, st);
            default: return launch_onesweep_db<KT, IPT, 8>(k0, k1, v0, v1, n_dev, n_host, cap, pass, shift, ss, look, hdr, st);
        }
    }
    switch (db) {
        case 5: return launch_radix_pass_db<KT, IPT, 5>(k0, k1, v0, v1, n_dev, n_host, cap, pass, shift, ss, table_all, st, have_table);
        case 6: return launch_radix_pass_db<KT, IPT, 6>(k0, k1, v0, v1, n_dev, n_host, cap, pass, shift, ss, table_all, st, have_table);
        case 7: return launch_radix_pass_db<KT, IPT, 7>(k0, k1, v0, v1, n_dev, n_host, cap, pass, shift, ss, table_all, st, have_table);
        default: return launch_radix_pass_db<KT, IPT, 8>(k0, k1, v0, v1, n_dev, n_host, cap, pass, shift, ss, table_all, st, have_table);
    }
}

// ---------------------------------------------------------------- K3 / K4
// K1's tile rectangles are clipped to the frame; binning clips them to the tile-row band [y0, y1).
__device__ __forceinline__ short4 band_rect(short4 q, int y0, int y1) {
    q.y = q.y > y0 ? q.y : (short)y0;
    q.w = q.w < y1 - 1 ? q.w : (short)(y1 - 1);
    return q;
}
__device__ __forceinline__ uint32_t band_count(short4 q, int y0, int y1) {
    q = band_rect(q, y0, y1);
    return q.y <= q.w ? (uint32_t)((q.z - q.x + 1) * (q.w - q.y + 1)) : 0u;
}

// Opt-in exact coverage (TCGS_COVER_ELLIPSE): the tiles of band-clipped rectangle q the ellipse touches.
__device__ __forceinline__ uint32_t cover_count(const CoverRec &cs, short4 q) {
    uint32_t n = 0;
    for (int ty = q.y; ty <= q.w; ty++) {
        int lo, hi;
        if (cover_row(cs, ty, q.x, q.z, lo, hi)) n += (uint32_t)(hi - lo + 1);
    }
    return n;
}

// Exact coverage of Gaussian g clipped to the band (q = band_rect(r)): its count, and -- for rectangles of at
// most COVER_MASK_TILES tiles -- its tile mask re-based to q (mask 0 with a count: walk the rows).
__device__ __forceinline__ uint32_t exact_cover(const Rec *rec, uint32_t g, short4 r, short4 q, unsigned long long &m) {
    m = 0ull;
    if (q.y > q.w) return 0u;
    const CoverRec cs = make_cover(rec[g]);
    const int w = r.z - r.x + 1;
    if (w * (r.w - r.y + 1) <= COVER_MASK_TILES) {
        m = mask_rows(cover_mask(cs, r.x, r.y, r.z, r.w), w, q.y - r.y, q.w - r.y);
        return (uint32_t)__popcll(m);
    }
    return cover_count(cs, q);
}

// Exclusive scan of the per-block counts -> write offsets and N; also plans the tile-key sort (every pass
// runs unless there are no splats).  Run by the last CTA of count_upsweep (blockDim.x threads).
__device__ void count_scan(unsigned long long *blocksum, int nblocks, DevCounters *ctr, int64_t cap,
                           SortState *ss_tile, int npass) {
    __shared__ unsigned long long wt[32];
    const int nt = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per = (nblocks + nt - 1) / nt;
    const int b0 = tid * per;
    unsigned long long s = 0;
    for (int b = b0; b < b0 + per && b < nblocks; b++) s += __ldcg(&blocksum[b]);
    unsigned long long x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wt[warp] = x;
    __syncthreads();
    unsigned long long pre = 0, tot = 0;
    for (int w = 0; w < nt / 32; w++) {
        pre += w < warp ? wt[w] : 0ull;
        tot += wt[w];
    }
    unsigned long long run = pre + x - s;
    for (int b = b0; b < b0 + per && b < nblocks; b++) {
        const unsigned long long v = __ldcg(&blocksum[b]);
        blocksum[b] = run;
        run += v;
    }
    if (tid == 0) {
        ctr->n_splats = tot;
        ctr->overflow = tot > (unsigned long long)cap ? 1ull : 0ull;
        const bool any = tot > 0ull;
        int cur = 0;
        for (int p = 0; p < npass; p++) {
            ss_tile->pass_in[p] = cur;
            ss_tile->pass_do[p] = any ? 1 : 0;
            if (any) cur ^= 1;
        }
        ss_tile->final_buf = cur;
        ctr->tile_cur = cur;
    }
}

// EXACT: opt-in TCGS_COVER_ELLIPSE (separate instantiation, so the default keeps its registers): also stores
// each Gaussian's band-clipped tile mask in depth order for K4.
template <bool EXACT>
__global__ void __launch_bounds__(DUP_THREADS) count_upsweep(const uint32_t *idx0, const uint32_t *idx1,
                                                             DevCounters *ctr, const short4 *rect, const Rec *rec,
                                                             unsigned long long *tmask,
                                                             int band_y0, int band_y1,
                                                             int64_t P, unsigned long long *blocksum, int64_t cap,
                                                             SortState *ss_tile, int npass, int per) {
    pdl_wait();
    pdl_launch();
    const uint32_t *order = ctr->depth_cur ? idx1 : idx0;
    const int64_t beg = (int64_t)blockIdx.x * per;
    unsigned long long s = 0;
    for (int u = 0; u * DUP_THREADS < per; u++) {
        const int64_t i = beg + u * DUP_THREADS + threadIdx.x;
        if (u * DUP_THREADS + (int)threadIdx.x < per && i < P) {
            const uint32_t g = order[i];
            if (!EXACT) {
                s += band_count(rect[g], band_y0, band_y1);  // (an empty rectangle: 0)
            } else {
                unsigned long long m = 0ull;
                const short4 r = rect[g];
                if (r.x <= r.z) s += exact_cover(rec, g, r, band_rect(r, band_y0, band_y1), m);
                tmask[i] = m;
            }
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ unsigned long long ws[DUP_THREADS / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    __shared__ int last;
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < DUP_THREADS / 32; w++) t += ws[w];
        blocksum[blockIdx.x] = t;
        __threadfence();
        last = atomicAdd(&ss_tile->done_ctas, 1) == (int)gridDim.x - 1;  // the last CTA scans (K3b)
    }
    __syncthreads();
    if (last) {
        __threadfence();
        count_scan(blocksum, (int)gridDim.x, ctr, cap, ss_tile, npass);
    }
}

__global__ void __launch_bounds__(256) bin_init(uint4 *zero, int64_t n16, uint2 *ranges, int64_t n_ranges,
                                                DevCounters *ctr, const OsHeader *hdr, uint4 *look, int64_t look16) {
    pdl_wait();
    pdl_launch();
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, step = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = t; i < n16; i += step) zero[i] = make_uint4(0u, 0u, 0u, 0u);
    // a fresh workspace: clear the onesweep look-back tables once (depth_fix_hist then stamps the header; nothing
    // here writes it, so every CTA sees the same answer)
    if (hdr->magic != OS_MAGIC)
        for (int64_t i = t; i < look16; i += step) look[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int64_t i = t; i < n_ranges; i += step) ranges[i] = make_uint2(0u, 0u);
    if (t == 0) {
        ctr->n_splats = 0ull;
        ctr->overflow = 0ull;
        ctr->n_long_runs = 0u;
        ctr->compact = 0;
    }
}

// Exclusive scan of the per-block counts (one CTA of 1024 threads) -> write offsets and N.

// K4: duplicate-with-keys.  Each CTA walks `per` depth-ordered Gaussians 256 at a time, scans their
// tile counts, then expands (Gaussian, covered tile) pairs cooperatively: consecutive threads write
// consecutive splats (binary search of the slot in the shared inclusive scan).
template <typename KT, bool EXACT>
__global__ void __launch_bounds__(DUP_THREADS) duplicate_keys(const uint32_t *idx0, const uint32_t *idx1,
                                                              const DevCounters *ctr, const short4 *rect, const Rec *rec,
                                                              const unsigned long long *tmask, int64_t P,
                                                              const unsigned long long *blockoff, int tiles_x,
                                                              int band_y0, int band_y1, int64_t cap, KT *tkey,
                                                              uint32_t *tval, SortState *ss_tile, int npass,
                                                              int per, int mark) {
    pdl_wait();
    pdl_launch();
    // TCGS_ONESWEEP only: digit histograms of the tile-key radix passes (the onesweep passes' digit totals), per CTA
    // then global (the default reduce-then-scan passes count their digits in their own upsweep)
    __shared__ uint32_t dhist[TCGS_ONESWEEP ? TILE_MAX_PASSES : 1][RADIX];
    if (TCGS_ONESWEEP) {
        for (int e = threadIdx.x; e < TILE_MAX_PASSES * RADIX; e += DUP_THREADS) (&dhist[0][0])[e] = 0u;
        __syncthreads();
    }
    auto count_key = [&](uint32_t key) {
        if (TCGS_ONESWEEP)
            for (int p = 0; p < npass; p++) atomicAdd(&dhist[p][(key >> (RADIX_BITS * p)) & (RADIX - 1)], 1u);
    };
    __shared__ uint32_t incl[DUP_THREADS];
    __shared__ uint32_t gid[DUP_THREADS];
    __shared__ short4 rc[DUP_THREADS];
    __shared__ unsigned long long msk[EXACT ? DUP_THREADS : 1];
    __shared__ uint32_t wt[8];
    // staging of one round's output: every thread writes its own rectangle (no search, no division), then
    // the CTA copies the round out with coalesced stores
    constexpr int DUP_STAGE = 4096;
    __shared__ KT skey[DUP_STAGE];
    __shared__ uint32_t sval[DUP_STAGE];
    const uint32_t *order = ctr->depth_cur ? idx1 : idx0;
    const int tid = threadIdx.x;
    constexpr bool exact = EXACT;
    const int64_t beg = (int64_t)blockIdx.x * per;
    unsigned long long base = blockoff[blockIdx.x];
    for (int r = 0; r * DUP_THREADS < per; r++) {
        const int64_t i = r * DUP_THREADS + tid < per ? beg + r * DUP_THREADS + tid : P;
        uint32_t c = 0, g = 0;
        unsigned long long m = 0ull;  // exact coverage: the tile mask over q (0: walk rows)
        short4 q = make_short4(0, 0, -1, -1);
        if (i < P) {
            g = order[i];
            const short4 r = rect[g];  // (an empty rectangle for Gaussians that touch no tile)
            q = band_rect(r, band_y0, band_y1);
            c = q.x <= q.z && q.y <= q.w ? (uint32_t)((q.z - q.x + 1) * (q.w - q.y + 1)) : 0u;
            if (c && exact) {  // K3's mask (depth order, coalesced); rows for large rectangles
                m = tmask[i];
                c = m ? (uint32_t)__popcll(m) : cover_count(make_cover(rec[g]), q);
            }
            if (!c) q = make_short4(0, 0, -1, -1);
        }
        uint32_t total;
        const uint32_t ex = block_excl_scan256(c, wt, &total);
        if (total <= (uint32_t)DUP_STAGE) {
            constexpr uint32_t SMALL = TCGS_DUP_SMALL;  // larger rectangles: the whole warp writes one
            if (c <= SMALL) {
                uint32_t o = ex;
                if (exact && m) {  // set bits of the mask, row-major
                    const int w = q.z - q.x + 1;
                    for (unsigned long long mm = m; mm; mm &= mm - 1ull, o++) {
                        const int b = __ffsll((long long)mm) - 1, ty = q.y + b / w, tx = q.x + b % w;
                        skey[o] = (KT)((ty - band_y0) * tiles_x + tx);
                        sval[o] = g;
                    }
                } else {
                    CoverRec cs;
                    if ((exact || mark) && c) cs = make_cover(rec[g]);
                    for (int ty = q.y; ty <= q.w; ty++) {
                        const uint32_t row = (uint32_t)((ty - band_y0) * tiles_x);
                        int lo = q.x, hi = q.z;
                        if (exact && !cover_row(cs, ty, q.x, q.z, lo, hi)) continue;
                        if (!exact && mark && !cover_row(cs, ty, q.x, q.z, lo, hi)) {  // the whole row is dead
                            lo = q.z + 1;
                            hi = q.z;
                        }
                        for (int tx = q.x; tx <= q.z; tx++) {
                            if (exact && (tx < lo || tx > hi)) continue;
                            skey[o] = (KT)(row + tx);
                            sval[o] = (!exact && mark && (tx < lo || tx > hi)) ? (g | LIST_DEAD) : g;
                            o++;
                        }
                    }
                }
            }
            const int lane = tid & 31;
            unsigned big = __ballot_sync(0xffffffffu, c > SMALL);
            while (big) {  // large rectangles: the whole warp writes one
                const int src = __ffs(big) - 1;
                big &= big - 1;
                const uint32_t bc = __shfl_sync(0xffffffffu, c, src), bg = __shfl_sync(0xffffffffu, g, src);
                const uint32_t bex = __shfl_sync(0xffffffffu, ex, src);
                const int bx0 = __shfl_sync(0xffffffffu, (int)q.x, src), by0 = __shfl_sync(0xffffffffu, (int)q.y, src);
                const int bw = __shfl_sync(0xffffffffu, (int)(q.z - q.x + 1), src);
                const unsigned long long bm = exact ? __shfl_sync(0xffffffffu, m, src) : 0ull;
                if (exact && bm) {  // mask: lane b takes bit b, its slot is the popcount below it
                    for (int b = lane; b < COVER_MASK_TILES; b += 32) {
                        if (!((bm >> b) & 1ull)) continue;
                        const uint32_t o = bex + (uint32_t)__popcll(bm & ((1ull << b) - 1ull));
                        skey[o] = (KT)((by0 + b / bw - band_y0) * tiles_x + bx0 + b % bw);
                        sval[o] = bg;
                    }
                } else if (exact) {  // row by row: every lane computes the (uniform) row span
                    const int by1 = __shfl_sync(0xffffffffu, (int)q.w, src);
                    const CoverRec cs = make_cover(rec[bg]);
                    uint32_t o = bex;
                    for (int ty = by0; ty <= by1; ty++) {
                        int lo, hi;
                        if (!cover_row(cs, ty, bx0, bx0 + bw - 1, lo, hi)) continue;
                        const uint32_t row = (uint32_t)((ty - band_y0) * tiles_x);
                        for (int tx = lo + lane; tx <= hi; tx += 32) {
                            skey[o + (uint32_t)(tx - lo)] = (KT)(row + tx);
                            sval[o + (uint32_t)(tx - lo)] = bg;
                        }
                        o += (uint32_t)(hi - lo + 1);
                    }
                } else if (mark) {  // every tile of the square; those the ellipse misses are marked dead
                    const CoverRec cs = make_cover(rec[bg]);
                    for (uint32_t kk = lane; kk < bc; kk += 32) {
                        const int ty = by0 + (int)(kk / bw), tx = bx0 + (int)(kk % bw);
                        int lo, hi;
                        skey[bex + kk] = (KT)((ty - band_y0) * tiles_x + tx);
                        sval[bex + kk] = cover_row(cs, ty, tx, tx, lo, hi) ? bg : (bg | LIST_DEAD);
                    }
                } else {
                    for (uint32_t kk = lane; kk < bc; kk += 32) {
                        skey[bex + kk] = (KT)((by0 + (int)(kk / bw) - band_y0) * tiles_x + bx0 + (int)(kk % bw));
                        sval[bex + kk] = bg;
                    }
                }
            }
            __syncthreads();
            for (uint32_t s2 = tid; s2 < total; s2 += DUP_THREADS) {
                const unsigned long long pos = base + s2;
                if (pos < (unsigned long long)cap) {
                    const KT key = skey[s2];
                    tkey[pos] = key;
                    tval[pos] = sval[s2];
                    count_key((uint32_t)key);
                }
            }
        } else {  // a round with huge rectangles: search-based expansion straight to global memory
            incl[tid] = ex + c;
            gid[tid] = g;
            rc[tid] = q;
            if (exact) msk[tid] = m;
            __syncthreads();
            for (uint32_t s = tid; s < total; s += DUP_THREADS) {
                int lo = 0, hi = DUP_THREADS - 1;  // first item whose inclusive count exceeds s
    #pragma unroll 8
                for (int step = 0; step < 8; step++) {
                    const int mid = (lo + hi) >> 1;
                    if (incl[mid] > s) hi = mid;
                    else lo = mid + 1;
                }
                uint32_t kk = s - (lo ? incl[lo - 1] : 0u);
                const short4 qq = rc[lo];
                const int w = qq.z - qq.x + 1;
                int ty = qq.y + (int)(kk / w), tx = qq.x + (int)(kk % w);
                if (exact && msk[lo]) {  // the kk-th set bit of the mask
                    unsigned long long mm = msk[lo];
                    for (uint32_t j = 0; j < kk; j++) mm &= mm - 1ull;
                    const int b = __ffsll((long long)mm) - 1;
                    ty = qq.y + b / w;
                    tx = qq.x + b % w;
                } else if (exact) {  // walk the rows to the kk-th covered tile
                    const CoverRec cs = make_cover(rec[gid[lo]]);
                    for (ty = qq.y; ty <= qq.w; ty++) {
                        int rlo, rhi;
                        if (!cover_row(cs, ty, qq.x, qq.z, rlo, rhi)) continue;
                        const uint32_t rw = (uint32_t)(rhi - rlo + 1);
                        if (kk < rw) {
                            tx = rlo + (int)kk;
                            break;
                        }
                        kk -= rw;
                    }
                }
                const uint32_t key = (uint32_t)((ty - band_y0) * tiles_x + tx);
                const unsigned long long pos = base + s;
                if (pos < (unsigned long long)cap) {
                    tkey[pos] = (KT)key;
                    tval[pos] = gid[lo];
                    count_key(key);
                }
            }
        }
        base += total;
        __syncthreads();
    }
    if (TCGS_ONESWEEP)
        for (int e = threadIdx.x; e < npass * RADIX; e += DUP_THREADS) {
            const uint32_t c = (&dhist[0][0])[e];
            if (c) atomicAdd(&(&ss_tile->ghist[0][0])[e], c);
        }
}

// K6: tile ranges from the sorted keys: each thread compares 8 consecutive keys (one 16-byte load for
// 16-bit keys) with their successors.
template <typename KT>
__global__ void __launch_bounds__(256) tile_ranges(const KT *k0, const KT *k1, const DevCounters *ctr, int64_t cap,
                                                   uint2 *ranges) {
    pdl_wait();
    pdl_launch();
    const KT *keys = ctr->tile_cur ? k1 : k0;
    const unsigned long long nn = ctr->n_splats;
    const int64_t n = (int64_t)(nn < (unsigned long long)cap ? nn : (unsigned long long)cap);
    constexpr int V = 8;
    for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * V; i0 < n;
         i0 += (int64_t)gridDim.x * blockDim.x * V) {
        uint32_t k[V + 1];
        if (sizeof(KT) == 2 && i0 + V <= n) {
            const uint4 q = *reinterpret_cast<const uint4 *>(keys + i0);
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int u = 0; u < 4; u++) {
                k[2 * u] = w[u] & 0xffffu;
                k[2 * u + 1] = w[u] >> 16;
            }
        } else {
#pragma unroll
            for (int u = 0; u < V; u++) k[u] = i0 + u < n ? (uint32_t)keys[i0 + u] : 0xffffffffu;
        }
        k[V] = i0 + V < n ? (uint32_t)keys[i0 + V] : 0xffffffffu;
        if (i0 == 0) ranges[k[0]].x = 0u;
#pragma unroll
        for (int u = 0; u < V; u++) {
            const int64_t i = i0 + u;
            if (i < n && k[u] != k[u + 1]) {  // last entry of tile k[u]
                ranges[k[u]].y = (uint32_t)(i + 1);
                if (i + 1 < n) ranges[k[u + 1]].x = (uint32_t)(i + 1);
            }
        }
    }
}

// Debug / KAT entry: pack caller-given projected records and CSR offsets.
__global__ void pack_records(int64_t P, const double *mean2d, const double *conic, const double *opacity,
                             const float *colors, Rec *rec) {
    pdl_wait();
    pdl_launch();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P) return;
    Rec r;
    r.mx = (float)mean2d[2 * i];
    r.mx_lo = (float)(mean2d[2 * i] - (double)r.mx);
    r.my = (float)mean2d[2 * i + 1];
    r.my_lo = (float)(mean2d[2 * i + 1] - (double)r.my);
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
    pdl_wait();
    pdl_launch();
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    ranges[t] = make_uint2((uint32_t)offsets[band_tile0 + t], (uint32_t)offsets[band_tile0 + t + 1]);
}

// Splats per tile row of the whole frame (sum over Gaussians of the covered tiles in that row), from K1's
// frame-clipped rectangles: the replicated input of the tile-band partition (multi-GPU).
__global__ void __launch_bounds__(256) row_counts_kernel(int64_t P, const short4 *rect,
                                                         const Rec *rec, int coverage, int tiles_y,
                                                         unsigned long long *out) {
    pdl_wait();
    pdl_launch();
    constexpr int SMEM_ROWS = 4096;
    __shared__ unsigned long long h[SMEM_ROWS];
    const bool priv = tiles_y <= SMEM_ROWS;
    if (priv)
        for (int r = threadIdx.x; r < tiles_y; r += blockDim.x) h[r] = 0ull;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
        const short4 q = rect[i];
        if (q.x > q.z) continue;  // touches no tile
        if (coverage == TCGS_COVER_ELLIPSE) {
            const CoverRec cs = make_cover(rec[i]);
            for (int y = q.y; y <= q.w; y++) {
                int lo, hi;
                if (cover_row(cs, y, q.x, q.z, lo, hi))
                    atomicAdd(priv ? &h[y] : &out[y], (unsigned long long)(hi - lo + 1));
            }
            continue;
        }
        const unsigned long long w = (unsigned long long)(q.z - q.x + 1);
        for (int y = q.y; y <= q.w; y++) atomicAdd(priv ? &h[y] : &out[y], w);
    }
    if (!priv) return;
    __syncthreads();
    for (int r = threadIdx.x; r < tiles_y; r += blockDim.x)
        if (h[r]) atomicAdd(&out[r], h[r]);
}

// Compacted live lists (see LIST_DEAD): one CTA per tile writes the tile's unmarked entries, in list order, to cid
// at the tile's own offsets, with the number of marked entries before each (cdb), and its live count (ccount).
// Chunks of 8 warps x CW x 32 entries: warp w takes CW consecutive 32-entry rows (coalesced loads, ballots keep the
// order), one block scan of the warp totals per chunk.
constexpr int CW = 16;
__global__ void __launch_bounds__(256) compact_lists(const uint32_t *v0, const uint32_t *v1, DevCounters *ctr,
                                                     const uint2 *ranges, uint32_t *cid, uint32_t *cdb,
                                                     uint32_t *ccount) {
    pdl_wait();
    pdl_launch();
    if (blockIdx.x == 0 && threadIdx.x == 0) ctr->compact = 1;
    const uint32_t *val = ctr->tile_cur ? v1 : v0;
    const uint2 rg = ranges[blockIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned lt = lanemask_lt();
    __shared__ uint32_t wt[8];
    uint32_t live = 0;  // live entries of the tile before this chunk
    for (uint32_t c0 = rg.x; c0 < rg.y; c0 += 256 * CW) {
        const uint32_t wb = c0 + (uint32_t)warp * 32 * CW;  // this warp's rows
        uint32_t v[CW];
        unsigned m[CW];
        uint32_t cnt = 0;
#pragma unroll
        for (int k = 0; k < CW; k++) {
            const uint32_t i = wb + 32 * k + lane;
            v[k] = i < rg.y ? val[i] : LIST_DEAD;
            m[k] = __ballot_sync(0xffffffffu, (v[k] & LIST_DEAD) == 0u);
            cnt += __popc(m[k]);
        }
        uint32_t total;
        uint32_t lp = live + block_excl_scan256(lane == 0 ? cnt : 0u, wt, &total);  // (synchronises the CTA)
        lp = __shfl_sync(0xffffffffu, lp, 0);  // this warp's base
#pragma unroll
        for (int k = 0; k < CW; k++) {
            if ((m[k] >> lane) & 1u) {
                const uint32_t p = lp + __popc(m[k] & lt);
                cid[rg.x + p] = v[k];
                cdb[rg.x + p] = (wb + 32 * k + lane - rg.x) - p;  // marked entries before it
            }
            lp += __popc(m[k]);
        }
        live += total;
    }
    if (threadIdx.x == 0) ccount[blockIdx.x] = live;
}

template <typename KT>
cudaError_t bin_tiles(int64_t P, const Band &band, void *ws, const Layout &L, int64_t cap, cudaStream_t st,
                      bool compact) {
    DevCounters *ctr = at<DevCounters>(ws, L.counters);
    SortState *ss_tile = at<SortState>(ws, L.sort_state[1]);
    const int bits = tile_key_bits(band);
    const int npass = (bits + RADIX_BITS - 1) / RADIX_BITS;
    KT *tk0 = at<KT>(ws, L.tkey[0]);
    KT *tk1 = at<KT>(ws, L.tkey[1]);
    uint32_t *tv0 = at<uint32_t>(ws, L.tval[0]);
    uint32_t *tv1 = at<uint32_t>(ws, L.tval[1]);
    unsigned long long *blocksum = at<unsigned long long>(ws, L.blocksum);
    // Gaussians per K3/K4 CTA: DUP_ITEMS, or fewer so that small scenes still fill the GPU (C1: 10k Gaussians
    // whose rectangles cover ~65 tiles each ran K4 on 10 CTAs)
    const int64_t Pp = P > 0 ? P : 1;
    const int per = (int)std::max<int64_t>(32, std::min<int64_t>(DUP_ITEMS, div_up(Pp, DUP_MIN_CTAS) + 31) & ~31);
    const int nblk = (int)div_up(Pp, per);
    // K3
    const bool exact = band.coverage == TCGS_COVER_ELLIPSE;
    cudaError_t e0 = launch_k(exact ? count_upsweep<true> : count_upsweep<false>, nblk, DUP_THREADS, 0, st,
        (const uint32_t *)at<uint32_t>(ws, L.idx[0]), (const uint32_t *)at<uint32_t>(ws, L.idx[1]), ctr,
        (const short4 *)at<short4>(ws, L.rect), (const Rec *)at<Rec>(ws, L.rec), at<unsigned long long>(ws, L.tmask),
        band.y0, band.y1, P, blocksum, cap, ss_tile, npass, per);
    if (e0 != cudaSuccess) return e0;
    // K4
    e0 = launch_k(exact ? duplicate_keys<KT, true> : duplicate_keys<KT, false>, nblk, DUP_THREADS, 0, st,
        (const uint32_t *)at<uint32_t>(ws, L.idx[0]), (const uint32_t *)at<uint32_t>(ws, L.idx[1]),
        (const DevCounters *)ctr, (const short4 *)at<short4>(ws, L.rect), (const Rec *)at<Rec>(ws, L.rec),
        (const unsigned long long *)at<unsigned long long>(ws, L.tmask), P, (const unsigned long long *)blocksum,
        band.tiles_x, band.y0, band.y1, cap, tk0, tv0, ss_tile, npass, per, compact && !exact ? 1 : 0);
    if (e0 != cudaSuccess) return e0;
    // K5
    // the key's bits split as evenly as possible over the passes (13 bits: 7 + 6, not 8 + 5)
    const int db0 = TCGS_TILE_DIGITS_EVEN ? (bits + npass - 1) / npass : RADIX_BITS;
    for (int p = 0, shift = 0; p < npass; p++) {
        const int db = std::min(db0, bits - shift);
        cudaError_t e = launch_radix_pass<KT, TILEKEY_IPT>(tk0, tk1, tv0, tv1, &ctr->n_splats, 0, cap, p, shift, db,
                                                          ss_tile, at<uint32_t>(ws, L.lb_tile),
                                                          at<OsHeader>(ws, L.os_hdr), st);
        shift += db;
        if (e != cudaSuccess) return e;
    }
    // K6
    cudaError_t e6 = launch_k(tile_ranges<KT>, (unsigned)div_up(div_up(cap, 8), 256), 256, 0, st, (const KT *)tk0,
                              (const KT *)tk1, (const DevCounters *)ctr, cap, at<uint2>(ws, L.ranges));
    if (e6 != cudaSuccess || !compact || exact || band.n_tiles() == 0) return e6;
    return launch_k(compact_lists, (unsigned)band.n_tiles(), 256, 0, st, (const uint32_t *)tv0, (const uint32_t *)tv1,
                    ctr, (const uint2 *)at<uint2>(ws, L.ranges), at<uint32_t>(ws, L.cid), at<uint32_t>(ws, L.cdb),
                    at<uint32_t>(ws, L.ccount));
}

}  // namespace

cudaError_t launch_row_counts(int64_t P, const Band &band, const void *ws, const Layout &L, int64_t *out,
                              cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(int64_t) * (size_t)band.tiles_y, st);
    if (e != cudaSuccess || P <= 0) return e;
    const int64_t blocks = div_up(P, 256 * 8);
    return launch_k(row_counts_kernel, (unsigned)(blocks < 4 * 148 ? blocks : 4 * 148), 256, 0, st, P,
                    (const short4 *)at<short4>(ws, L.rect), (const Rec *)at<Rec>(ws, L.rec), band.coverage,
                    band.tiles_y, reinterpret_cast<unsigned long long *>(out));
}

namespace {
__global__ void strip_marks(const uint32_t *src, uint32_t *dst, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i] & ~LIST_DEAD;
}
}  // namespace

// Tile-list ids without K4's dead marks (tcgs_copy_lists).
cudaError_t launch_strip_marks(const uint32_t *src, uint32_t *dst, int64_t n, cudaStream_t st) {
    const int64_t blocks = div_up(n, 256);
    strip_marks<<<(unsigned)(blocks < 4 * 148 ? blocks : 4 * 148), 256, 0, st>>>(src, dst, n);
    return cudaGetLastError();
}

int tile_key_bits(const Band &band) {
    const int nt = band.n_tiles();
    int bits = 1;
    while ((1 << bits) < nt) bits++;
    return bits;
}

cudaError_t launch_bin(int64_t P, const Band &band, void *ws, const Layout &L, int64_t cap, cudaStream_t st,
                       bool compact) {
    DevCounters *ctr = at<DevCounters>(ws, L.counters);
    SortState *ss_depth = at<SortState>(ws, L.sort_state[0]);
    // one kernel clears the sort state, the tile ranges and the per-binning counters (K1's dropped /
    // n_visible / key_min / key_max stay)
    cudaError_t e = launch_k(bin_init, 2 * 148, 256, 0, st,
                             reinterpret_cast<uint4 *>(static_cast<char *>(ws) + L.zero_begin),
                             (int64_t)(L.zero_bytes / sizeof(uint4)), at<uint2>(ws, L.ranges),
                             (int64_t)(band.n_tiles() ? band.n_tiles() : 1), ctr, (const OsHeader *)at<OsHeader>(ws, L.os_hdr),
                             reinterpret_cast<uint4 *>(static_cast<char *>(ws) + L.lb_depth),
                             (int64_t)(L.lb_bytes / sizeof(uint4)));
    if (e != cudaSuccess) return e;
    uint32_t *k0 = at<uint32_t>(ws, L.key64[0]);
    uint32_t *k1 = at<uint32_t>(ws, L.key64[1]);
    uint32_t *i0 = at<uint32_t>(ws, L.idx[0]);
    uint32_t *i1 = at<uint32_t>(ws, L.idx[1]);
    if (P > 0) {
        // K2: 24-bit depth-prefix radix sort + exact float64 fix-up of equal prefixes
        const unsigned long long *src = at<unsigned long long>(ws, L.key_src);
        const int64_t T0 = div_up(P, OS_THREADS * DEPTH_IPT);  // radix tiles of the depth passes
        e = launch_k(depth_fix_hist, (unsigned)T0, OS_THREADS, 0, st, src, k0, i0, P, ctr, ss_depth,
                     at<OsHeader>(ws, L.os_hdr), TCGS_ONESWEEP ? nullptr : at<uint32_t>(ws, L.lb_depth), T0);
        if (e != cudaSuccess) return e;
        for (int p = 0; p < DEPTH_PASSES; p++) {
            // pass 0's digit table comes from depth_fix_hist
            e = launch_radix_pass<uint32_t, DEPTH_IPT>(k0, k1, i0, i1, nullptr, P, P, p, RADIX_BITS * p, RADIX_BITS,
                                                       ss_depth, at<uint32_t>(ws, L.lb_depth),
                                                       at<OsHeader>(ws, L.os_hdr), st, p == 0 && !TCGS_ONESWEEP);
            if (e != cudaSuccess) return e;
        }
        e = launch_k(depth_fixup, (unsigned)std::min<int64_t>(div_up(P, 256), 8 * 148), 256, 0, st,
                     (const uint32_t *)k0, (const uint32_t *)k1, i0, i1, src, P, ctr, at<uint32_t>(ws, L.long_runs));
        if (e == cudaSuccess)
            e = launch_k(depth_fixup_long, 148, 256, 0, st, (const uint32_t *)k0, (const uint32_t *)k1, i0, i1, src, P,
                         ctr, (const uint32_t *)at<uint32_t>(ws, L.long_runs), at<unsigned long long>(ws, L.fix_scratch));
        if (e != cudaSuccess) return e;
    }
    if (band.n_tiles() <= 65536) return bin_tiles<uint16_t>(P, band, ws, L, cap, st, compact);
    return bin_tiles<uint32_t>(P, band, ws, L, cap, st, compact);
}

cudaError_t launch_pack_lists(int64_t P, const double *mean2d, const double *conic, const double *opacity,
                              const float *colors, const int64_t *offsets, const Band &band, void *ws,
                              const Layout &L, cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    if (P > 0) e = launch_k(pack_records, (unsigned)((P + 255) / 256), 256, 0, st, P, mean2d, conic, opacity, colors,
                            at<Rec>(ws, L.rec));
    const int nt = band.n_tiles();
    if (e == cudaSuccess && nt > 0)
        e = launch_k(pack_ranges, (nt + 255) / 256, 256, 0, st, offsets, band.y0 * band.tiles_x, nt, at<uint2>(ws, L.ranges));
    return e;
}

}  // namespace tcgs
