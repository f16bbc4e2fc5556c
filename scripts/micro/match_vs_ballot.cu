// Microbenchmark (not part of the product): warp peer masks of 8-bit digits by __match_any_sync vs 8 ballots.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned peers_ballot(int d) {
    unsigned peers = 0xffffffffu;
#pragma unroll
    for (int b = 0; b < 8; b++) {
        const bool bit = (d >> b) & 1;
        const unsigned m = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? m : ~m;
    }
    return peers;
}

template <int MODE>
__global__ void k(const uint32_t *in, uint32_t *out, int iters) {
    uint32_t x = in[blockIdx.x * blockDim.x + threadIdx.x];
    uint32_t acc = 0;
    for (int i = 0; i < iters; i++) {
        const int d = (x >> (i & 7)) & 0xff;
        const unsigned p = MODE == 0 ? peers_ballot(d) : __match_any_sync(0xffffffffu, d);
        acc += __popc(p & ((1u << (threadIdx.x & 31)) - 1u));
        x = x * 1664525u + 1013904223u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    uint32_t *in, *out;
    cudaMalloc(&in, blocks * threads * 4);
    cudaMalloc(&out, blocks * threads * 4);
    cudaMemset(in, 0x5a, blocks * threads * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int mode = 0; mode < 2; mode++) {
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            if (mode == 0) k<0><<<blocks, threads>>>(in, out, iters);
            else k<1><<<blocks, threads>>>(in, out, iters);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double warp_ops = (double)blocks * threads / 32 * iters;
            printf("%s: %.3f ms, %.2f ns per warp-peer-mask per SM\n", mode == 0 ? "8 ballots" : "match.any", ms,
                   ms * 1e6 / (warp_ops / 148));
        }
    }
    return 0;
}
