// Microbenchmarks of basic latencies on the B200 (profiling aid, not product code):
// dependent-chain L2 / HBM / shared loads, barrier, shared atomics, shuffles.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void chase_global(const uint32_t* __restrict__ next, int steps, long long* out, uint32_t* sink) {
    uint32_t p = 0;
    // warm pass
    for (int i = 0; i < steps; ++i) p = __ldcg(&next[p]);
    long long t0 = clock64();
    for (int i = 0; i < steps; ++i) p = __ldcg(&next[p]);
    long long t1 = clock64();
    out[0] = (t1 - t0) / steps;
    sink[0] = p;
}
__global__ void chase_cold(const uint32_t* __restrict__ next, int steps, long long* out, uint32_t* sink) {
    uint32_t p = 0;
    long long t0 = clock64();
    for (int i = 0; i < steps; ++i) p = __ldcg(&next[p]);
    long long t1 = clock64();
    out[0] = (t1 - t0) / steps;
    sink[0] = p;
}
__global__ void prims(long long* out, uint32_t* sink) {
    __shared__ uint32_t s[4096];
    __shared__ int cnt[32];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = (i * 97 + 13) & 4095;
    if (threadIdx.x < 32) cnt[threadIdx.x] = 0;
    __syncthreads();
    long long t0, t1;
    uint32_t p = threadIdx.x & 4095;
    // LDS chain
    t0 = clock64();
    for (int i = 0; i < 256; ++i) p = s[p];
    t1 = clock64();
    if (threadIdx.x == 0) out[0] = (t1 - t0) / 256;
    __syncthreads();
    // barrier
    t0 = clock64();
    for (int i = 0; i < 256; ++i) __syncthreads();
    t1 = clock64();
    if (threadIdx.x == 0) out[1] = (t1 - t0) / 256;
    // smem atomics, dependent, one warp, distinct addresses
    if (threadIdx.x < 32) {
        int v = 0;
        t0 = clock64();
        for (int i = 0; i < 256; ++i) v = atomicAdd(&cnt[(threadIdx.x + v) & 31], 1) & 0;
        t1 = clock64();
        if (threadIdx.x == 0) out[2] = (t1 - t0) / 256;
        p += v;
        // same address from all lanes
        t0 = clock64();
        for (int i = 0; i < 256; ++i) v = atomicAdd(&cnt[v & 0], 1) & 0;
        t1 = clock64();
        if (threadIdx.x == 0) out[3] = (t1 - t0) / 256;
        p += v;
        // shuffle chain
        float f = (float)threadIdx.x;
        t0 = clock64();
        for (int i = 0; i < 256; ++i) f = __shfl_xor_sync(0xffffffffu, f, 1 + (i & 15)) + 1.0f;
        t1 = clock64();
        if (threadIdx.x == 0) out[4] = (t1 - t0) / 256;
        p += (uint32_t)f;
        // ballot chain
        unsigned b = threadIdx.x;
        t0 = clock64();
        for (int i = 0; i < 256; ++i) b = __ballot_sync(0xffffffffu, (b >> (threadIdx.x & 31)) & 1) + threadIdx.x;
        t1 = clock64();
        if (threadIdx.x == 0) out[5] = (t1 - t0) / 256;
        p += b;
        // dependent fp64 fma chain
        double d = threadIdx.x;
        t0 = clock64();
        for (int i = 0; i < 256; ++i) d = fma(d, 1.0000001, 0.5);
        t1 = clock64();
        if (threadIdx.x == 0) out[6] = (t1 - t0) / 256;
        p += (uint32_t)d;
        // dependent fp32 fma chain
        float g = threadIdx.x;
        t0 = clock64();
        for (int i = 0; i < 256; ++i) g = fmaf(g, 1.0000001f, 0.5f);
        t1 = clock64();
        if (threadIdx.x == 0) out[7] = (t1 - t0) / 256;
        p += (uint32_t)g;
    }
    sink[threadIdx.x] = p;
}
int main() {
    long long* d_out; uint32_t* sink;
    cudaMalloc(&d_out, 64 * 8); cudaMalloc(&sink, 4096 * 4);
    long long h[8];
    for (size_t mb : {4, 32, 96, 1024}) {
        size_t n = mb * (1 << 20) / 4;
        uint32_t* hn = new uint32_t[n];
        // random cycle with stride >= 128 B
        size_t m = n / 32;
        uint32_t* perm = new uint32_t[m];
        for (size_t i = 0; i < m; ++i) perm[i] = i;
        uint64_t x = 88172645463325252ull;
        for (size_t i = m - 1; i > 0; --i) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; size_t j = x % (i + 1); uint32_t t = perm[i]; perm[i] = perm[j]; perm[j] = t; }
        for (size_t i = 0; i < m; ++i) hn[perm[i] * 32] = perm[(i + 1) % m] * 32;
        uint32_t* dn; cudaMalloc(&dn, n * 4);
        cudaMemcpy(dn, hn, n * 4, cudaMemcpyHostToDevice);
        for (int blk : {0, 7, 74, 140}) {
            // launch 1 thread on some SM (block index picks a different SM in practice)
            chase_global<<<blk + 1, 1>>>(dn, 2048, d_out, sink);
            cudaMemcpy(h, d_out, 8, cudaMemcpyDeviceToHost);
            printf("global chase %zu MB (warm, grid %d): %lld cycles/load\n", mb, blk + 1, h[0]);
        }
        delete[] hn; delete[] perm; cudaFree(dn);
    }
    for (int t : {32, 512, 1024}) {
        prims<<<1, t>>>(d_out, sink);
        cudaMemcpy(h, d_out, 64, cudaMemcpyDeviceToHost);
        printf("threads %d: lds %lld, bar.sync %lld, atoms distinct %lld, atoms same %lld, shfl+fadd %lld, ballot %lld, dfma %lld, ffma %lld cycles\n",
               t, h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7]);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
