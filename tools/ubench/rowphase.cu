// Microbenchmark: the LM head's last-tile row phase in isolation (one warp per
// row over 60 rows of 256 staged logits in shared memory, 14 warps): row max and
// exp-sum by shuffles, the KP-th largest lane maximum by a warp bitonic sort, the
// admission ballots and appends. Cycles per phase, per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rowphase rowphase.cu && ./rowphase
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int V>
__global__ void rowphase(const float* gz, long long* out, float* sink) {
    extern __shared__ float zs[];           // [60][260]
    __shared__ float bv[60 * 65];
    __shared__ int bp[60 * 65];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 60 * 260; i += blockDim.x) zs[i] = gz[i];
    __syncthreads();
    long long t0 = clock64();
    const float L2E = 1.4426950408889634f;
    const int KP = 18;
    float acc = 0.f;
    for (int rr = warp; rr < 60; rr += blockDim.x / 32) {
        float v[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = zs[rr * 260 + lane + 32 * j];
        float lm = v[0];
#pragma unroll
        for (int j = 1; j < 8; ++j) lm = fmaxf(lm, v[j]);
        float M = lm;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        float s = 0.f;
        if (V & 1) {
            const float mb = M * L2E;
#pragma unroll
            for (int j = 0; j < 8; ++j) s += ex2f(fmaf(v[j], L2E, -mb));
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        }
        float B = -INFINITY;
        if (V & 2) {
            float x = lm;
#pragma unroll
            for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
                for (int j = k >> 1; j > 0; j >>= 1) {
                    const float y = __shfl_xor_sync(0xffffffffu, x, j);
                    x = (((lane & k) == 0) == ((lane & j) == 0)) ? fmaxf(x, y) : fminf(x, y);
                }
            B = __shfl_sync(0xffffffffu, x, KP - 1);
        }
        if (V & 4) {
            uint32_t bal[8];
            int pos = 0;
            const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                bal[j] = __ballot_sync(0xffffffffu, v[j] >= B);
                if ((bal[j] >> lane) & 1u) {
                    const int sl = pos + __popc(bal[j] & lt);
                    if (sl < 64) { bv[rr * 65 + sl] = v[j]; bp[rr * 65 + sl] = lane + 32 * j; }
                }
                pos += __popc(bal[j]);
            }
        }
        acc += s + B;
    }
    __syncwarp();
    long long t1 = clock64();
    if (lane == 0 && warp == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[0] = acc;
}

int main() {
    float* gz; long long* d; float* sink;
    cudaMalloc(&gz, 60 * 260 * 4); cudaMalloc(&d, 148 * 8); cudaMalloc(&sink, 4);
    float h[60 * 260];
    unsigned x = 1;
    for (int i = 0; i < 60 * 260; ++i) { x = x * 1664525u + 1013904223u; h[i] = (float)(x >> 8) / 16777216.f * 4.f - 2.f; }
    cudaMemcpy(gz, h, sizeof(h), cudaMemcpyHostToDevice);
    long long hh[148];
    int smem_bytes = 60 * 260 * 4;
    char* fl; cudaMalloc(&fl, 512 << 20);
    bool flush = false;
    auto run = [&](auto k, const char* name, int warps) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
        for (int it = 0; it < 3; ++it) {
            if (flush) cudaMemsetAsync(fl, it, 512 << 20);
            k<<<148, 32 * warps, smem_bytes>>>(gz, d, sink);
        }
        cudaDeviceSynchronize();
        cudaMemcpy(hh, d, sizeof(hh), cudaMemcpyDeviceToHost);
        double m = 0; for (int i = 0; i < 148; ++i) m += hh[i];
        printf("%-28s warps=%2d: %.0f cycles (%s)\n", name, warps, m / 148, cudaGetErrorString(cudaGetLastError()));
    };
    for (int sm : {0, 1}) {
    flush = sm;
    printf("L2 flushed before each launch: %d\n", sm);
    for (int w : {14}) {
        run(rowphase<0>, "max only", w);
        run(rowphase<1>, "max+sum", w);
        run(rowphase<3>, "max+sum+bitonic", w);
        run(rowphase<7>, "all", w);
    }
    }
    return 0;
}
