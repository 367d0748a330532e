// Microbenchmark: the finalisation's warp-level steps in isolation (rolled
// bitonic KP-th largest, unrolled warp max, a 5-iteration smem/expf loop),
// to compare with their in-kernel cost (fin64.cuh, EVOSPEC_TRACE clock stamps).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float kth_rolled(float x, int kth) {
    const int lane = threadIdx.x & 31;
#pragma unroll 1
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            const float y = __shfl_xor_sync(0xffffffffu, x, j);
            x = (((lane & j) == 0) == ((lane & k) == 0)) ? fmaxf(x, y) : fminf(x, y);
        }
    }
    return __shfl_sync(0xffffffffu, x, kth - 1);
}
__device__ __forceinline__ float kth_unrolled(float x, int kth) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const float y = __shfl_xor_sync(0xffffffffu, x, j);
            x = (((lane & j) == 0) == ((lane & k) == 0)) ? fmaxf(x, y) : fminf(x, y);
        }
    }
    return __shfl_sync(0xffffffffu, x, kth - 1);
}

__global__ void steps(const float* in, int n, int kth, long long* out, float* sink) {
    __shared__ float l_m[320], l_s[320];
    for (int i = threadIdx.x; i < 320; i += blockDim.x) { l_m[i] = in[i]; l_s[i] = in[i + 320]; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    float acc = 0.0f;
    if (threadIdx.x < 32) {
        long long t[6];
        t[0] = clock64();
        float lm = -INFINITY;
#pragma unroll 1
        for (int c = lane; c < n; c += 32) lm = fmaxf(lm, l_m[c]);
        t[1] = clock64();
        float th = kth_rolled(lm, kth);
        t[2] = clock64();
        float th2 = kth_unrolled(lm + th * 1e-30f, kth);
        t[3] = clock64();
        float M = lm;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
        t[4] = clock64();
        float S = 0.0f;
        int nq = 0;
#pragma unroll 1
        for (int c0 = 0; c0 < n; c0 += 32) {
            const int c = c0 + lane;
            const float h = c < n ? l_m[c] : -INFINITY;
            if (h != -INFINITY) S += l_s[c] * expf(h - M);
            const unsigned qm = __ballot_sync(0xffffffffu, h >= th);
            nq += __popc(qm);
        }
        t[5] = clock64();
        acc = S + th + th2 + nq;
        if (lane == 0 && blockIdx.x == 0)
            for (int i = 0; i < 5; ++i) out[i] = t[i + 1] - t[i];
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
    float h[640];
    for (int i = 0; i < 640; ++i) h[i] = (float)((i * 7919) % 1000) / 100.0f;
    float *d_in, *sink; long long* d_out;
    cudaMalloc(&d_in, sizeof(h)); cudaMalloc(&sink, 148 * 128 * 4); cudaMalloc(&d_out, 64);
    cudaMemcpy(d_in, h, sizeof(h), cudaMemcpyHostToDevice);
    for (int g : {1, 60, 148})
        for (int rep = 0; rep < 2; ++rep) {
            steps<<<g, 128>>>(d_in, 148, 18, d_out, sink);
            long long o[5];
            cudaMemcpy(o, d_out, 40, cudaMemcpyDeviceToHost);
            printf("grid %3d rep %d: lane-max loop %lld, kth rolled %lld, kth unrolled %lld, warp_max %lld, S/ballot loop %lld cycles\n",
                   g, rep, o[0], o[1], o[2], o[3], o[4]);
        }
    return 0;
}
