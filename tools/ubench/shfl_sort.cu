// Microbenchmark: cycles of a single-warp bitonic sort32 (rolled / unrolled)
// while the rest of the CTA waits at a barrier. Profiling aid, not product code.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ bool before(float a, int ida, float b, int idb) { return a > b || (a == b && ida < idb); }
template <bool ROLL>
__device__ __forceinline__ void sort32(float& v, int& p) {
    const int lane = threadIdx.x & 31;
    if (ROLL) {
#pragma unroll 1
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll 1
            for (int j = k >> 1; j > 0; j >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, v, j);
                const int op = __shfl_xor_sync(0xffffffffu, p, j);
                const bool kb = ((lane & j) == 0) == ((lane & k) == 0);
                if (kb == before(ov, op, v, p)) { v = ov; p = op; }
            }
        }
    } else {
#pragma unroll
        for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
            for (int j = k >> 1; j > 0; j >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, v, j);
                const int op = __shfl_xor_sync(0xffffffffu, p, j);
                const bool kb = ((lane & j) == 0) == ((lane & k) == 0);
                if (kb == before(ov, op, v, p)) { v = ov; p = op; }
            }
        }
    }
}
template <bool ROLL>
__global__ void k_sort(long long* out, float* sink, int reps) {
    float v = (float)((threadIdx.x * 7919) % 113);
    int p = threadIdx.x;
    __syncthreads();
    if (threadIdx.x < 32) {
        long long t0 = clock64();
        for (int i = 0; i < reps; ++i) { sort32<ROLL>(v, p); v += 1.0f; }
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    sink[threadIdx.x] = v + p;
}
int main() {
    long long* d; float* s;
    cudaMalloc(&d, 1024 * 8); cudaMalloc(&s, 4096 * 4);
    for (int roll = 0; roll < 2; ++roll)
        for (int threads : {32, 512})
            for (int reps : {1, 2, 16}) {
                long long h = 0;
                for (int it = 0; it < 3; ++it) {
                    if (roll) k_sort<true><<<1, threads>>>(d, s, reps); else k_sort<false><<<1, threads>>>(d, s, reps);
                    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                    printf("roll=%d threads=%d reps=%d iter=%d: %lld cycles/sort\n", roll, threads, reps, it, h / reps);
                }
            }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
