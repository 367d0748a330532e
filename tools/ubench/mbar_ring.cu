// Microbenchmark: cost per slot of an S-slot mbarrier ring between a producer
// warp and a consumer warp (no data), with optional extra warps spinning on
// another barrier -- the handshake skeleton of the LM-head kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbar_ring mbar_ring.cu && ./mbar_ring
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
template <int MODE>
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
    if (MODE == 0) {
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par) : "memory");
    } else if (MODE == 1) {
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par) : "memory");
    } else {
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par), "r"(20) : "memory");
    }
}

template <int MODE>
__global__ void ring(int iters, int S, int spinners, long long* out) {
    __shared__ uint64_t full[16], empty[16], never;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { init(&full[s], 32); init(&empty[s], 32); }
        init(&never, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int warp = threadIdx.x / 32;
    long long t0 = clock64();
    if (warp == 0) {   // producer
        int st = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            wait<MODE>(&empty[st], ph ^ 1);
            arrive(&full[st]);
            if (++st == S) { st = 0; ph ^= 1; }
        }
    } else if (warp == 1) {   // consumer
        int st = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            wait<MODE>(&full[st], ph);
            arrive(&empty[st]);
            if (++st == S) { st = 0; ph ^= 1; }
        }
        if (threadIdx.x == 32) { out[blockIdx.x] = clock64() - t0; arrive(&never); }
    } else if (warp - 2 < spinners) {
        wait<MODE>(&never, 0);
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    long long h[148];
    for (int mode = 0; mode < 3; ++mode)
        for (int S : {4, 10})
            for (int sp : {0, 8}) {
                const int iters = 640;
                auto k = mode == 0 ? ring<0> : mode == 1 ? ring<1> : ring<2>;
                k<<<148, 32 * (2 + sp)>>>(iters, S, sp, d);
                k<<<148, 32 * (2 + sp)>>>(iters, S, sp, d);
                cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                double m = 0;
                for (int i = 0; i < 148; ++i) m += h[i];
                printf("mode %d (%s) S=%2d spinners=%d: %.1f cycles per slot  (%s)\n", mode,
                       mode == 0 ? "try_wait" : mode == 1 ? "test_wait" : "try_wait hint 20ns", S, sp, m / 148 / iters,
                       cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
