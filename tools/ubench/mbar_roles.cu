// Microbenchmark: the LM-head kernel's barrier skeleton (no data): 4 producer
// warps (128 arrivals) + 1 loader lane on full[s] (count 129), one MMA warp
// waiting full[s] (all lanes or one lane) and arriving on empty[s], 8 warps
// waiting on a barrier that completes at the end. Cycles per slot.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbar_roles mbar_roles.cu && ./mbar_roles
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void init(uint64_t* b, int n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n)); }
__device__ __forceinline__ void arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory"); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(par) : "memory");
}

__global__ void roles(int iters, int S, int variant, long long* out) {
    __shared__ uint64_t full[16], empty[16], done;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nprod = (variant & 4) ? 32 : 128;   // 4: one arrival per producer warp... (lane 0 only)
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) { init(&full[s], ((variant & 4) ? 4 : 128) + 1); init(&empty[s], 1); }
        init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    (void)nprod;
    long long t0 = clock64();
    const bool prod = (warp & 3) >= 2 && warp < 8;
    if (prod) {
        int st = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            if (variant & 2) { if (lane == 0) wait(&empty[st], ph ^ 1); __syncwarp(); }
            else wait(&empty[st], ph ^ 1);
            if (!(variant & 4) || lane == 0) arrive(&full[st]);
            if (++st == S) { st = 0; ph ^= 1; }
        }
    } else if (warp == 11) {
        if (lane == 0) {
            int st = 0; uint32_t ph = 0;
            for (int i = 0; i < iters; ++i) {
                wait(&empty[st], ph ^ 1);
                arrive(&full[st]);
                if (++st == S) { st = 0; ph ^= 1; }
            }
        }
    } else if (warp == 10) {
        int st = 0; uint32_t ph = 0;
        for (int i = 0; i < iters; ++i) {
            if (variant & 1) { if (lane == 0) wait(&full[st], ph); __syncwarp(); }
            else wait(&full[st], ph);
            if (lane == 0) arrive(&empty[st]);
            if (++st == S) { st = 0; ph ^= 1; }
        }
        if (lane == 0) { out[blockIdx.x] = clock64() - t0; arrive(&done); }
    } else if ((warp & 3) < 2 && !(variant & 8)) {
        wait(&done, 0);
    }
    __syncthreads();
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    long long h[148];
    const char* names[] = {"base (all lanes poll)", "mma: lane0 polls", "prod: lane0 polls", "both lane0",
                           "prod: 1 arrival/warp", "", "", "lane0 polls + 1 arrival/warp", "no epilogue waiters"};
    for (int v : {0, 1, 2, 3, 4, 7, 8}) {
        for (int S : {4, 10}) {
            const int iters = 640;
            roles<<<148, 448>>>(iters, S, v, d);
            roles<<<148, 448>>>(iters, S, v, d);
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double m = 0;
            for (int i = 0; i < 148; ++i) m += h[i];
            printf("variant %d %-32s S=%2d: %.1f cycles per slot (%s)\n", v, names[v], S, m / 148 / iters,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
