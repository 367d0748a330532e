// Microbenchmark: cost of executing straight-line code the first time (cold
// instruction fetch) vs again (warm), for a single warp per CTA -- the
// regime of the LM head's last-tile fold and the finalisation (code run once).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o icache icache.cu && ./icache
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define A8 asm volatile("add.f32 %0, %0, %8;\n add.f32 %1, %1, %8;\n add.f32 %2, %2, %8;\n add.f32 %3, %3, %8;\n" \
                        "add.f32 %4, %4, %8;\n add.f32 %5, %5, %8;\n add.f32 %6, %6, %8;\n add.f32 %7, %7, %8;\n" \
                        : "+f"(x0), "+f"(x1), "+f"(x2), "+f"(x3), "+f"(x4), "+f"(x5), "+f"(x6), "+f"(x7) : "f"(c));
#define A64 A8 A8 A8 A8 A8 A8 A8 A8
#define A512 A64 A64 A64 A64 A64 A64 A64 A64

template <int REP>
__global__ void straight(float c, long long* out, float* sink) {
    float x0 = threadIdx.x, x1 = x0 * 2.f, x2 = x0 * 3.f, x3 = x0 * 5.f, x4 = x0 * 7.f, x5 = x0 * 11.f, x6 = x0 * 13.f, x7 = x0 * 17.f;
    long long t0 = clock64();
#pragma unroll
    for (int r = 0; r < REP; ++r) { A512 }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// the same block twice inside one launch: pass 1 cold, pass 2 from the SM's instruction caches
template <int REP>
__global__ void twice(float c, long long* out, float* sink) {
    float x0 = threadIdx.x, x1 = x0 * 2.f, x2 = x0 * 3.f, x3 = x0 * 5.f, x4 = x0 * 7.f, x5 = x0 * 11.f, x6 = x0 * 13.f, x7 = x0 * 17.f;
    long long t[3];
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
        t[pass] = clock64();
#pragma unroll
        for (int r = 0; r < REP; ++r) { A512 }
    }
    t[2] = clock64();
    if (threadIdx.x == 0) { out[2 * blockIdx.x] = t[1] - t[0]; out[2 * blockIdx.x + 1] = t[2] - t[1]; }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main() {
    long long* d_out; float* sink; char* flush;
    cudaMalloc(&d_out, 148 * 8); cudaMalloc(&sink, 148 * 1024 * 4); cudaMalloc(&flush, 256 << 20);
    long long h[148];
    auto run = [&](const char* name, int grid, int block, bool do_flush, auto kern, int n_instr) {
        if (do_flush) cudaMemset(flush, 1, 256 << 20);
        kern<<<grid, block>>>(1.0f, d_out, sink);
        cudaMemcpy(h, d_out, grid * 8, cudaMemcpyDeviceToHost);
        long long mx = 0, mn = 1LL << 60, s = 0;
        for (int i = 0; i < grid; ++i) { mx = h[i] > mx ? h[i] : mx; mn = h[i] < mn ? h[i] : mn; s += h[i]; }
        printf("%-28s grid %3d block %4d: cycles min %7lld mean %7lld max %7lld  (%.2f cyc/instr at mean)\n", name, grid,
               block, mn, s / grid, mx, (double)(s / grid) / n_instr);
    };
    for (int g : {1, 148}) {
        for (int b : {32, 128}) {
            run("4096 instr, L2 flushed", g, b, true, straight<8>, 4096);
            run("4096 instr, again (warm)", g, b, false, straight<8>, 4096);
            run("16384 instr, L2 flushed", g, b, true, straight<32>, 16384);
            run("16384 instr, again (warm)", g, b, false, straight<32>, 16384);
        }
    }
    for (int g : {1, 148}) {
        auto tw = [&](const char* name, auto kern, int n) {
            cudaMemset(flush, 1, 256 << 20);
            kern<<<g, 128>>>(1.0f, d_out, sink);
            long long hh[296];
            cudaMemcpy(hh, d_out, 2 * g * 8, cudaMemcpyDeviceToHost);
            double a = 0, b = 0;
            for (int i = 0; i < g; ++i) { a += hh[2 * i]; b += hh[2 * i + 1]; }
            printf("%-28s grid %3d: pass 1 %.2f cyc/instr, pass 2 %.2f cyc/instr\n", name, g, a / g / n, b / g / n);
        };
        tw("twice 512 instr", twice<1>, 512);
        tw("twice 2048 instr", twice<4>, 2048);
        tw("twice 4096 instr", twice<8>, 4096);
        tw("twice 8192 instr", twice<16>, 8192);
    }
    return 0;
}
