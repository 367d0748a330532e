// Isolated timing of the LM-head finalisation (fin64.cuh) on synthetic partial
// lists shaped like the llama draft step (148 lists x 60 rows, ~20 buffered
// candidates per list, gid keys), with its clock64 phase stamps (profiling aid).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I paper_2605_27390_b200/csrc -o /tmp/fin_iso tools/ubench/fin_iso.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <cmath>
#include <algorithm>
#include <functional>
#include "fin64.cuh"
using namespace es;

int main(int argc, char** argv) {
    const int n_cta = 148, n_h = 60, k = 10, KP = 18, d = 4096, V = 32768;
    const int LS = 64;
    std::mt19937 rng(1);
    std::normal_distribution<float> nd(0.f, 1.28f);
    std::vector<float> val((size_t)n_cta * n_h * LS, -INFINITY), m(n_cta * n_h), s(n_cta * n_h);
    std::vector<int> id((size_t)n_cta * n_h * LS, 0), cnt(n_cta * n_h, 0), xcnt(n_cta * n_h);
    for (int c = 0; c < n_cta; ++c)
        for (int r = 0; r < n_h; ++r) {
            const size_t o = (size_t)c * n_h + r, so = (size_t)r * n_cta + c;   // lists [cta][row], state [row][cta]
            // the list: the CTA's 249 values' best ~25 (a gaussian sample, sorted desc)
            std::vector<float> x(249);
            for (auto& v : x) v = nd(rng);
            std::sort(x.begin(), x.end(), std::greater<float>());
            const int nc = 20 + (int)(rng() % 10);
            for (int i = 0; i < nc; ++i) { val[o * LS + i] = x[i]; id[o * LS + i] = (int)(rng() % V); }
            std::swap(val[o * LS], val[o * LS + nc / 2]);   // unsorted buffer, max somewhere
            std::swap(id[o * LS], id[o * LS + nc / 2]);
            m[so] = x[0];
            double ss = 0; for (float v : x) ss += std::exp(v - x[0]);
            s[so] = (float)ss;
            xcnt[so] = nc;
        }
    LmhArgs a{};
    float *dv, *dm, *ds, *wmax; int *di, *dc, *dx, *flags;
    cudaMalloc(&dv, val.size() * 4); cudaMalloc(&di, id.size() * 4); cudaMalloc(&dm, m.size() * 4);
    cudaMalloc(&ds, s.size() * 4); cudaMalloc(&dc, cnt.size() * 4); cudaMalloc(&dx, xcnt.size() * 4);
    cudaMemcpy(dv, val.data(), val.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(di, id.data(), id.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dm, m.data(), m.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, s.data(), s.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dc, cnt.data(), cnt.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dx, xcnt.data(), xcnt.size() * 4, cudaMemcpyHostToDevice);
    void *W, *H; cudaMalloc(&W, (size_t)V * d * 2); cudaMalloc(&H, (size_t)n_h * d * 2);
    cudaMemset(W, 0x3c, (size_t)V * d * 2); cudaMemset(H, 0x3c, (size_t)n_h * d * 2);
    cudaMalloc(&wmax, 4); float wm = 1.4f; cudaMemcpy(wmax, &wm, 4, cudaMemcpyHostToDevice);
    cudaMalloc(&flags, 4); cudaMemset(flags, 0, 4);
    long long* trace; cudaMalloc(&trace, 8 * 4096); cudaMemset(trace, 0, 8 * 4096);
    int32_t* ids; float *vals, *rm, *rs; cudaMalloc(&ids, n_h * k * 4); cudaMalloc(&vals, n_h * k * 4);
    cudaMalloc(&rm, n_h * 4); cudaMalloc(&rs, n_h * 4);
    a.W = W; a.d = d; a.w_dtype = 0; a.H = H; a.n_h = n_h; a.h_dtype = 0; a.R = 1; a.KP = KP; a.LS = LS;
    a.inv_temp = 1.0f; a.part = LmhPartials{dv, di, dm, ds, dc, dx, n_cta}; a.fin_opt = 15; a.gid_keys = 1;
    a.trace = trace;
    // gamma: make runs frequent (~ the LM head's 2^-16 envelope scaled to these values)
    const float gamma = argc > 1 ? atof(argv[1]) : 1.0f / 65536.0f;
    auto kern = lmh_fin64_kernel<256>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(e0);
        kern<<<n_h, 256, 120 * 1024>>>(a, n_cta, k, gamma, wmax, ids, vals, rm, rs, flags);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        std::vector<long long> t(4096);
        cudaMemcpy(t.data(), trace, 8 * 4096, cudaMemcpyDeviceToHost);
        long long g0 = 1LL << 62, g1 = 0;
        for (int r = 0; r < n_h; ++r) { g0 = std::min(g0, t[148 * 8 + r * 8]); g1 = std::max(g1, t[148 * 8 + r * 8 + 6]); }
        const long long* dt = &t[2 * 148 * 8 + 16];
        printf("rep %d: event %.1f us, rows start->end max %.2f us, row0 cycles:", rep, ms * 1e3, (g1 - g0) / 1e3);
        for (int i = 1; i <= 6; ++i) printf(" %lld", dt[i] - dt[0]);
        printf("  ncand0 %lld err %s\n", t[148 * 8 + 7], cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
