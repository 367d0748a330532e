// coverage.cu -- N4: coverage of the active vocabulary V_t
// against a target distribution: the covered mass of Eq. 2's constraint
// "sum_{x in V_t} p >= 1 - eps_cov" and Appendix E's covered
// probability mass and Recall@k.
//
// Row r (one CTA per row): p_r(v) = exp(z_r[v] it - m_r) / s_r over [0, V),
// fp64; mass_r = sum_{v in S} p_r(v); recall_r[k] = |S n top-k(p_r)| / k with
// top-k by (p desc, id asc) -- p orders as the fp32 logit (it > 0), so the
// top-k boundary is found exactly on the logits: a block radix select (8-bit
// digits of the monotone float key, 4 passes) gives the k-th largest key tau;
// among the elements equal to tau the smaller ids win, found by a second radix
// select on ~id over the tied elements only when the boundary is tied. Then one
// pass over S counts its members above the boundary. HBM: V fp32 per row once
// (the further passes hit L2) plus the n_S gathered logits.
#include "common.cuh"
#include "kernels.cuh"

namespace es {

constexpr int kCovThreads = 1024;
constexpr int kCovWarps = kCovThreads / 32;

struct CovSmem {
    uint32_t hist[256];
    double red_d[kCovWarps];
    float red_f[kCovWarps];
    int red_i[kCovWarps];
    double s_d;
    float s_f;
    uint32_t s_prefix, s_mask;
    int s_need, s_cnt;
};

ES_DEV double cov_block_sum(double v, CovSmem& sm) {
    const int lane = lane_id(), wid = warp_id();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sm.red_d[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = lane < kCovWarps ? sm.red_d[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) sm.s_d = t;
    }
    __syncthreads();
    const double r = sm.s_d;
    __syncthreads();
    return r;
}

ES_DEV int cov_block_count(int v, CovSmem& sm) {
    const int lane = lane_id(), wid = warp_id();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sm.red_i[wid] = v;
    __syncthreads();
    if (wid == 0) {
        int t = lane < kCovWarps ? sm.red_i[lane] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) sm.s_cnt = t;
    }
    __syncthreads();
    const int r = sm.s_cnt;
    __syncthreads();
    return r;
}

// The K-th largest 32-bit key (1 <= K <= participants) among the participating
// elements of [0, V): KEY(v, &key) returns whether v participates. 4 passes of
// 8-bit digits, most significant first.
template <typename KeyFn>
ES_DEV uint32_t cov_select(int V, int K, KeyFn KEY, CovSmem& sm) {
    const int tid = threadIdx.x, lane = lane_id();
    if (tid == 0) { sm.s_prefix = 0u; sm.s_mask = 0u; sm.s_need = K; }
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        for (int b = tid; b < 256; b += kCovThreads) sm.hist[b] = 0u;
        __syncthreads();
        const uint32_t prefix = sm.s_prefix, mask = sm.s_mask;
        for (int v = tid; v < V; v += kCovThreads) {
            uint32_t key;
            if (KEY(v, key) && (key & mask) == prefix) atomicAdd(&sm.hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (tid < 32) {   // one warp: 8 bins per lane, descending
            uint32_t c[8], tot = 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) { c[i] = sm.hist[255 - (lane * 8 + i)]; tot += c[i]; }
            uint32_t incl = tot;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += t;
            }
            uint32_t run = incl - tot;   // count in the bins above this lane's
            const int need = sm.s_need;
            for (int i = 0; i < 8; ++i) {
                if ((int)run < need && (int)(run + c[i]) >= need) {
                    const uint32_t bin = 255u - (uint32_t)(lane * 8 + i);
                    sm.s_prefix = prefix | (bin << shift);
                    sm.s_mask = mask | (255u << shift);
                    sm.s_need = need - (int)run;
                }
                run += c[i];
            }
        }
        __syncthreads();
    }
    const uint32_t tau = sm.s_prefix;
    __syncthreads();
    return tau;
}

__global__ void __launch_bounds__(kCovThreads)
coverage_kernel(const float* __restrict__ z, int V, const int32_t* __restrict__ S, int n_S, double it,
                const int32_t* __restrict__ ks, int n_ks, double* __restrict__ mass, double* __restrict__ recall) {
    __shared__ CovSmem sm;
    pdl_trigger();
    pdl_wait();
    const int r = blockIdx.x, tid = threadIdx.x, lane = lane_id(), wid = warp_id();
    const float* zr = z + (size_t)r * V;
    // 1. maximum, fp32 (orders as the fp64 product with it > 0)
    float mx = -INFINITY;
    for (int v = tid; v < V; v += kCovThreads) mx = fmaxf(mx, __ldg(&zr[v]));
    mx = warp_max(mx);
    if (lane == 0) sm.red_f[wid] = mx;
    __syncthreads();
    if (wid == 0) {
        float t = lane < kCovWarps ? sm.red_f[lane] : -INFINITY;
        t = warp_max(t);
        if (lane == 0) sm.s_f = t;
    }
    __syncthreads();
    const double M = (double)sm.s_f * it;
    // 2. s and the covered mass, fp64
    double ls = 0.0;
    for (int v = tid; v < V; v += kCovThreads) ls += exp((double)__ldg(&zr[v]) * it - M);
    const double s = cov_block_sum(ls, sm);
    double lm = 0.0;
    for (int i = tid; i < n_S; i += kCovThreads) lm += exp((double)__ldg(&zr[__ldg(&S[i])]) * it - M);
    const double cm = cov_block_sum(lm, sm) / s;
    if (tid == 0) mass[r] = cm;
    // 3. Recall@k: the top-k boundary (tau, iota) and the members of S above it
    for (int t = 0; t < n_ks; ++t) {
        const int K = __ldg(&ks[t]);
        const uint32_t tau = cov_select(V, K, [&](int v, uint32_t& key) { key = float_key(__ldg(&zr[v])); return true; }, sm);
        int gt = 0, eq = 0;
        for (int v = tid; v < V; v += kCovThreads) {
            const uint32_t key = float_key(__ldg(&zr[v]));
            gt += key > tau;
            eq += key == tau;
        }
        gt = cov_block_count(gt, sm);
        eq = cov_block_count(eq, sm);
        // tied at tau: the (K - gt) smallest ids win -- iota = the largest winning id
        uint32_t iota = 0xFFFFFFFFu;
        if (eq > K - gt) {
            const uint32_t t2 = cov_select(V, K - gt, [&](int v, uint32_t& key) {
                key = 0xFFFFFFFFu - (uint32_t)v;
                return float_key(__ldg(&zr[v])) == tau;
            }, sm);
            iota = 0xFFFFFFFFu - t2;
        }
        int hit = 0;
        for (int i = tid; i < n_S; i += kCovThreads) {
            const int v = __ldg(&S[i]);
            const uint32_t key = float_key(__ldg(&zr[v]));
            hit += key > tau || (key == tau && (uint32_t)v <= iota);
        }
        hit = cov_block_count(hit, sm);
        if (tid == 0) recall[(size_t)r * n_ks + t] = (double)hit / (double)K;
    }
}

void launch_coverage(const float* z, int n_rows, int V, const int32_t* S, int n_S, double it, const int32_t* ks,
                     int n_ks, double* mass, double* recall, cudaStream_t st) {
    launch_pdl(coverage_kernel, dim3(n_rows), dim3(kCovThreads), 0, st, z, V, S, n_S, it, ks, n_ks, mass, recall);
}

}  // namespace es
