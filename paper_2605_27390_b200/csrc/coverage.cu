// coverage.cu -- N4: coverage of the active vocabulary V_t
// against a target distribution: the covered mass of Eq. 2's constraint
// "sum_{x in V_t} p >= 1 - eps_cov" and Appendix E's covered
// probability mass and Recall@k.
//
// Row r (one CTA per row): p_r(v) = exp(z_r[v] it - m_r) / s_r over [0, V),
// fp64; mass_r = sum_{v in S} p_r(v); recall_r[k] = |S n top-k(p_r)| / k with
// top-k by (p desc, id asc) -- p orders as the fp32 logit (it > 0), so the
// top-k boundary is found exactly on the logits: one block radix select (8-bit
// digits of the monotone float key, 4 passes) gives the K-th largest key tau for
// K = max(ks); among the elements equal to tau the smaller ids win (a second
// radix select on ~id over the tied elements, only when the boundary is tied).
// The K elements above the boundary are ranked exactly by counting and tested
// for membership in S by binary search; Recall@k is a prefix count over ranks.
// HBM: V fp32 per row once (the further passes hit L2) plus the n_S gathered
// logits.
#include "common.cuh"
#include "kernels.cuh"

namespace es {

constexpr int kCovThreads = 1024;
constexpr int kCovWarps = kCovThreads / 32;

constexpr int kCovMaxK = 1024;   // largest k of Recall@k (the header's bound)

struct CovSmem {
    uint32_t hist[256];
    uint32_t top_key[kCovMaxK];
    int top_id[kCovMaxK];
    int hit_at[kCovMaxK];
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
            __syncwarp();                // every lane has read s_need before one lane updates it
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
                const int32_t* __restrict__ ks, int n_ks, double* __restrict__ mass, double* __restrict__ recall,
                int* __restrict__ flags) {
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
    // 3. Recall@k: ONE selection of the K = max(ks) boundary (tau, iota); the (at
    //    most kCovMaxK) elements above it are gathered, ranked exactly by counting
    //    under (key desc, id asc), tested for membership in S by binary search, and
    //    Recall@k for every k is the member count among ranks < k.
    if (n_ks == 0) return;
    int K = 0;
    for (int t = 0; t < n_ks; ++t) K = max(K, __ldg(&ks[t]));
    if (K < 1 || K > kCovMaxK || K > V) {   // outside the header's range: NaN
        if (tid < n_ks) recall[(size_t)r * n_ks + tid] = __longlong_as_double(0x7ff8000000000000ll);
        if (tid == 0 && flags) atomicOr(flags, kFlagBadIds);
        return;
    }
    const uint32_t tau = cov_select(V, K, [&](int v, uint32_t& key) { key = float_key(__ldg(&zr[v])); return true; }, sm);
    int gt = 0, eq = 0;
    for (int v = tid; v < V; v += kCovThreads) {
        const uint32_t key = float_key(__ldg(&zr[v]));
        gt += key > tau;
        eq += key == tau;
    }
    gt = cov_block_count(gt, sm);
    eq = cov_block_count(eq, sm);
    uint32_t iota = 0xFFFFFFFFu;   // tied at tau: the (K - gt) smallest ids win
    if (eq > K - gt) {
        const uint32_t t2 = cov_select(V, K - gt, [&](int v, uint32_t& key) {
            key = 0xFFFFFFFFu - (uint32_t)v;
            return float_key(__ldg(&zr[v])) == tau;
        }, sm);
        iota = 0xFFFFFFFFu - t2;
    }
    if (tid == 0) sm.s_cnt = 0;
    __syncthreads();
    for (int v = tid; v < V; v += kCovThreads) {
        const uint32_t key = float_key(__ldg(&zr[v]));
        if (key > tau || (key == tau && (uint32_t)v <= iota)) {
            const int slot = atomicAdd(&sm.s_cnt, 1);
            if (slot < kCovMaxK) { sm.top_key[slot] = key; sm.top_id[slot] = v; }
        }
    }
    __syncthreads();
    const int nt = min(sm.s_cnt, kCovMaxK);   // == K
    for (int i = tid; i < kCovMaxK; i += kCovThreads) sm.hit_at[i] = 0;
    __syncthreads();
    for (int i = tid; i < nt; i += kCovThreads) {
        const uint32_t ki = sm.top_key[i];
        const int vi = sm.top_id[i];
        int rank = 0;
        for (int j = 0; j < nt; ++j) {
            const uint32_t kj = sm.top_key[j];
            rank += kj > ki || (kj == ki && sm.top_id[j] < vi);
        }
        int lo = 0, hi = n_S;   // membership of vi in the sorted S
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(&S[mid]) < vi) lo = mid + 1; else hi = mid;
        }
        sm.hit_at[rank] = (lo < n_S && __ldg(&S[lo]) == vi) ? 1 : 0;
    }
    __syncthreads();
    if (wid == 0) {   // prefix counts over ranks, one lane per k
        for (int t = lane; t < n_ks; t += 32) {
            const int k = __ldg(&ks[t]);
            if (k < 1) {   // (k > K cannot happen: K is the maximum)
                recall[(size_t)r * n_ks + t] = __longlong_as_double(0x7ff8000000000000ll);
                if (flags) atomicOr(flags, kFlagBadIds);
                continue;
            }
            int hit = 0;
            for (int i = 0; i < k; ++i) hit += sm.hit_at[i];
            recall[(size_t)r * n_ks + t] = (double)hit / (double)k;
        }
    }
}

void launch_coverage(const float* z, int n_rows, int V, const int32_t* S, int n_S, double it, const int32_t* ks,
                     int n_ks, double* mass, double* recall, int* flags, cudaStream_t st) {
    launch_pdl(coverage_kernel, dim3(n_rows), dim3(kCovThreads), 0, st, z, V, S, n_S, it, ks, n_ks, mass, recall,
               flags);
}

}  // namespace es
