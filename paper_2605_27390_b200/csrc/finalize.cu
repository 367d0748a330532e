// finalize.cu -- per-shard finalisation of the LM-head partials (a6/a7),
// the vocab-shard merge (a8), and two off-path helpers.
//
// lmh_finalize_kernel (one CTA per H row):
//   1. combine the per-CTA online-softmax states: M = max m_c,
//      s = sum_c s_c exp(m_c - M);
//   2. k-way merge of the per-CTA sorted fp32 candidate lists into the best
//      KP = k + kTopkPad candidates under (z desc, id asc);
//   3. EXACT re-score of those KP candidates in fp64 (bf16 x bf16 / fp32
//      products are exact in fp64) and re-order by (z64 desc, id asc);
//   4. certification: every candidate that was dropped has fp32 value
//      <= v_KP, hence exact value <= v_KP + delta; if the k-th exact value
//      exceeds v_KP + delta the returned top-k is the exact top-k
//      (DESIGN.md "Exact top-k"); otherwise EVOSPEC_FLAG_UNCERTIFIED is set.
//      delta = gamma * ||h_r||_2 * max_v ||W_v||_2 * inv_temp, gamma the
//      accumulation-error constant of the kernel that produced the fp32 values.
// merge_kernel (one warp per H row): the shard merge of SURVEY §8(c) step 12.
#include "common.cuh"
#include "kernels.cuh"

namespace es {

constexpr int kFinThreads = 256;

__global__ void __launch_bounds__(kFinThreads)
lmh_finalize_kernel(LmhArgs a, int n_cta, int k, float gamma, const float* __restrict__ wmax_dev,
                    int32_t* __restrict__ topk_ids, float* __restrict__ topk_vals,
                    float* __restrict__ row_max, float* __restrict__ row_sumexp, int* flags) {
    const int r = blockIdx.x;
    const int KP = a.KP;
    const int lane = lane_id(), warp = warp_id(), nwarps = blockDim.x / 32;
    extern __shared__ unsigned char f_sm[];
    int* head = (int*)f_sm;                         // [n_cta]
    __shared__ float c_v32[kMaxKP];
    __shared__ int32_t c_id[kMaxKP];
    __shared__ double c_e[kMaxKP];
    __shared__ int n_kept_s, total_s;
    __shared__ float red_m[32], red_s[32];
    __shared__ int red_t[32];
    __shared__ double hn2_s;

    // 1. softmax state
    float M = -INFINITY;
    for (int c = threadIdx.x; c < n_cta; c += blockDim.x) {
        size_t o = (size_t)c * a.n_h + r;
        if (a.part.s[o] > 0.0f) M = fmaxf(M, a.part.m[o]);
        head[c] = 0;
    }
    M = warp_max(M);
    if (lane == 0) red_m[warp] = M;
    __syncthreads();
    M = -INFINITY;
    for (int w = 0; w < nwarps; ++w) M = fmaxf(M, red_m[w]);
    float S = 0.0f;
    int tot = 0;
    for (int c = threadIdx.x; c < n_cta; c += blockDim.x) {
        size_t o = (size_t)c * a.n_h + r;
        float sc = a.part.s[o];
        if (sc > 0.0f) S += sc * expf(a.part.m[o] - M);
        tot += a.part.cnt[o];
    }
    S = warp_sum(S);
    tot = warp_sum_i(tot);
    if (lane == 0) { red_s[warp] = S; red_t[warp] = tot; }
    __syncthreads();
    if (threadIdx.x == 0) {
        float s_all = 0.0f;
        int t_all = 0;
        for (int w = 0; w < nwarps; ++w) { s_all += red_s[w]; t_all += red_t[w]; }
        row_max[r] = M;
        row_sumexp[r] = s_all;
        total_s = t_all;
    }
    // 2. k-way merge (warp 0)
    if (warp == 0) {
        int produced = 0;
        for (; produced < KP; ++produced) {
            float bv = -INFINITY;
            int bid = 0x7fffffff;
            for (int c = lane; c < n_cta; c += 32) {
                size_t o = (size_t)c * a.n_h + r;
                int h = head[c];
                if (h < a.part.cnt[o]) {
                    float v = a.part.val[o * KP + h];
                    int id = a.part.id[o * KP + h];
                    if (before(v, id, bv, bid)) { bv = v; bid = id; }
                }
            }
            warp_argbest(bv, bid);
            if (bid == 0x7fffffff) break;
            for (int c = lane; c < n_cta; c += 32) {
                size_t o = (size_t)c * a.n_h + r;
                int h = head[c];
                if (h < a.part.cnt[o] && a.part.id[o * KP + h] == bid) head[c] = h + 1;
            }
            if (lane == 0) { c_v32[produced] = bv; c_id[produced] = bid; }
            __syncwarp();
        }
        if (lane == 0) n_kept_s = produced;
    }
    __syncthreads();
    const int nk = n_kept_s;
    // 3. exact re-score + ||h_r||^2
    const int d = a.d;
    const int welems = a.w_dtype == 0 ? 8 : 4;
    for (int c = warp; c <= nk; c += nwarps) {
        double acc = 0.0;
        if (c < nk) {
            const int64_t row = c_id[c] / a.R;
            for (int c0 = lane * welems; c0 < d; c0 += 32 * welems) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (j >= welems) break;
                    const int col = c0 + j;
                    double w = a.w_dtype == 0 ? (double)bf16_bits_to_f32(((const uint16_t*)a.W)[row * d + col])
                                              : (double)((const float*)a.W)[row * d + col];
                    double h = a.h_dtype == 0 ? (double)bf16_bits_to_f32(((const uint16_t*)a.H)[(size_t)r * d + col])
                                              : (double)((const float*)a.H)[(size_t)r * d + col];
                    acc = fma(w, h, acc);
                }
            }
        } else {  // the extra "candidate" nk computes ||h_r||^2
            for (int col = lane; col < d; col += 32) {
                double h = a.h_dtype == 0 ? (double)bf16_bits_to_f32(((const uint16_t*)a.H)[(size_t)r * d + col])
                                          : (double)((const float*)a.H)[(size_t)r * d + col];
                acc = fma(h, h, acc);
            }
        }
        acc = warp_sum_d(acc);
        if (lane == 0) {
            if (c < nk) c_e[c] = acc * (double)a.inv_temp;
            else hn2_s = acc;
        }
    }
    __syncthreads();
    // 4. order by exact value, certify, write
    if (threadIdx.x == 0) {
        const float v_last = nk > 0 ? c_v32[nk - 1] : -INFINITY;
        for (int i = 1; i < nk; ++i) {
            double e = c_e[i];
            int32_t id = c_id[i];
            float v = c_v32[i];
            int j = i - 1;
            while (j >= 0 && before(e, id, c_e[j], c_id[j])) {
                c_e[j + 1] = c_e[j]; c_id[j + 1] = c_id[j]; c_v32[j + 1] = c_v32[j];
                --j;
            }
            c_e[j + 1] = e; c_id[j + 1] = id; c_v32[j + 1] = v;
        }
        const bool dropped = total_s > nk;
        if (dropped && nk >= k) {
            const double wmax = (double)*wmax_dev;
            const double delta = (double)gamma * sqrt(hn2_s) * wmax * (double)a.inv_temp +
                                 fabs((double)v_last) * 2.4e-7;
            if (!(c_e[k - 1] > (double)v_last + delta)) atomicOr(flags, kFlagUncertified);
        }
        for (int i = 0; i < k; ++i) {
            topk_ids[(size_t)r * k + i] = i < nk ? c_id[i] : -1;
            topk_vals[(size_t)r * k + i] = i < nk ? (float)c_e[i] : -INFINITY;
        }
    }
}

void launch_lmh_finalize(const LmhArgs& a, int n_cta, int k, const float* wmax_dev, int32_t* topk_ids,
                         float* topk_vals, float* row_max, float* row_sumexp, int* flags, cudaStream_t st,
                         float gamma) {
    size_t smem = (size_t)n_cta * sizeof(int);
    lmh_finalize_kernel<<<a.n_h, kFinThreads, smem, st>>>(a, n_cta, k, gamma, wmax_dev, topk_ids, topk_vals,
                                                           row_max, row_sumexp, flags);
}

// ------------------------------------------------------------ shard merge
__global__ void __launch_bounds__(256)
merge_kernel(int R, int n_h, int k, const int32_t* __restrict__ ids, const float* __restrict__ vals,
             const float* __restrict__ m, const float* __restrict__ s, int32_t* __restrict__ out_ids,
             float* __restrict__ out_vals, float* __restrict__ out_lse, float* __restrict__ out_probs) {
    const int r = blockIdx.x * (blockDim.x / 32) + warp_id();
    if (r >= n_h) return;
    const int lane = lane_id();
    float M = -INFINITY;
    for (int t = 0; t < R; ++t) {
        float st = s[(size_t)t * n_h + r];
        if (st > 0.0f) M = fmaxf(M, m[(size_t)t * n_h + r]);
    }
    float sig = 0.0f;
    for (int t = 0; t < R; ++t) {
        float st = s[(size_t)t * n_h + r];
        if (st > 0.0f) sig += st * expf(m[(size_t)t * n_h + r] - M);
    }
    const float L = sig > 0.0f ? M + logf(sig) : -INFINITY;
    if (lane == 0 && out_lse) out_lse[r] = L;
    const int nc = R * k;
    unsigned long long taken = 0;  // per-lane bitmask over its candidates (<= 64 per lane)
    for (int i = 0; i < k; ++i) {
        float bv = -INFINITY;
        int bid = 0x7fffffff, bslot = -1;
        for (int c = lane, q = 0; c < nc; c += 32, ++q) {
            if ((taken >> q) & 1ull) continue;
            const int t = c / k, j = c % k;
            const size_t o = ((size_t)t * n_h + r) * k + j;
            const int id = ids[o];
            if (id < 0) continue;
            const float v = vals[o];
            if (before(v, id, bv, bid)) { bv = v; bid = id; bslot = q; }
        }
        float wv = bv;
        int wid = bid;
        warp_argbest(wv, wid);
        if (wid != 0x7fffffff && wid == bid && bslot >= 0 && wv == bv) taken |= 1ull << bslot;
        if (lane == 0) {
            const size_t o = (size_t)r * k + i;
            out_ids[o] = wid == 0x7fffffff ? -1 : wid;
            out_vals[o] = wid == 0x7fffffff ? -INFINITY : wv;
            if (out_probs) out_probs[o] = wid == 0x7fffffff ? 0.0f : expf(wv - L);
        }
    }
}

void launch_merge(int R, int n_h, int k, const int32_t* ids, const float* vals, const float* m,
                  const float* s, int32_t* out_ids, float* out_vals, float* out_lse, float* out_probs,
                  cudaStream_t st) {
    const int grid = (n_h + 7) / 8;
    merge_kernel<<<grid, 256, 0, st>>>(R, n_h, k, ids, vals, m, s, out_ids, out_vals, out_lse, out_probs);
}

// ------------------------------------------------------------ helpers
// max_v ||W_v||_2 (setup time, once per weight tensor), rounded up.
__global__ void rownorm_max_kernel(const void* __restrict__ W, int w_dtype, int64_t n_rows, int d,
                                   float* __restrict__ out) {
    const int lane = lane_id();
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) / 32;
    float best = 0.0f;
    for (int64_t row = gw; row < n_rows; row += nw) {
        double acc = 0.0;
        for (int c = lane; c < d; c += 32) {
            double w = w_dtype == 0 ? (double)bf16_bits_to_f32(((const uint16_t*)W)[row * d + c])
                                    : (double)((const float*)W)[row * d + c];
            acc += w * w;
        }
        acc = warp_sum_d(acc);
        best = fmaxf(best, (float)(sqrt(acc) * (1.0 + 1e-6)));
    }
    if (lane == 0) atomicMax((int*)out, __float_as_int(best));   // non-negative floats order as ints
}

void launch_rownorm_max(const void* W, int w_dtype, int64_t n_rows, int d, float* out, cudaStream_t st) {
    cudaMemsetAsync(out, 0, sizeof(float), st);
    rownorm_max_kernel<<<kNumSMs * 4, 256, 0, st>>>(W, w_dtype, n_rows, d, out);
}

// debug: ids sorted strictly ascending and inside [0, V)
__global__ void check_sorted_kernel(const int32_t* __restrict__ ids, const int* __restrict__ n_dev, int n_host,
                                    int V, int* flags) {
    const int n = n_dev ? min(*n_dev, n_host) : n_host;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int v = ids[i];
        if (v < 0 || v >= V || (i > 0 && ids[i - 1] >= v)) atomicOr(flags, 1);
    }
}

void launch_check_sorted(const int32_t* ids, const int* n_dev, int n_host, int V, int* flags, cudaStream_t st) {
    check_sorted_kernel<<<kNumSMs, 256, 0, st>>>(ids, n_dev, n_host, V, flags);
}

}  // namespace es
