// finalize.cu -- per-shard finalisation of the LM-head partials (a6/a7),
// the vocab-shard merge (a8), and two off-path helpers.
//
// lmh_finalize_kernel (one CTA per H row):
//   1. combine the per-CTA online-softmax states: M = max m_c,
//      s = sum_c s_c exp(m_c - M);
//   2. k-way merge of the per-CTA sorted fp32 candidate lists into the best
//      KP = k + kTopkPad candidates under (z desc, id asc);
//   3. exactness: every fp32 value is within
//      delta = gamma * ||h_r||_2 * max_v ||W_v||_2 * inv_temp of the exact
//      value (gamma: accumulation-error constant of the producing kernel).
//      Consecutive kept candidates closer than 2*delta form a "run" whose
//      internal order is uncertain; every run that reaches into the top k is
//      re-scored EXACTLY in fp64 (bf16 x bf16 / fp32 products are exact in
//      fp64) and re-ordered by (z64 desc, id asc). Runs are separated by gaps
//      > 2*delta, so the order between runs is certain. If the run holding
//      the k-th candidate reaches the last kept candidate while candidates
//      were dropped, the result cannot be certified: EVOSPEC_FLAG_UNCERTIFIED.
// merge_kernel (one warp per H row): the shard merge of SURVEY §8(c) step 12.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "lmh_epilogue.cuh"   // warp_kth_largest
#include "fin64.cuh"       // lmh_fin64_kernel (k + 8 <= 32)

namespace es {

constexpr int kFinThreads = 256;

// profiling stamps (EVOSPEC_TRACE): slots [148*8 + row*8 + i]
// fine-grained clock64 stamps of row 0 (thread 0 / warp 0 lane 0), slots [2*148*8 + 16 + i]
#define FIN_DT(i) do { if (a.trace && blockIdx.x == 0) a.trace[2 * 148 * 8 + 16 + (i)] = clock64(); } while (0)
#define FIN_TRACE(slot) do { if (a.trace && blockIdx.x < 148) a.trace[148 * 8 + (size_t)blockIdx.x * 8 + (slot)] = fin_gtime(); } while (0)

ES_DEV double load_elem(const void* p, int dtype, size_t i) {
    return dtype == 0 ? (double)bf16_bits_to_f32(((const uint16_t*)p)[i]) : (double)((const float*)p)[i];
}

__global__ void __launch_bounds__(kFinThreads)
lmh_finalize_kernel(LmhArgs a, int n_cta, int k, float gamma, const float* __restrict__ wmax_dev,
                    int32_t* __restrict__ topk_ids, float* __restrict__ topk_vals,
                    float* __restrict__ row_max, float* __restrict__ row_sumexp, int* flags) {
    const int r = blockIdx.x;
    const int KP = a.KP;
    if (threadIdx.x == 0) FIN_TRACE(0);
    const int lane = lane_id(), warp = warp_id(), nwarps = blockDim.x / 32;
    extern __shared__ unsigned char f_sm[];
    int* head = (int*)f_sm;                         // [n_cta]
    int* l_cnt = head + n_cta;                      // [n_cta]
    float* l_val = (float*)(l_cnt + n_cta);         // [n_cta][KP]
    int32_t* l_id = (int32_t*)(l_val + (size_t)n_cta * KP);  // [n_cta][KP]
    __shared__ float c_v32[kMaxKP];
    __shared__ int32_t c_id[kMaxKP];
    __shared__ double c_e[kMaxKP];
    __shared__ int c_need[kMaxKP];
    __shared__ int n_kept_s, total_s, n_need_s;
    __shared__ int need_list[kMaxKP];
    __shared__ float red_m[32], red_s[32];
    __shared__ int red_t[32];
    __shared__ double hn2_s;
    __shared__ double red_d[32];

    // 1. softmax state; ||h_r||^2 (warp 7) for delta
    float M = -INFINITY;
    for (int c = threadIdx.x; c < n_cta; c += blockDim.x) {
        const size_t o = part_st(a.part, c, r);
        if (a.part.s[o] > 0.0f) M = fmaxf(M, a.part.m[o]);
        head[c] = 0;
    }
    M = warp_max(M);
    if (lane == 0) red_m[warp] = M;
    {   // ||h_r||^2 by all threads (independent loads), fp64
        double acc = 0.0;
        if (a.h_dtype == 0 && a.d % 8 == 0) {
            const uint4* hp = (const uint4*)((const uint16_t*)a.H + (size_t)r * a.d);
            for (int c = threadIdx.x; c < a.d / 8; c += blockDim.x) {
                float f[8];
                unpack_bf16x8(hp[c], f);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc = fma((double)f[j], (double)f[j], acc);
            }
        } else {
            for (int col = threadIdx.x; col < a.d; col += blockDim.x) {
                const double h = load_elem(a.H, a.h_dtype, (size_t)r * a.d + col);
                acc = fma(h, h, acc);
            }
        }
        acc = warp_sum_d(acc);
        if (lane == 0) red_d[warp] = acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) FIN_TRACE(1);
    if (threadIdx.x == 0) {
        double hn = 0.0;
        for (int w = 0; w < nwarps; ++w) hn += red_d[w];
        hn2_s = hn;
    }
    M = -INFINITY;
    for (int w = 0; w < nwarps; ++w) M = fmaxf(M, red_m[w]);
    float S = 0.0f;
    int tot = 0;
    for (int c = threadIdx.x; c < n_cta; c += blockDim.x) {
        const size_t o = part_st(a.part, c, r);
        float sc = a.part.s[o];
        if (sc > 0.0f) S += sc * expf(a.part.m[o] - M);
        tot += a.part.cnt[o];
    }
    S = warp_sum(S);
    tot = warp_sum_i(tot);
    if (lane == 0) { red_s[warp] = S; red_t[warp] = tot; }
    // stage every CTA's sorted list in shared memory: flat, 4 independent loads
    // in flight per thread (entries past a list's count are -inf / -1)
    for (int c = threadIdx.x; c < n_cta; c += blockDim.x) l_cnt[c] = a.part.cnt[part_st(a.part, c, r)];
    for (int f0 = 0; f0 < n_cta * KP; f0 += 4 * blockDim.x) {
        float vv[4];
        int32_t ii[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int f = f0 + u * blockDim.x + threadIdx.x;
            const int c = f / KP, i = f - c * KP;
            const size_t o = ((size_t)c * a.n_h + r) * KP + i;
            vv[u] = f < n_cta * KP ? __ldcg(&a.part.val[o]) : -INFINITY;
            ii[u] = f < n_cta * KP ? __ldcg(&a.part.id[o]) : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int f = f0 + u * blockDim.x + threadIdx.x;
            if (f < n_cta * KP) { l_val[f] = vv[u]; l_id[f] = ii[u]; }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) FIN_TRACE(2);
    if (threadIdx.x == 0) {
        float s_all = 0.0f;
        int t_all = 0;
        for (int w = 0; w < nwarps; ++w) { s_all += red_s[w]; t_all += red_t[w]; }
        row_max[r] = M;
        row_sumexp[r] = s_all;
        total_s = t_all;
    }
    // 2. the best KP of the per-CTA sorted lists (warp 0)
    if (warp == 0 && KP <= 32) {
        // pre-threshold: KP-th largest of the lane maxima of the list heads (a lower
        // bound of the KP-th best entry); entries >= it are inserted into a sorted
        // register list (lane i = entry i) by ballot rank + shfl_up shift.
        float lm = -INFINITY;
        for (int c = lane; c < n_cta; c += 32)
            if (l_cnt[c] > 0) lm = fmaxf(lm, l_val[(size_t)c * KP]);
        const float th0 = warp_kth_largest(lm, KP);
        float Lv = -INFINITY, tv = -INFINITY;
        int Lid = 0x7fffffff, tid_ = 0x7fffffff, cnt = 0;
        for (int c0 = 0; c0 < n_cta; c0 += 32) {
            const int c = c0 + lane;
            const int len = c < n_cta ? l_cnt[c] : 0;
            for (int i = 0;; ++i) {
                const bool has = i < len && l_val[(size_t)c * KP + i] >= th0;
                const float x = has ? l_val[(size_t)c * KP + i] : 0.0f;
                const int xid = has ? l_id[(size_t)c * KP + i] : 0;
                unsigned m = __ballot_sync(0xffffffffu, has);
                if (!m) break;
                while (m) {
                    const int src = __ffs(m) - 1;
                    m &= m - 1;
                    const float xv = __shfl_sync(0xffffffffu, x, src);
                    const int xi = __shfl_sync(0xffffffffu, xid, src);
                    if (cnt == KP && !before(xv, xi, tv, tid_)) continue;
                    const int at = __popc(__ballot_sync(0xffffffffu, lane < cnt && before(Lv, Lid, xv, xi)));
                    const float pv = __shfl_up_sync(0xffffffffu, Lv, 1);
                    const int pi = __shfl_up_sync(0xffffffffu, Lid, 1);
                    if (lane > at) { Lv = pv; Lid = pi; }
                    if (lane == at) { Lv = xv; Lid = xi; }
                    cnt = min(cnt + 1, KP);
                    if (cnt == KP) { tv = __shfl_sync(0xffffffffu, Lv, KP - 1); tid_ = __shfl_sync(0xffffffffu, Lid, KP - 1); }
                }
            }
        }
        if (lane < cnt) { c_v32[lane] = Lv; c_id[lane] = Lid; }
        if (lane == 0) n_kept_s = cnt;
    } else if (warp == 0) {   // KP > 32: k-way merge of the list heads
        int produced = 0;
        for (; produced < KP; ++produced) {
            float bv = -INFINITY;
            int bid = 0x7fffffff;
            int bc = -1;
            for (int c = lane; c < n_cta; c += 32) {
                const int h = head[c];
                if (h < l_cnt[c]) {
                    const float v = l_val[(size_t)c * KP + h];
                    const int id = l_id[(size_t)c * KP + h];
                    if (before(v, id, bv, bid)) { bv = v; bid = id; bc = c; }
                }
            }
            const int my_id = bid;
            warp_argbest(bv, bid);
            if (bid == 0x7fffffff) break;
            if (bc >= 0 && my_id == bid) head[bc] += 1;   // ids are unique: one owner
            if (lane == 0) { c_v32[produced] = bv; c_id[produced] = bid; }
            __syncwarp();
        }
        if (lane == 0) n_kept_s = produced;
    }
    __syncthreads();
    if (threadIdx.x == 0) FIN_TRACE(3);
    const int nk = n_kept_s;
    // 3. runs of candidates closer than 2 delta that reach into the top k
    if (threadIdx.x == 0) {
        const double delta = (double)gamma * sqrt(hn2_s) * (double)*wmax_dev * (double)a.inv_temp;
        int nn = 0;
        int i = 0;
        bool uncertain = false;
        while (i < nk) {
            int j = i;
            while (j + 1 < nk && (double)c_v32[j] - (double)c_v32[j + 1] <= 2.0 * delta + 2.4e-7 * fabs((double)c_v32[j]))
                ++j;
            const bool in_topk = i < k;
            const bool multi = j > i;
            // exact_vals (the triple feeds a merge across shards / parts): every top-k entry
            // is re-scored, so the merge compares the exact logits (rounded to fp32)
            for (int t = i; t <= j; ++t) {
                const bool nd = (in_topk && multi) || (a.exact_vals && t < k);
                c_need[t] = nd ? 1 : 0;
                if (nd) need_list[nn++] = t;
            }
            if (in_topk && j == nk - 1 && total_s > nk && j >= k - 1) uncertain = true;
            if (!(delta >= 0.0) || isinf(delta)) uncertain = true;   // weights not prepared
            i = j + 1;
        }
        n_need_s = nn;
        if (uncertain) atomicOr(flags, kFlagUncertified);
    }
    __syncthreads();
    if (threadIdx.x == 0) FIN_TRACE(4);
    // exact re-score of the flagged candidates (one warp per candidate)
    const int nn = n_need_s;
    for (int q = warp; q < nn; q += nwarps) {
        const int c = need_list[q];
        const size_t row = (size_t)(lmh_id_at(a, c_id[c]) / a.R);
        double acc = 0.0;
        if (a.w_dtype == 0 && a.h_dtype == 0 && a.d % 8 == 0) {   // 16-byte loads, 4 in flight per lane
            const uint4* wp = (const uint4*)((const uint16_t*)a.W + row * a.d);
            const uint4* hp = (const uint4*)((const uint16_t*)a.H + (size_t)r * a.d);
            const int nc = a.d / 8;
            for (int c0 = lane; c0 < nc; c0 += 32 * 4) {
                uint4 wv[4], hv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int cc = c0 + 32 * u;
                    wv[u] = cc < nc ? wp[cc] : make_uint4(0, 0, 0, 0);
                    hv[u] = cc < nc ? hp[cc] : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    float fw[8], fh[8];
                    unpack_bf16x8(wv[u], fw);
                    unpack_bf16x8(hv[u], fh);
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc = fma((double)fw[j], (double)fh[j], acc);
                }
            }
        } else {
            for (int col = lane; col < a.d; col += 32)
                acc = fma(load_elem(a.W, a.w_dtype, row * a.d + col), load_elem(a.H, a.h_dtype, (size_t)r * a.d + col), acc);
        }
        acc = warp_sum_d(acc);
        if (lane == 0) c_e[c] = acc * (double)a.inv_temp;
    }
    __syncthreads();
    if (threadIdx.x == 0) FIN_TRACE(5);
    // 4. order each re-scored run exactly, write the top k
    if (threadIdx.x == 0) {
        for (int i = 0; i < nk; ++i)
            if (!c_need[i]) c_e[i] = (double)c_v32[i];
        int i = 0;
        while (i < nk) {
            if (!c_need[i]) { ++i; continue; }
            int j = i;
            while (j + 1 < nk && c_need[j + 1]) ++j;   // contiguous re-scored block

            for (int u = i + 1; u <= j; ++u) {   // insertion sort by (exact desc, id asc)
                double e = c_e[u];
                int32_t id = c_id[u];
                int w = u - 1;
                while (w >= i && before(e, id, c_e[w], c_id[w])) { c_e[w + 1] = c_e[w]; c_id[w + 1] = c_id[w]; --w; }
                c_e[w + 1] = e;
                c_id[w + 1] = id;
            }
            i = j + 1;
        }
        const float lse = row_sumexp[r] > 0.0f ? row_max[r] + logf(row_sumexp[r]) : -INFINITY;
        for (int t = 0; t < k; ++t) {
            const int oid = t < nk ? lmh_id_at(a, c_id[t]) : -1;
            topk_ids[(size_t)r * k + t] = oid;
            topk_vals[(size_t)r * k + t] = t < nk ? (float)c_e[t] : -INFINITY;
            if (a.m_ids) {   // fused single-shard merge (R = 1)
                a.m_ids[(size_t)r * k + t] = oid;
                a.m_vals[(size_t)r * k + t] = t < nk ? (float)c_e[t] : -INFINITY;
                if (a.m_probs) a.m_probs[(size_t)r * k + t] = t < nk ? expf((float)c_e[t] - lse) : 0.0f;
            }
        }
        if (a.m_ids) a.m_lse[r] = lse;
        FIN_TRACE(6);
        if (a.trace && blockIdx.x < 148) a.trace[148 * 8 + (size_t)blockIdx.x * 8 + 7] = nn;   // re-scored count
    }
}



bool launch_lmh_finalize(const LmhArgs& a, int n_cta, int k, const float* wmax_dev, int32_t* topk_ids,
                         float* topk_vals, float* row_max, float* row_sumexp, int* flags, cudaStream_t st,
                         float gamma) {
    if (a.KP <= 32 && (a.LS == 64 || a.LS == kTcListLS) && n_cta <= kF64MaxCta) {
        // one CTA per SM while the rows fit one wave (the dynamic allocation is only a
        // placement hint: CTAs sharing an SM measured slower in round 1)
        // (256 threads; 512 measured slower)
        auto kern = lmh_fin64_kernel<kF64Threads>;
        static thread_local bool attr_set = false;
        if (!attr_set)
            attr_set = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 120 * 1024) == cudaSuccess;
        launch_pdl(kern, dim3(a.n_h), dim3(kF64Threads), a.n_h <= kNumSMs ? (size_t)120 * 1024 : 0, st, a, n_cta, k,
                   gamma, wmax_dev, topk_ids, topk_vals, row_max, row_sumexp, flags);
        return true;
    }
    if (a.KP <= 32) return false;   // (lists of a shape only fin64 reads: more lists than kF64MaxCta)
    size_t smem = (size_t)n_cta * 2 * sizeof(int) + (size_t)n_cta * a.KP * 8;
    cudaFuncSetAttribute(lmh_finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    lmh_finalize_kernel<<<a.n_h, kFinThreads, smem, st>>>(a, n_cta, k, gamma, wmax_dev, topk_ids, topk_vals,
                                                           row_max, row_sumexp, flags);
    return true;
}

// ------------------------------------------------------------ segment schedule
// CTAs per segment for a segment-mode LM-head launch (the work is rows of W streamed)
__global__ void seg_schedule_kernel(const int32_t* __restrict__ seg_pos, const SegRows seg_h_p, int nseg, int grid,
                                    int32_t* __restrict__ seg_cta) {
    // CTAs per segment minimising the largest per-CTA share of rows: the smallest L with
    // sum_b ceil(size_b / L) <= grid over the active segments (binary search, one warp;
    // a segment's CTAs split its rows evenly), then an exclusive prefix sum
    const int* seg_h = seg_h_p.h;
    pdl_trigger();
    pdl_wait();
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    auto size_of = [&](int b) -> int {
        const int sz = seg_pos[b + 1] - seg_pos[b];
        return (sz > 0 && seg_h[b + 1] > seg_h[b]) ? sz : 0;
    };
    int mx = 0;
    for (int b = lane; b < nseg; b += 32) mx = max(mx, size_of(b));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int lo = 1, hi = max(1, mx);   // need(hi) <= number of active segments <= grid
    while (lo < hi) {
        const int L = (lo + hi) >> 1;
        int need = 0;
        for (int b = lane; b < nseg; b += 32) need += (size_of(b) + L - 1) / L;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) need += __shfl_xor_sync(0xffffffffu, need, o);
        if (need <= grid) hi = L; else lo = L + 1;
    }
    const int L = lo;
    if (lane == 0) {
        int acc = 0;
        for (int b = 0; b < nseg; ++b) {
            seg_cta[b] = acc;
            acc += (size_of(b) + L - 1) / L;
        }
        seg_cta[nseg] = min(acc, grid);
    }
}

void launch_seg_schedule(const int32_t* seg_pos, const int32_t* seg_h_host, int nseg, int grid, int32_t* seg_cta,
                         cudaStream_t st) {
    SegRows sr{};
    for (int b = 0; b <= nseg && b <= kMaxSeg; ++b) sr.h[b] = seg_h_host[b];
    launch_pdl(seg_schedule_kernel, dim3(1), dim3(32), 0, st, seg_pos, sr, nseg, grid, seg_cta);
}

// ------------------------------------------------------------ shard merge
__global__ void __launch_bounds__(256)
merge_kernel(int R, int n_h, int k, const int32_t* __restrict__ ids, const float* __restrict__ vals,
             const float* __restrict__ m, const float* __restrict__ s, int32_t* __restrict__ out_ids,
             float* __restrict__ out_vals, float* __restrict__ out_lse, float* __restrict__ out_probs,
             float* __restrict__ out_m, float* __restrict__ out_s) {
    pdl_trigger();
    pdl_wait();
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
    if (lane == 0 && out_m) { out_m[r] = sig > 0.0f ? M : -INFINITY; out_s[r] = sig; }
    const int nc = R * k;
    extern __shared__ unsigned char m_sm[];
    float* sv = (float*)m_sm + (size_t)warp_id() * nc * 2;
    int* si = (int*)(sv + nc);
    for (int c = lane; c < nc; c += 32) {          // independent loads, then smem only
        const int t = c / k, j = c - t * k;
        const size_t o = ((size_t)t * n_h + r) * k + j;
        si[c] = ids[o];
        sv[c] = vals[o];
    }
    __syncwarp();
    for (int i = 0; i < k; ++i) {
        float bv = -INFINITY;
        int bid = 0x7fffffff, bc = -1;
        for (int c = lane; c < nc; c += 32) {
            const int id = si[c];
            if (id < 0) continue;                     // padding or taken
            if (before(sv[c], id, bv, bid)) { bv = sv[c]; bid = id; bc = c; }
        }
        const int my = bid;
        float wv = bv;
        int wid = bid;
        warp_argbest(wv, wid);
        if (bc >= 0 && my == wid) si[bc] = -2;       // ids are unique across shards
        __syncwarp();
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
                  cudaStream_t st, float* out_m, float* out_s) {
    const int grid = (n_h + 7) / 8;
    const size_t smem = (size_t)8 * R * k * 8;
    cudaFuncSetAttribute(merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(merge_kernel, dim3(grid), dim3(256), smem, st, R, n_h, k, ids, vals, m, s, out_ids, out_vals, out_lse,
               out_probs, out_m, out_s);
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
            double w = load_elem(W, w_dtype, (size_t)row * d + c);
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
        if (v < 0 || v >= V || (i > 0 && ids[i - 1] >= v)) atomicOr(flags, kFlagBadIds);
    }
}

void launch_check_sorted(const int32_t* ids, const int* n_dev, int n_host, int V, int* flags, cudaStream_t st) {
    check_sorted_kernel<<<kNumSMs, 256, 0, st>>>(ids, n_dev, n_host, V, flags);
}

}  // namespace es
