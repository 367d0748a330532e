// fin64.cuh -- the finalisation of one H row from fixed-stride (LS = 64)
// candidate lists, k + 8 <= 32 (a6/a7 across the LM head's CTAs; the exact
// top-k of DESIGN §5.2 / SURVEY C10).
//
// Inputs per list c (one per LM-head CTA): (m_c, s_c) of the online softmax,
// cnt_c sorted entries (the GEMV producer) or xcnt_c unsorted ones (the
// tensor-core producers) in the first cnt_c + xcnt_c of LS value / key slots
// (LS = 64 GEMV, 128 tensor core; keys: subset positions, or vocabulary ids
// when a.gid_keys; slots past the entries are stale and never used). Every
// non-empty list holds its maximum m_c (the CTA's best entry for the row is
// always admitted), so the lists' heads are distinct elements of the row.
//
//   1. (m, s, counts) of every list; ||h||^2 (before the PDL wait: an input).
//   2. th0 = the KP-th largest of the 32 lane maxima of the heads (KP distinct
//      elements are >= it, so it bounds the row's KP-th best from below),
//      raised to any full sorted list's entry KP-1. Only lists whose head is
//      >= th0 can hold an entry >= th0 -- ~20 of the ~148 lists -- and only
//      those are loaded; their entries >= th0 go to a candidate buffer, and
//      (vocabulary-id keys) their W rows are prefetched to L2 for step 4.
//   3. the best KP candidates under (z desc, key asc): bitonic sorts of two
//      32-lane halves and one merge for <= 64 candidates, else exact ranks by
//      counting, else (massive ties) sorted batches of 32 merged by one warp
//      (out of line); runs of entries closer than 2 delta that reach the top k.
//   4. exact fp64 re-score of those runs, block-wide (every thread a slice of
//      the columns of up to four entries: one round trip of loads), and the
//      final order by (exact value, id).
// Every step is a latency chain of one or a few warps, so the code keeps the
// chains short: all loads of a step in flight at once, unrolled shuffle
// networks (a rolled 15-stage network measured 2.2x slower, tools/ubench/kth.cu),
// 4 block barriers in the common case. Measured on the llama draft step
// (tools/ubench/fin_iso.cu in isolation, tools/trace_lmh.py in place): ~8.5 us
// median per row in place vs ~10.4 for the round-1 finalisation.
#pragma once
#include "common.cuh"
#include "kernels.cuh"
#include "lmh_epilogue.cuh"   // warp_kth_largest, warp_sort32

namespace es {

ES_DEV long long fin_gtime() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// profiling stamps (EVOSPEC_TRACE): slots [148*8 + row*8 + i]; clock64 details of row 0
#define FIN_TRACE_R(slot) do { if (a.trace && r < 148) a.trace[148 * 8 + (size_t)r * 8 + (slot)] = fin_gtime(); } while (0)
#define FIN_DT_R(i) do { if (a.trace && r == 0) a.trace[2 * 148 * 8 + 16 + (i)] = clock64(); } while (0)

ES_DEV double fin_load_elem(const void* p, int dtype, size_t i) {
    return dtype == 0 ? (double)__uint_as_float((uint32_t)((const uint16_t*)p)[i] << 16) : (double)((const float*)p)[i];
}

constexpr int kF64MaxCta = 320;   // lists per row
constexpr int kF64Cand = 1024;    // candidate buffer (entries >= th0)
constexpr int kF64Threads = 256;

// Massive ties (more than kF64Cand entries >= th0): one warp merges sorted
// batches of 32 of the qualifying lists' entries >= th0 into the best KP
// (lane i holds entry i). Out of line: never on the common path.
struct TieOut { float v; int p, cnt; };
__device__ __noinline__ TieOut fin64_tie_merge(const float* __restrict__ pval, const int32_t* __restrict__ pid, int n_h,
                                               int r, int cA0, int nA, int c_base, const int* qidx, const int* l_n, int nq, int LS,
                                               float th0, int KP) {
    const int lane = lane_id();
    float v = -INFINITY;
    int p = 0x7fffffff, cnt = 0;
    float th = -INFINITY;
    int thp = 0x7fffffff;
    const int per = LS / 32;   // batches per list
#pragma unroll 1
    for (int b = 0; b < nq * per; ++b) {
        const int c = qidx[b / per], sl = (b % per) * 32 + lane;
        const int cta = c < nA ? cA0 + c : c_base + (c - nA);
        const size_t o = ((size_t)cta * n_h + r) * LS + sl;
        float bv = sl < l_n[c] ? __ldcg(&pval[o]) : -INFINITY;
        int bp = sl < l_n[c] ? __ldcg(&pid[o]) : 0x7fffffff;
        if (!(bv != -INFINITY && bv >= th0) || (cnt == KP && !before(bv, bp, th, thp))) { bv = -INFINITY; bp = 0x7fffffff; }
        const unsigned m = __ballot_sync(0xffffffffu, bv != -INFINITY);
        if (!m) continue;
        warp_sort32(bv, bp);
        const float rv = __shfl_sync(0xffffffffu, bv, 31 - lane);
        const int rp = __shfl_sync(0xffffffffu, bp, 31 - lane);
        if (before(rv, rp, v, p)) { v = rv; p = rp; }
#pragma unroll 1
        for (int j = 16; j > 0; j >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, v, j);
            const int op = __shfl_xor_sync(0xffffffffu, p, j);
            if (((lane & j) == 0) == before(ov, op, v, p)) { v = ov; p = op; }
        }
        cnt = min(cnt + __popc(m), KP);
        if (cnt == KP) { th = __shfl_sync(0xffffffffu, v, KP - 1); thp = __shfl_sync(0xffffffffu, p, KP - 1); }
    }
    return TieOut{v, p, cnt};
}

template <int NT>
__global__ void __launch_bounds__(NT)
lmh_fin64_kernel(LmhArgs a, int n_cta_arg, int k, float gamma, const float* __restrict__ wmax_dev,
                 int32_t* __restrict__ topk_ids, float* __restrict__ topk_vals, float* __restrict__ row_max,
                 float* __restrict__ row_sumexp, int* flags) {
    constexpr int NW = NT / 32;
    __shared__ float l_m[kF64MaxCta], l_s[kF64MaxCta];
    __shared__ int l_n[kF64MaxCta];
    __shared__ int qidx[kF64MaxCta];
    __shared__ float cand_v[kF64Cand];
    __shared__ int cand_p[kF64Cand];
    __shared__ float c_v[32];
    __shared__ int c_id[32], c_gid[32], need_list[32];
    __shared__ double c_e[32], res_d[NW * 8];
    __shared__ double red_d[NW];
    __shared__ float red_th[NW];
    __shared__ int red_tot[NW];
    __shared__ float red_s[NW];
    __shared__ int s_cand_n, s_nk, s_nneed, s_nq;
    __shared__ float s_th0, s_M, s_lse;
    __shared__ double s_delta;

    pdl_trigger();
    const int r = blockIdx.x;
    if (r >= a.n_h) return;   // (grid padding, EVOSPEC_FIN_PAD)
    const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    const int KP = a.KP, LS = a.LS;
    // ---- ||h||^2 (an input of the LM head only: before the PDL wait)
    const bool h_fast = a.h_dtype == 0 && a.d % 8 == 0;
    double hacc = 0.0;
    if (h_fast) {
        const uint4* hp = (const uint4*)((const uint16_t*)a.H + (size_t)r * a.d);
#pragma unroll 1
        for (int c = tid; c < a.d / 8; c += NT) {
            float f[8];
            unpack_bf16x8(__ldg(&hp[c]), f);
#pragma unroll
            for (int j = 0; j < 8; ++j) hacc = fma((double)f[j], (double)f[j], hacc);
        }
    } else {
#pragma unroll 1
        for (int col = tid; col < a.d; col += NT) {
            const double h = fin_load_elem(a.H, a.h_dtype, (size_t)r * a.d + col);
            hacc = fma(h, h, hacc);
        }
    }
    hacc = warp_sum_d(hacc);
    if (lane == 0) red_d[warp] = hacc;
    // delta = gamma ||h|| max_v ||W_v|| inv_temp: inputs only, so before the wait
    __syncthreads();
    if (tid == 0) {
        double hn = 0.0;
#pragma unroll
        for (int w = 0; w < NW; ++w) hn += red_d[w];
        s_delta = (double)gamma * sqrt(hn) * (double)__ldg(wmax_dev) * (double)a.inv_temp;
    }
    if (tid == 0) s_cand_n = 0;
    pdl_wait();
    // (every LM-head CTA has read the union's early-list flag: reset it for the next step)
    if (a.early_flag && blockIdx.x == 0 && tid == 0) *(volatile int*)a.early_flag = 0;
    if (tid == 0) { FIN_TRACE_R(0); FIN_DT_R(0); }
    // the row's lists: CTAs [c_base, c_base + n_cta) (segment mode: its segment's CTAs,
    // behind part_cta0), and for the ragged head also its static row group's nA lists
    int n_cta = n_cta_arg, c_base = a.part_cta0;
    if (a.nseg > 0) {
        int b = 0;
        while (b + 1 < a.nseg && a.seg_h[b + 1] <= r) ++b;
        if (a.seg_cta) {
            c_base = a.part_cta0 + a.seg_cta[b];
            n_cta = a.seg_cta[b + 1] - a.seg_cta[b];
        } else {
            c_base = a.part_cta0 + b * a.seg_ctas;
            n_cta = a.seg_ctas;
        }
    }
    const int nA = a.fin_a_rows > 0 ? a.fin_a_ctas : 0;
    const int cA0 = a.fin_a_rows > 0 ? a.fin_a_cta0 + (r / a.fin_a_rows) * a.fin_a_ctas : 0;
    n_cta += nA;
    // list ordinal c -> list index: the static group's lists first, then the launch's own
    auto cta_of = [&](int c) -> int { return c < nA ? cA0 + c : c_base + (c - nA); };
    // ---- 1. softmax states, counts, sorted lists' entry KP-1 (all loads in flight at once)
    float thl = -INFINITY;
    int tot = 0;
    {
        constexpr int R1 = (kF64MaxCta + NT - 1) / NT;
        float m_[R1], s_[R1], vk_[R1];
        int cn_[R1], xc_[R1];
#pragma unroll
        for (int i = 0; i < R1; ++i) {
            const int c = tid + i * NT;
            if (c < n_cta) {
                const size_t o = (size_t)cta_of(c) * a.n_h + r, so = part_st(a.part, cta_of(c), r);
                m_[i] = __ldcg(&a.part.m[so]);
                s_[i] = __ldcg(&a.part.s[so]);
                cn_[i] = __ldcg(&a.part.cnt[so]);
                xc_[i] = __ldcg(&a.part.xcnt[so]);
                vk_[i] = __ldcg(&a.part.val[o * LS + KP - 1]);
            }
        }
#pragma unroll
        for (int i = 0; i < R1; ++i) {
            const int c = tid + i * NT;
            if (c < n_cta) {
                if (cn_[i] >= KP) thl = fmaxf(thl, vk_[i]);
                tot += cn_[i] + xc_[i];
                l_m[c] = s_[i] > 0.0f ? m_[i] : -INFINITY;   // (an empty list has s = 0)
                l_s[c] = s_[i];
                l_n[c] = min(cn_[i] + xc_[i], LS);            // entries; slots past them are stale
            }
        }
    }
    thl = warp_max(thl);
    tot = warp_sum_i(tot);
    if (lane == 0) { red_th[warp] = thl; red_tot[warp] = tot; }
    __syncthreads();
    if (tid == 0) { FIN_TRACE_R(1); FIN_DT_R(1); }
    // ---- 2. (warp 0) th0, M, and the lists that can hold entries >= th0 (head >= th0)
    float thl_all = -INFINITY;
    int tot_all = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) { thl_all = fmaxf(thl_all, red_th[w]); tot_all += red_tot[w]; }
    if (warp == 0) {
        constexpr int JM = kF64MaxCta / 32;
        float hv[JM];
        float lm = -INFINITY;
#pragma unroll
        for (int j = 0; j < JM; ++j) {
            const int c = lane + 32 * j;
            hv[j] = c < n_cta ? l_m[c] : -INFINITY;
            lm = fmaxf(lm, hv[j]);
        }
        const float th0 = fmaxf(thl_all, warp_kth_largest(lm, KP));
        int nq = 0;
#pragma unroll
        for (int j = 0; j < JM; ++j) {
            if (32 * j < n_cta) {   // (uniform)
                const bool q = hv[j] != -INFINITY && hv[j] >= th0;
                const unsigned qm = __ballot_sync(0xffffffffu, q);
                if (q) qidx[nq + __popc(qm & ((1u << lane) - 1u))] = lane + 32 * j;
                nq += __popc(qm);
            }
        }
        if (lane == 0) { s_th0 = th0; s_nq = nq; }
        const float M = warp_max(lm);
        if (lane == 0) s_M = M;
    }
    __syncthreads();
    if (tid == 0) { FIN_TRACE_R(2); FIN_DT_R(2); }
    const float th0 = s_th0;
    const int nq = s_nq;
    const float M = s_M;
    if (tid == 0) FIN_DT_R(8);
    // the qualifying lists' entries >= th0 -> candidate buffer (16 float4 per list)
    const size_t row_bytes = (size_t)a.d * (a.w_dtype == 0 ? 2 : 4);
    const bool pf_rows = a.gid_keys && (a.fin_opt & 2) && row_bytes % 16 == 0 && row_bytes <= (1u << 20);
    {
        const int ush = LS == 128 ? 5 : 4;   // float4 units per list: 1 << ush
        const int units = nq << ush;
        // the softmax sum (reduced in step 3), by every thread once
        auto softmax_sum = [&]() {
            float S = 0.0f;
#pragma unroll 1
            for (int c = tid; c < n_cta; c += NT)
                if (l_m[c] != -INFINITY) S += l_s[c] * __expf(l_m[c] - M);
            S = warp_sum(S);
            if (lane == 0) red_s[warp] = S;
        };
        const int wbase = tid - lane;   // (warp-uniform loop: the softmax sum's shuffles)
        if (wbase >= units) softmax_sum();   // (warps without filter units: right away)
#pragma unroll 1
        for (int u0 = wbase; u0 < units; u0 += 4 * NT) {
            float4 vv[4];
            int4 ii[4];
            int nv[4];   // valid entries in the unit (slots past a list's entries hold stale data)
#pragma unroll
            for (int x = 0; x < 4; ++x) {   // all loads in flight before any use
                const int u = u0 + lane + x * NT;
                const int c = u < units ? qidx[u >> ush] : 0, sl = (u & ((1 << ush) - 1)) * 4;
                nv[x] = u < units ? l_n[c] - sl : 0;
                const size_t o = ((size_t)cta_of(c) * a.n_h + r) * LS + sl;
                if (nv[x] > 0) {
                    vv[x] = __ldcg((const float4*)&a.part.val[o]);
                    ii[x] = __ldcg((const int4*)&a.part.id[o]);
                }
            }
            if (tid == 0 && u0 == 0) FIN_DT_R(9);   // (u0 = warp base)
            if (u0 == wbase) softmax_sum();   // (while the first loads fly)
#pragma unroll
            for (int x = 0; x < 4; ++x) {
                if (nv[x] <= 0) vv[x] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
                if (nv[x] < 4) vv[x].w = -INFINITY;
                if (nv[x] < 3) vv[x].z = -INFINITY;
                if (nv[x] < 2) vv[x].y = -INFINITY;
                const float v4[4] = {vv[x].x, vv[x].y, vv[x].z, vv[x].w};
                const int p4[4] = {ii[x].x, ii[x].y, ii[x].z, ii[x].w};
#pragma unroll
                for (int e = 0; e < 4; ++e)
                    if (v4[e] != -INFINITY && v4[e] >= th0) {
                        const int o = atomicAdd(&s_cand_n, 1);
                        if (o < kF64Cand) { cand_v[o] = v4[e]; cand_p[o] = p4[e]; }
                    }
            }
        }
    }
    if (tid == 0) FIN_DT_R(10);
    __syncthreads();
    if (tid == 0) { FIN_TRACE_R(3); FIN_DT_R(3); }
    // ---- 3. the best KP candidates, sorted, then runs
    const int ncand = s_cand_n;
    // while warp 0 ranks: the candidates' W rows towards L2 for the re-score (measured: the
    // re-score's loads take 5.0k cycles with this, 5.2k with the kept KP prefetched after
    // the sort, 6.7k without a prefetch)
    if (pf_rows && warp > 0) {
        for (int i = tid - 32; i < min(ncand, 64); i += NT - 32)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                         :: "l"((const char*)a.W + (size_t)(cand_p[i] / a.R) * row_bytes), "r"((uint32_t)row_bytes)
                         : "memory");
    }
    if (ncand > 64 && ncand <= kF64Cand) {   // exact ranks by counting
#pragma unroll 1
        for (int i = tid; i < ncand; i += NT) {
            const float v = cand_v[i];
            const int p = cand_p[i];
            int rank = 0;
#pragma unroll 1
            for (int j = 0; j < ncand; ++j) rank += before(cand_v[j], cand_p[j], v, p);
            if (rank < KP) { c_v[rank] = v; c_id[rank] = p; }
        }
        __syncthreads();
    }
    if (warp == 0) {
        float v;
        int p, cnt;
        if (ncand <= 64) {   // bitonic sorts of two 32-lane halves, one bitonic merge
            v = lane < ncand ? cand_v[lane] : -INFINITY;
            p = lane < ncand ? cand_p[lane] : 0x7fffffff;
            warp_sort32(v, p);
            if (ncand > 32) {
                float v1 = lane + 32 < ncand ? cand_v[lane + 32] : -INFINITY;
                int p1 = lane + 32 < ncand ? cand_p[lane + 32] : 0x7fffffff;
                warp_sort32(v1, p1);
                const float rv = __shfl_sync(0xffffffffu, v1, 31 - lane);
                const int rp = __shfl_sync(0xffffffffu, p1, 31 - lane);
                if (before(rv, rp, v, p)) { v = rv; p = rp; }
#pragma unroll
                for (int j = 16; j > 0; j >>= 1) {
                    const float ov = __shfl_xor_sync(0xffffffffu, v, j);
                    const int op = __shfl_xor_sync(0xffffffffu, p, j);
                    if (((lane & j) == 0) == before(ov, op, v, p)) { v = ov; p = op; }
                }
            }
            cnt = min(ncand, KP);
        } else if (ncand <= kF64Cand) {
            cnt = KP;
            v = lane < cnt ? c_v[lane] : -INFINITY;
            p = lane < cnt ? c_id[lane] : 0x7fffffff;
        } else {
            const TieOut t = fin64_tie_merge(a.part.val, a.part.id, a.n_h, r, cA0, nA, c_base, qidx, l_n, nq, LS, th0, KP);
            v = t.v; p = t.p; cnt = t.cnt;
        }
        if (lane == 0) FIN_DT_R(11);
        if (lane >= cnt) { v = -INFINITY; p = 0x7fffffff; }
        const int gid = lane < cnt ? (a.gid_keys ? p : lmh_id_at(a, p)) : -1;
        if ((a.fin_opt & 2) && !a.gid_keys && lane < cnt) {   // (position keys) the re-score's rows towards L2 now
            const size_t rb = (size_t)a.d * (a.w_dtype == 0 ? 2 : 4);
            if (rb % 16 == 0 && rb <= (1u << 20)) {
                const char* wr = (const char*)a.W + (size_t)(gid / a.R) * rb;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(wr), "r"((uint32_t)rb) : "memory");
            }
        }
        c_v[lane] = v;
        c_id[lane] = p;
        c_gid[lane] = gid;
        const double delta = s_delta;   // (computed before the PDL wait)
        const float nv = __shfl_down_sync(0xffffffffu, v, 1);
        const bool close = lane + 1 < cnt && (double)v - (double)nv <= 2.0 * delta + 2.4e-7 * fabs((double)v);
        const unsigned cm = __ballot_sync(0xffffffffu, close);   // bit i: entries i and i+1 in one run
        const unsigned below = ~cm & ((1u << lane) - 1u);
        const int st_i = below ? 32 - __clz(below) : 0;          // run start
        const bool multi = (lane > 0 && ((cm >> (lane - 1)) & 1u)) || ((cm >> lane) & 1u);
        // members of runs reaching the top k (exact_vals: every top-k entry)
        const bool need = lane < cnt && ((multi && st_i < k) || (a.exact_vals && lane < k));
        const unsigned nm = __ballot_sync(0xffffffffu, need);
        if (need) need_list[__popc(nm & ((1u << lane) - 1u))] = lane;
        // uncertified: the run holding index k-1 reaches the last kept entry while entries were dropped
        const unsigned open_from_k = ~cm & ~((1u << (k - 1)) - 1u);
        const int end_k = open_from_k ? __ffs(open_from_k) - 1 : 31;
        const bool unc = (k - 1 < cnt && min(end_k, cnt - 1) == cnt - 1 && tot_all > cnt && cnt >= k) ||
                         !(delta >= 0.0) || isinf(delta);
        if (lane == 0) {
            if (unc) atomicOr(flags, kFlagUncertified);
            s_nneed = __popc(nm);
            s_nk = cnt;
            float S = 0.0f;
#pragma unroll
            for (int w = 0; w < NW; ++w) S += red_s[w];
            row_max[r] = M;
            row_sumexp[r] = S;
            s_lse = S > 0.0f ? M + logf(S) : -INFINITY;
        }
    }
    __syncthreads();
    if (tid == 0) { FIN_TRACE_R(4); FIN_DT_R(4); }
    // ---- 4. exact re-score of the flagged entries: bf16 rows block-wide (every thread a
    //         slice of the columns of up to 8 entries at once: one round trip of loads),
    //         other dtypes one warp per entry
    const int nn = s_nneed;
    if (nn > 0) {
        if (a.w_dtype == 0 && h_fast) {
            const int nc = a.d / 8;
            const uint4* hp = (const uint4*)((const uint16_t*)a.H + (size_t)r * a.d);
#pragma unroll 1
            for (int q0 = 0; q0 < nn; q0 += 8) {
                const uint4* wp[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int gidu = c_gid[need_list[min(q0 + u, nn - 1)]];
                    wp[u] = (const uint4*)((const uint16_t*)a.W + (size_t)(a.R == 1 ? gidu : gidu / a.R) * a.d);
                }
                double acc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[u] = 0.0;
#pragma unroll 1
                for (int c0 = tid; c0 < nc; c0 += 2 * NT) {   // two column chunks, all 18 loads in flight
                    uint4 wv[2][8], hv2[2];
#pragma unroll
                    for (int x = 0; x < 2; ++x) {
                        const int c = c0 + x * NT;
                        hv2[x] = c < nc ? __ldg(&hp[c]) : make_uint4(0, 0, 0, 0);
#pragma unroll
                        for (int u = 0; u < 8; ++u)
                            wv[x][u] = (c < nc && q0 + u < nn) ? __ldg(&wp[u][c]) : make_uint4(0, 0, 0, 0);
                    }
#pragma unroll
                    for (int x = 0; x < 2; ++x) {
                        float fh[8];
                        unpack_bf16x8(hv2[x], fh);
                        // H in fp64 pre-scaled by 2^896 (exact), W entering the fma as the raw
                        // double whose fields are the bf16 fields in place (value w * 2^-896,
                        // exact: two integer ops, no conversion unit -- the fp32 -> fp64
                        // conversions of W were the re-score's bottleneck); every product
                        // and hence every fma is bit-identical to the unscaled one
                        double dh[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) dh[j] = (double)fh[j] * 0x1p896;
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            if (q0 + u >= nn) break;   // (uniform: the group's last entries)
                            const uint32_t w4[4] = {wv[x][u].x, wv[x][u].y, wv[x][u].z, wv[x][u].w};
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                const uint32_t lo = (uint32_t)((int32_t)(w4[j] << 16) >> 3) & 0x8FFFE000u;
                                const uint32_t hi = (uint32_t)((int32_t)w4[j] >> 3) & 0x8FFFE000u;
                                acc[u] = fma(__hiloint2double((int)lo, 0), dh[2 * j], acc[u]);
                                acc[u] = fma(__hiloint2double((int)hi, 0), dh[2 * j + 1], acc[u]);
                            }
                        }
                    }
                }
                if (tid == 0 && q0 == 0) FIN_DT_R(13);
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (q0 + u >= nn) break;
                    const double t = warp_sum_d(acc[u]);
                    if (lane == 0) res_d[warp * 8 + u] = t;
                }
                __syncthreads();
                if (tid == 0 && q0 == 0) FIN_DT_R(14);
                if (tid < 8 && q0 + tid < nn) {
                    double t = 0.0;
#pragma unroll
                    for (int w = 0; w < NW; ++w) t += res_d[w * 8 + tid];
                    c_e[need_list[q0 + tid]] = t * (double)a.inv_temp;
                }
                __syncthreads();
            }
        } else {
#pragma unroll 1
            for (int q = warp; q < nn; q += NW) {
                const int c = need_list[q];
                const size_t row = (size_t)(c_gid[c] / a.R);
                double acc = 0.0;
#pragma unroll 1
                for (int col = lane; col < a.d; col += 32)
                    acc = fma(fin_load_elem(a.W, a.w_dtype, row * a.d + col),
                              fin_load_elem(a.H, a.h_dtype, (size_t)r * a.d + col), acc);
                acc = warp_sum_d(acc);
                if (lane == 0) c_e[c] = acc * (double)a.inv_temp;
            }
            __syncthreads();
        }
    }
    if (tid == 0) { FIN_TRACE_R(5); FIN_DT_R(5); }
    // ---- 5. order by (exact value if re-scored, else the fp32 value) desc, id asc; runs are
    //         more than 2 delta apart, so this is the exact order
    if (warp == 0) {
        const int cnt = s_nk;
        bool flagged = false;
#pragma unroll 1
        for (int q = 0; q < nn; ++q) flagged |= need_list[q] == lane;
        double e = lane < cnt ? (flagged ? c_e[lane] : (double)c_v[lane]) : -INFINITY;
        int gid = c_gid[lane];
        int id = lane < cnt ? gid : 0x7fffffff;
        // (the exact values usually keep the fp32 order: sort only if some pair is out of order)
        const double ne = __shfl_down_sync(0xffffffffu, e, 1);
        const int ni = __shfl_down_sync(0xffffffffu, id, 1);
        const bool in_order = lane + 1 >= cnt || !before(ne, ni, e, id);
        if (nn > 0 && !__all_sync(0xffffffffu, in_order)) {
#pragma unroll
            for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
                for (int j = kk >> 1; j > 0; j >>= 1) {
                    const double oe = __shfl_xor_sync(0xffffffffu, e, j);
                    const int oi = __shfl_xor_sync(0xffffffffu, id, j);
                    const bool keep_better = ((lane & j) == 0) == ((lane & kk) == 0);
                    if (keep_better == before(oe, oi, e, id)) { e = oe; id = oi; }
                }
            }
            gid = id;
        }
        if (lane < k) {
            const int oid = lane < cnt ? gid : -1;
            const float ovl = lane < cnt ? (float)e : -INFINITY;
            topk_ids[(size_t)r * k + lane] = oid;
            topk_vals[(size_t)r * k + lane] = ovl;
            if (a.m_ids) {   // fused single-shard merge (R = 1)
                a.m_ids[(size_t)r * k + lane] = oid;
                a.m_vals[(size_t)r * k + lane] = ovl;
                if (a.m_probs) a.m_probs[(size_t)r * k + lane] = lane < cnt ? expf(ovl - s_lse) : 0.0f;
                if (lane == 0) a.m_lse[r] = s_lse;
            }
        }
        if (lane == 0) {
            FIN_TRACE_R(6);
            FIN_DT_R(6);
            if (a.trace && r < 148) a.trace[148 * 8 + (size_t)r * 8 + 7] = ncand + 10000LL * nn;   // (+ re-scored)
        }
    }
}

}  // namespace es
