// finalize32.cuh -- the k + 8 <= 32 LM-head finalisation of one H row (the
// finalisation kernel, finalize.cu).
#pragma once
#include "common.cuh"
#include "kernels.cuh"
#include "lmh_epilogue.cuh"

namespace es {

constexpr int kFinCand32 = 1024;   // candidate buffer of the threshold filter
constexpr int kFin32MaxD = 8192;   // H row staged in shared memory (d <= this for the fast re-score)

ES_DEV long long fin32_gtime() {
    long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
// profiling stamps (EVOSPEC_TRACE): slots [148*8 + row*8 + i]; clock64 details of row 0
#define FIN_TRACE_R(slot) do { if (a.trace && r < 148) a.trace[148 * 8 + (size_t)r * 8 + (slot)] = fin32_gtime(); } while (0)
#define FIN_DT_R(i) do { if (a.trace && r == 0) a.trace[2 * 148 * 8 + 16 + (i)] = clock64(); } while (0)

ES_DEV double fin32_load_elem(const void* p, int dtype, size_t i) {
    return dtype == 0 ? (double)__uint_as_float((uint32_t)((const uint16_t*)p)[i] << 16) : (double)((const float*)p)[i];
}

struct Fin32Smem {
    float *w_M, *w_S, *w_th;
    int* w_tot;
    double* red_d;
    float* cand_v;
    int* cand_p;
    float* c_v;
    int32_t *c_id, *c_gid;
    double* c_e;
    int* need_list;
    int* scal;      // n_need, nk, tot, cand_n
    float* fscal;   // lse, th
    float* s_head;
    uint32_t* head_cnt;   // [nt] packed (gt, ge) head ranks
    double* res_d;        // [32] re-score partials (one per warp slice)
    uint16_t* h_row;
};

__host__ __device__ inline size_t fin32_smem_bytes(int nt) {
    const int nw = nt / 32;
    return (size_t)kFin32MaxD * 2 + (size_t)nw * 8 + (size_t)32 * 8 + (size_t)kFinCand32 * 8 + (size_t)nw * 16 +
           32 * 16 + 8 * 4 + 4 * 4 + (size_t)nt * 8 + 32 * 8 + 256;
}

ES_DEV Fin32Smem fin32_carve(unsigned char* p, int nt) {
    const int nw = nt / 32;
    Fin32Smem m;
    // align by pointer arithmetic (an integer round trip would turn every shared
    // access below into a generic LD/ST)
    p += (16u - ((uint32_t)__cvta_generic_to_shared(p) & 15u)) & 15u;
    m.h_row = (uint16_t*)p;     p += (size_t)kFin32MaxD * 2;
    m.red_d = (double*)p;       p += (size_t)nw * 8;
    m.c_e = (double*)p;         p += 32 * 8;
    m.res_d = (double*)p;       p += 32 * 8;
    m.cand_v = (float*)p;       p += (size_t)kFinCand32 * 4;
    m.cand_p = (int*)p;         p += (size_t)kFinCand32 * 4;
    m.w_M = (float*)p;          p += (size_t)nw * 4;
    m.w_S = (float*)p;          p += (size_t)nw * 4;
    m.w_th = (float*)p;         p += (size_t)nw * 4;
    m.w_tot = (int*)p;          p += (size_t)nw * 4;
    m.c_v = (float*)p;          p += 32 * 4;
    m.c_id = (int32_t*)p;       p += 32 * 4;
    m.c_gid = (int32_t*)p;      p += 32 * 4;
    m.need_list = (int*)p;      p += 32 * 4;
    m.scal = (int*)p;           p += 8 * 4;
    m.fscal = (float*)p;        p += 4 * 4;
    m.s_head = (float*)p;       p += (size_t)nt * 4;
    m.head_cnt = (uint32_t*)p;
    return m;
}

// Finalisation for KP <= 32 (k <= 24). The partial lists have a fixed stride of
// kFin32LS = 64 slots and unused slots hold -inf (epi_store), so a row's
// entries form one flat array of n_cta * 64 values, loaded in one round trip
// into registers (U float4 + int4 per thread):
//   A. loads; per list (thread c): softmax state and th_c = its sorted entry
//      KP-1 when the sorted part is full (th_c <= the row's KP-th best)
//   B. th0 = max_c th_c; the entries >= th0 (every top-KP entry among them)
//      are appended to a candidate buffer
//   C. exact ranks: candidate i's rank is the number of candidates before it
//      under (value desc, id asc) -- one thread per candidate, no sort network;
//      ranks < KP give the sorted list. Warp 0 then finds the runs (consecutive
//      entries closer than 2 delta) that reach the top k.
//   D. exact fp64 re-score of those run members (one warp each)
//   E. one warp sort by (exact-if-re-scored value desc, id asc); write the top k
// Degenerate rows (more than kFin32RankMax candidates: massive ties, or no
// full list) take a slower exact path: warp 0 merges sorted batches of 32.
constexpr int kFin32Threads = 512;
constexpr int kFin32LS = 64;
constexpr int kFin32RankMax = 256;

ES_DEV void sort32_rolled(float& v, int& p) {
    const int lane = lane_id();
#pragma unroll 1
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll 1
        for (int j = k >> 1; j > 0; j >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, v, j);
            const int op = __shfl_xor_sync(0xffffffffu, p, j);
            const bool keep_better = ((lane & j) == 0) == ((lane & k) == 0);
            if (keep_better == before(ov, op, v, p)) { v = ov; p = op; }
        }
    }
}

// One H row's finalisation by a block of NT threads; shared memory comes from
// the caller (fin32_carve).
// H row r into shared memory and this thread's share of ||h||^2. Reads only
// the LM head's inputs (H), never its outputs, so the standalone kernel runs it
// before griddepcontrol.wait, overlapping the LM head's tail.
template <int NT>
ES_DEV double fin32_stage_h(const LmhArgs& a, const int r, const Fin32Smem& sm) {
    double hacc = 0.0;
    const bool h_fast = a.h_dtype == 0 && a.d % 8 == 0 && a.d <= kFin32MaxD;
    if (h_fast) {
        const uint4* hp = (const uint4*)((const uint16_t*)a.H + (size_t)r * a.d);
        for (int c = threadIdx.x; c < a.d / 8; c += NT) {
            const uint4 hv = __ldg(&hp[c]);
            ((uint4*)sm.h_row)[c] = hv;
            float f[8];
            unpack_bf16x8(hv, f);
#pragma unroll
            for (int j = 0; j < 8; ++j) hacc = fma((double)f[j], (double)f[j], hacc);
        }
    } else {
#pragma unroll 1
        for (int col = threadIdx.x; col < a.d; col += NT) {
            const double h = fin32_load_elem(a.H, a.h_dtype, (size_t)r * a.d + col);
            hacc = fma(h, h, hacc);
        }
    }
    return hacc;
}

// LSX: list stride. 64 = the unsorted candidate buffers of lmh_tc_kernel (cnt = 0,
// xcnt = entries); 32 = the sorted exact per-CTA top-KP lists of lmh_hl_kernel
// (cnt = entries, xcnt = 1 when the CTA dropped entries beyond its list).
template <int U, int NT, int LSX = kFin32LS>
ES_DEV void fin32_row(const LmhArgs& a, const int r, int n_cta_arg, int k, float gamma,
                      const float* __restrict__ wmax_dev, int32_t* __restrict__ topk_ids,
                      float* __restrict__ topk_vals, float* __restrict__ row_max, float* __restrict__ row_sumexp,
                      int* flags, const Fin32Smem& sm, bool h_staged = false, double hacc_pre = 0.0) {
    const int KP = a.KP;
    const int lane = lane_id(), warp = warp_id();
    constexpr int nwarps = NT / 32;
    float* w_M = sm.w_M; float* w_S = sm.w_S; float* w_th = sm.w_th; int* w_tot = sm.w_tot;
    double* red_d = sm.red_d;
    float* cand_v = sm.cand_v; int* cand_p = sm.cand_p;
    float* c_v = sm.c_v; int32_t* c_id = sm.c_id; int32_t* c_gid = sm.c_gid; double* c_e = sm.c_e;
    int* need_list = sm.need_list;
    int& n_need_s = sm.scal[0]; int& nk_s = sm.scal[1]; int& cand_n = sm.scal[3];
    float& lse_s = sm.fscal[0]; float& th_s = sm.fscal[1];
    float* s_head = sm.s_head;
    uint16_t* h_row = sm.h_row;
    if (threadIdx.x == 0) { FIN_TRACE_R(0); FIN_DT_R(0); }
    // the row's lists: CTAs [c_base, c_base + n_cta) (segment mode: its segment's CTAs)
    int n_cta = n_cta_arg, c_base = 0;
    if (a.nseg > 0) {
        int b = 0;
        while (b + 1 < a.nseg && a.seg_h[b + 1] <= r) ++b;
        if (a.seg_cta) {
            c_base = a.seg_cta[b];
            n_cta = a.seg_cta[b + 1] - c_base;
        } else {
            c_base = b * a.seg_ctas;
            n_cta = a.seg_ctas;
        }
    }
    // A. every global load at once
    constexpr int QL = LSX / 4;   // float4 per list
    const int nq = n_cta * QL;
    float4 vv[U];
    int4 ii[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const int q = threadIdx.x + u * NT;
        vv[u] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        if (q < nq) {
            const size_t o = ((size_t)(c_base + q / QL) * a.n_h + r) * LSX + (q % QL) * 4;
            vv[u] = __ldcg((const float4*)&a.part.val[o]);
            ii[u] = __ldcg((const int4*)&a.part.id[o]);
        }
    }
    float cm_ = -INFINITY, cs_ = 0.0f, thl = -INFINITY;
    int dropped = 0;   // sorted lists: entries a CTA dropped (counted into tot, the uncertified test)
    if ((int)threadIdx.x < n_cta) {
        const size_t o = (size_t)(c_base + threadIdx.x) * a.n_h + r;
        cm_ = __ldcg(&a.part.m[o]);
        cs_ = __ldcg(&a.part.s[o]);
        const int cn = __ldcg(&a.part.cnt[o]);
        const float vk = __ldcg(&a.part.val[o * LSX + KP - 1]);
        if (cn >= KP) thl = vk;
        if (LSX == 32) dropped = __ldcg(&a.part.xcnt[o]);
        // the list maximum: every producer keeps the CTA row's best entry, whose value
        // is the row's running maximum m (sorted lists: also slot 0)
        s_head[threadIdx.x] = cm_;
        sm.head_cnt[threadIdx.x] = 0u;
    }
    const float wmax = __ldg(wmax_dev);
    const bool h_fast = a.h_dtype == 0 && a.d % 8 == 0 && a.d <= kFin32MaxD;
    double hacc = h_staged ? hacc_pre : fin32_stage_h<NT>(a, r, sm);
    if (threadIdx.x == 0) { cand_n = 0; th_s = -INFINITY; }
    {   // (the list entries vv / ii are still in flight: first consumed by the filter,
        //  so their latency overlaps this and the head threshold below)
        const float Mw = warp_max(cs_ > 0.0f ? cm_ : -INFINITY);
        const float Sw = warp_sum(cs_ > 0.0f ? cs_ * expf(cm_ - Mw) : 0.0f);
        thl = warp_max(thl);
        hacc = warp_sum_d(hacc);
        if (lane == 0) { w_M[warp] = Mw; w_S[warp] = Sw; w_th[warp] = thl; red_d[warp] = hacc; }
    }
    __syncthreads();
    if (threadIdx.x == 0) { FIN_TRACE_R(1); FIN_DT_R(1); }
    // B. threshold: the KP-th largest list head (KP distinct entries) and any full
    //    list's entry KP-1 both bound the row's KP-th best from below
    // (NT / n_cta threads per head, each counting a slice of the heads; a packed
    //  shared atomic per head: gt in the low 16 bits, ge in the high 16)
    if (n_cta >= KP) {
        const int per = (a.fin_opt & 8) ? max(1, NT / n_cta) : 1;
        const int c = threadIdx.x / per, part = threadIdx.x % per;
        if (c < n_cta) {
            const float hv = s_head[c];
            const int c0 = n_cta * part / per, c1 = n_cta * (part + 1) / per;
            int gt = 0, ge = 0;
#pragma unroll 4
            for (int j = c0; j < c1; ++j) {
                const float o = s_head[j];
                gt += o > hv;
                ge += o >= hv;
            }
            if (per == 1) {
                if (hv != -INFINITY && gt < KP && KP <= ge) th_s = hv;   // the KP-th largest head value
            } else {
                atomicAdd(&sm.head_cnt[c], (uint32_t)gt | ((uint32_t)ge << 16));
            }
        }
        if (per > 1) {
            __syncthreads();
            if ((int)threadIdx.x < n_cta) {
                const uint32_t pc = sm.head_cnt[threadIdx.x];
                const int gt = (int)(pc & 0xffffu), ge = (int)(pc >> 16);
                const float hv = s_head[threadIdx.x];
                if (hv != -INFINITY && gt < KP && KP <= ge) th_s = hv;
            }
        }
    }
    __syncthreads();
    float th0 = th_s;
#pragma unroll
    for (int w = 0; w < nwarps; ++w) th0 = fmaxf(th0, w_th[w]);
    if (warp == 0) {   // softmax combine and entry count (lanes = warps)
        const bool have = lane < nwarps && w_S[lane] > 0.0f;
        const float M = warp_max(have ? w_M[lane] : -INFINITY);
        const float S = warp_sum(have ? w_S[lane] * expf(w_M[lane] - M) : 0.0f);
        if (lane == 0) {
            row_max[r] = M;
            row_sumexp[r] = S;
            lse_s = S > 0.0f ? M + logf(S) : -INFINITY;
        }
    }
    {
        auto keep = [&](float x) { return x != -INFINITY && x >= th0; };
        int nk = 0, tcnt = dropped;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            nk += keep(vv[u].x) + keep(vv[u].y) + keep(vv[u].z) + keep(vv[u].w);
            tcnt += (vv[u].x != -INFINITY) + (vv[u].y != -INFINITY) + (vv[u].z != -INFINITY) + (vv[u].w != -INFINITY);
        }
        tcnt = warp_sum_i(tcnt);
        if (lane == 0) w_tot[warp] = tcnt;
        if (nk) {
            int o = atomicAdd(&cand_n, nk);
            auto put = [&](float x, int id) {
                if (keep(x)) {
                    if (o < kFinCand32) { cand_v[o] = x; cand_p[o] = id; }
                    ++o;
                }
            };
#pragma unroll
            for (int u = 0; u < U; ++u) { put(vv[u].x, ii[u].x); put(vv[u].y, ii[u].y); put(vv[u].z, ii[u].z); put(vv[u].w, ii[u].w); }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) { FIN_TRACE_R(2); FIN_DT_R(2); }
    const int ncand = cand_n;
    if (ncand <= kFin32RankMax) {
        // C1. exact ranks, one thread per candidate
        if ((int)threadIdx.x < ncand) {
            const float v = cand_v[threadIdx.x];
            const int p = cand_p[threadIdx.x];
            const int gid = lmh_id_at(a, p);   // position -> vocabulary id (in flight during the ranks)
            int rank = 0;
#pragma unroll 4
            for (int j = 0; j < ncand; ++j) rank += before(cand_v[j], cand_p[j], v, p);
            if (rank < KP) {
                c_v[rank] = v;
                c_id[rank] = p;
                c_gid[rank] = gid;
                // the re-score reads a few of these rows: start them towards L2 now
                const size_t rb = (size_t)a.d * (a.w_dtype == 0 ? 2 : 4);
                if ((a.fin_opt & 2) && rb % 16 == 0 && rb <= (1u << 20)) {
                    const char* wr = (const char*)a.W + (size_t)(gid / a.R) * rb;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(wr), "r"((uint32_t)rb) : "memory");
                }
            }
        }
        if (threadIdx.x == 0) nk_s = min(ncand, KP);
    } else if (warp == 0) {
        // C1'. degenerate rows: sorted batches of 32 merged into the register list,
        //      from the candidate buffer or (overflow) the whole row in the partials
        float Lv = -INFINITY, th = -INFINITY;
        int Lp = 0x7fffffff, thp = 0x7fffffff, cnt = 0;
        const bool all = ncand > kFinCand32;
        const int nb = all ? ((nq + 31) / 32) * 4 : (ncand + 31) / 32;
#pragma unroll 1
        for (int b = 0; b < nb; ++b) {
            float bv = -INFINITY;
            int bp = 0x7fffffff;
            if (!all) {
                const int i = b * 32 + lane;
                if (i < ncand) { bv = cand_v[i]; bp = cand_p[i]; }
            } else {
                const int q = (b >> 2) * 32 + lane, comp = b & 3;
                if (q < nq) {
                    const size_t o = ((size_t)(c_base + q / QL) * a.n_h + r) * LSX + (q % QL) * 4 + comp;
                    bv = __ldcg(&a.part.val[o]);
                    bp = __ldcg(&a.part.id[o]);
                }
            }
            if (cnt == KP && !before(bv, bp, th, thp)) { bv = -INFINITY; bp = 0x7fffffff; }
            const unsigned m = __ballot_sync(0xffffffffu, bv != -INFINITY);
            if (!m) continue;
            sort32_rolled(bv, bp);
            const float rv = __shfl_sync(0xffffffffu, bv, 31 - lane);
            const int rp = __shfl_sync(0xffffffffu, bp, 31 - lane);
            if (before(rv, rp, Lv, Lp)) { Lv = rv; Lp = rp; }
#pragma unroll 1
            for (int j = 16; j > 0; j >>= 1) {
                const float ov = __shfl_xor_sync(0xffffffffu, Lv, j);
                const int op = __shfl_xor_sync(0xffffffffu, Lp, j);
                if (((lane & j) == 0) == before(ov, op, Lv, Lp)) { Lv = ov; Lp = op; }
            }
            cnt = min(cnt + __popc(m), KP);
            if (cnt == KP) { th = __shfl_sync(0xffffffffu, Lv, KP - 1); thp = __shfl_sync(0xffffffffu, Lp, KP - 1); }
        }
        c_v[lane] = Lv;
        c_id[lane] = Lp;
        if (lane == 0) nk_s = cnt;
    }
    __syncthreads();
    if (threadIdx.x == 0) { FIN_TRACE_R(3); FIN_DT_R(3); }
    if (warp == 0) {
        // C2. runs: consecutive kept entries closer than 2 delta; those reaching the top k are re-scored
        const int cnt = nk_s, tot = warp_sum_i(lane < nwarps ? w_tot[lane] : 0);
        const float Lv = lane < cnt ? c_v[lane] : -INFINITY;
        // position -> vocabulary id (the rank path stored it already)
        if (ncand > kFin32RankMax) c_gid[lane] = lane < cnt ? lmh_id_at(a, c_id[lane]) : -1;
        else if (lane >= cnt) c_gid[lane] = -1;
        double hn = 0.0;
#pragma unroll
        for (int w = 0; w < nwarps; ++w) hn += red_d[w];
        const double delta = (double)gamma * sqrt(hn) * (double)wmax * (double)a.inv_temp;
        const float nv = __shfl_down_sync(0xffffffffu, Lv, 1);
        const bool close = lane + 1 < cnt && (double)Lv - (double)nv <= 2.0 * delta + 2.4e-7 * fabs((double)Lv);
        const unsigned cm = __ballot_sync(0xffffffffu, close);   // bit i: entry i and i+1 in one run
        // run start: just above the highest open link below the lane
        const unsigned below = ~cm & ((1u << lane) - 1u);
        const int st_i = below ? 32 - __clz(below) : 0;
        const bool multi = (lane > 0 && ((cm >> (lane - 1)) & 1u)) || ((cm >> lane) & 1u);
        // members of runs reaching the top k; with exact_vals (the triple feeds a merge
        // across shards or across the static / dynamic parts of the ragged head) every
        // top-k entry, so that the merge compares the exact logits (rounded to fp32)
        const bool need = lane < cnt && ((multi && st_i < k) || (a.exact_vals && lane < k));
        const unsigned nm = __ballot_sync(0xffffffffu, need);
        if (need) need_list[__popc(nm & ((1u << lane) - 1u))] = lane;
        // uncertified: the run holding index k-1 reaches the last kept entry while entries were dropped
        const unsigned open_from_k = ~cm & ~((1u << (k - 1)) - 1u);   // open links at index >= k-1
        const int end_k = open_from_k ? __ffs(open_from_k) - 1 : 31;
        const bool unc = (k - 1 < cnt && min(end_k, cnt - 1) == cnt - 1 && tot > cnt && cnt >= k) ||
                         !(delta >= 0.0) || isinf(delta);
        if (lane == 0) {
            if (unc) atomicOr(flags, kFlagUncertified);
            n_need_s = __popc(nm);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) { FIN_TRACE_R(4); FIN_DT_R(4); }
    // D. exact re-score of the flagged entries: each is split over nwarps / nn
    //    warps (contiguous slices of the row, W loads in flight), partials summed
    //    per entry (order-free: exact products, the fp64 sum is within the envelope)
    const int nn = n_need_s;
    const int wpc = (a.fin_opt & 4) && nn > 0 && nn <= nwarps ? nwarps / nn : 1;
    for (int q = warp; q < nn * wpc; q += nwarps) {
        const int ci = q / wpc, part = q - ci * wpc;
        const int c = need_list[ci];
        const size_t row = (size_t)(c_gid[c] / a.R);
        double acc = 0.0;
        if (a.w_dtype == 0 && h_fast) {
            const uint4* wp = (const uint4*)((const uint16_t*)a.W + row * a.d);
            const int nc = a.d / 8;
            const int s0 = (int)((long long)nc * part / wpc), s1 = (int)((long long)nc * (part + 1) / wpc);
            double a4[4] = {0.0, 0.0, 0.0, 0.0};
            for (int c0 = s0; c0 < s1; c0 += 32 * 4) {
                uint4 wv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int cc = c0 + lane + 32 * u;
                    wv[u] = cc < s1 ? __ldg(&wp[cc]) : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int cc = c0 + lane + 32 * u;
                    if (cc < s1) {
                        float fw[8], fh[8];
                        unpack_bf16x8(wv[u], fw);
                        unpack_bf16x8(((const uint4*)h_row)[cc], fh);
#pragma unroll
                        for (int j = 0; j < 8; ++j) a4[j & 3] = fma((double)fw[j], (double)fh[j], a4[j & 3]);
                    }
                }
            }
            acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
        } else {
            const int s0 = (int)((long long)a.d * part / wpc), s1 = (int)((long long)a.d * (part + 1) / wpc);
#pragma unroll 1
            for (int col = s0 + lane; col < s1; col += 32)
                acc = fma(fin32_load_elem(a.W, a.w_dtype, row * a.d + col), fin32_load_elem(a.H, a.h_dtype, (size_t)r * a.d + col), acc);
        }
        acc = warp_sum_d(acc);
        if (lane == 0) {
            if (wpc == 1) c_e[c] = acc * (double)a.inv_temp;
            else sm.res_d[q] = acc;
        }
    }
    if (wpc > 1) {
        __syncthreads();
        if ((int)threadIdx.x < nn) {
            double t = 0.0;
            for (int p = 0; p < wpc; ++p) t += sm.res_d[threadIdx.x * wpc + p];
            c_e[need_list[threadIdx.x]] = t * (double)a.inv_temp;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) { FIN_TRACE_R(5); FIN_DT_R(5); }
    // E. one sort by (exact value if re-scored else fp32 value desc, id asc): runs are
    //    more than 2 delta apart, so this is the exact order; write the top k
    if (warp == 0) {
        const int cnt = nk_s;
        bool flagged = false;
        for (int q = 0; q < nn; ++q) flagged |= need_list[q] == lane;
        double e = lane < cnt ? (flagged ? c_e[lane] : (double)c_v[lane]) : -INFINITY;
        // ties on the vocabulary id (one sorted list: the same order as the positions;
        // two-list mode: the positions of the two lists interleave in id order)
        int id = lane < cnt ? c_gid[lane] : 0x7fffffff;
        int gid = c_gid[lane];
        if (nn > 0) {   // only re-scored runs can change the order
#pragma unroll 1
            for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll 1
                for (int j = kk >> 1; j > 0; j >>= 1) {
                    const double oe = __shfl_xor_sync(0xffffffffu, e, j);
                    const int oi = __shfl_xor_sync(0xffffffffu, id, j);
                    const int og = __shfl_xor_sync(0xffffffffu, gid, j);
                    const bool keep_better = ((lane & j) == 0) == ((lane & kk) == 0);
                    if (keep_better == before(oe, oi, e, id)) { e = oe; id = oi; gid = og; }
                }
            }
        }
        if (lane < k) {
            const int oid = lane < cnt ? gid : -1;
            const float ovl = lane < cnt ? (float)e : -INFINITY;
            topk_ids[(size_t)r * k + lane] = oid;
            topk_vals[(size_t)r * k + lane] = ovl;
            if (a.m_ids) {   // fused single-shard merge (R = 1)
                a.m_ids[(size_t)r * k + lane] = oid;
                a.m_vals[(size_t)r * k + lane] = ovl;
                if (a.m_probs) a.m_probs[(size_t)r * k + lane] = lane < cnt ? expf(ovl - lse_s) : 0.0f;
                if (lane == 0) a.m_lse[r] = lse_s;
            }
        }
        if (lane == 0) {
            FIN_TRACE_R(6);
            FIN_DT_R(6);
            if (a.trace && r < 148) a.trace[148 * 8 + (size_t)r * 8 + 7] = ncand;
        }
    }
}

}  // namespace es
