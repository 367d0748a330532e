// lmh_epilogue.cuh -- fused online softmax + top-k epilogue shared by the
// LM-head kernels (a6/a7: Eq. 1 P:47 restricted to V_t; top-k feeding the
// draft tree).
//
// A CTA owns a contiguous, ascending run of subset positions and visits it in
// tiles of kTile positions. For each tile the producer kernel leaves
//   tile[r][p] = z = inv_temp * logit   (r < n_h, p < kTile)
// in shared memory; the epilogue folds the tile into per-H-row state
//   m_r, s_r  (online softmax: s = s*exp(m_old - m_new) + sum exp(z - m_new))
//   the best KP = k + kTopkPad (z, position) pairs, ordered (z desc, pos asc).
// Positions ascend with token id (the subset is sorted), so "lower id wins
// ties" is "earlier position wins"; state from earlier tiles always wins a tie
// against the current tile.
//
// Top-KP fold (one warp per H row): the sorted list lives in registers, entry
// i on lane i % 32, slot i / 32. Tile values above the list's KP-th entry are
// inserted one at a time (ballot -> rank, shfl_up -> shift), so the cost is
// proportional to the number of values that actually enter. For a row whose
// list is not yet full, a pre-threshold theta0 = the KP-th largest of the 32
// per-lane maxima (a lower bound of the tile's KP-th value: those KP maxima
// are KP distinct tile elements) filters the tile first.
#pragma once
#include "common.cuh"
#include "kernels.cuh"

namespace es {

constexpr int kTile = 128;
constexpr int kTileJ = kTile / 32;

constexpr int kBuf = 64;   // unsorted candidate buffer per row (buffered path, KP <= 32)

struct EpiSmem {
    float* tile;     // [n_h][kTile]
    float* st_val;   // [n_h][cap]  cap = KP (sorted list) or kBuf (buffered path)
    int* st_pos;     // [n_h][cap]
    float* st_thv;   // [n_h] buffered path: admission bound (value, position)
    int* st_thp;     // [n_h]
    int* st_cnt;     // [n_h]
    float* st_m;     // [n_h]   running max
    float* st_ls;    // [n_h][32] per-lane partial sum of exp(z - m)
    int* st_xcnt;    // [n_h] extras appended by the last tile (global partials)
    float* scr_v;    // [n_warps][32] candidate batch scratch
    int* scr_p;      // [n_warps][32]
    int* st_flag;    // [4] block flags (thread-parallel fold: a row overflowed)
    int* tile_id;    // [kTile] buffered path: the key of each tile position (its vocabulary
                     // id), or null: keys are the subset positions themselves
};

// Key of tile position p (the order of ties: value desc, key asc)
ES_DEV int tile_key(const EpiSmem& e, int base_pos, int p) { return e.tile_id ? e.tile_id[p] : base_pos + p; }

__host__ __device__ inline size_t epi_smem_bytes(int n_h, int cap, int n_warps) {
    return (size_t)n_h * kTile * 4 + (size_t)n_h * cap * 8 + (size_t)n_h * 20 + (size_t)n_h * 32 * 4 +
           (size_t)n_warps * 32 * 8 + 16 + kTile * 4;
}

ES_DEV EpiSmem epi_carve(unsigned char* p, int n_h, int cap, int n_warps, bool keys = false) {
    EpiSmem e;
    e.tile = (float*)p;        p += (size_t)n_h * kTile * 4;
    e.st_val = (float*)p;      p += (size_t)n_h * cap * 4;
    e.st_pos = (int*)p;        p += (size_t)n_h * cap * 4;
    e.st_thv = (float*)p;      p += (size_t)n_h * 4;
    e.st_thp = (int*)p;        p += (size_t)n_h * 4;
    e.st_cnt = (int*)p;        p += (size_t)n_h * 4;
    e.st_m = (float*)p;        p += (size_t)n_h * 4;
    e.st_ls = (float*)p;       p += (size_t)n_h * 32 * 4;
    e.st_xcnt = (int*)p;       p += (size_t)n_h * 4;
    e.scr_v = (float*)p;       p += (size_t)n_warps * 32 * 4;
    e.scr_p = (int*)p;         p += (size_t)n_warps * 32 * 4;
    e.st_flag = (int*)p;       p += 16;
    e.tile_id = keys ? (int*)p : nullptr;
    return e;
}

ES_DEV void epi_init(const EpiSmem& e, int n_h) {
    for (int r = threadIdx.x; r < n_h; r += blockDim.x) {
        e.st_cnt[r] = 0;
        e.st_xcnt[r] = 0;
        if (r == 0) e.st_flag[0] = 0;
        e.st_m[r] = -INFINITY;
        e.st_thv[r] = -INFINITY;
        e.st_thp[r] = 0x7fffffff;
    }
    for (int i = threadIdx.x; i < n_h * 32; i += blockDim.x) e.st_ls[i] = 0.0f;
}

// KP-th largest value (1-based) of the 32 lane values, every lane gets it.
ES_DEV float warp_kth_largest(float x, int kth) {
    // bitonic sort descending across the warp (15 compare-exchange stages)
    const int lane = lane_id();
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const float y = __shfl_xor_sync(0xffffffffu, x, j);
            const bool lower = (lane & j) == 0;
            const bool desc = (lane & k) == 0;
            // in a descending block the lower lane keeps the larger value
            const bool keep_max = (lower == desc);
            x = keep_max ? fmaxf(x, y) : fminf(x, y);
        }
    }
    return __shfl_sync(0xffffffffu, x, kth - 1);
}

template <int SLOTS>
struct TopList {
    float v[SLOTS];
    int p[SLOTS];
};

// Online softmax for one row: lazy max (a warp reduction only when some value
// exceeds the running max), per-lane partial sums of exp(z - m) kept in smem
// and reduced across the warp only once, in epi_store.
ES_DEV void fold_softmax(const EpiSmem& e, int r, const float (&v)[kTileJ], float lane_max) {
    const int lane = lane_id();
    const float m_old = e.st_m[r];
    float m_new = m_old, scale = 1.0f;
    if (__any_sync(0xffffffffu, lane_max > m_old)) {
        m_new = fmaxf(m_old, warp_max(lane_max));
        scale = m_old == -INFINITY ? 0.0f : __expf(m_old - m_new);
    }
    float acc = e.st_ls[r * 32 + lane] * scale;
#pragma unroll
    for (int j = 0; j < kTileJ; ++j)
        if (v[j] != -INFINITY) acc += __expf(v[j] - m_new);   // ex2.approx: ~1e-6 rel., far inside C15
    e.st_ls[r * 32 + lane] = acc;
    __syncwarp();
    if (lane == 0) e.st_m[r] = m_new;
}

// Descending bitonic sort of 32 (value, position) pairs, one per lane, under
// (value desc, position asc).
ES_DEV void warp_sort32(float& v, int& p) {
    const int lane = lane_id();
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, v, j);
            const int op = __shfl_xor_sync(0xffffffffu, p, j);
            const bool keep_better = ((lane & j) == 0) == ((lane & k) == 0);
            const bool o_better = before(ov, op, v, p);
            if (keep_better == o_better) { v = ov; p = op; }
        }
    }
}

// Top-KP fold for KP <= 32: candidates above the threshold are compacted
// into batches of 32, each batch bitonic-sorted and merged into the sorted
// register list with one bitonic merge -- no per-candidate shuffle chains.
ES_DEV void fold_topk32(const EpiSmem& e, int r, int KP, int tn, int base_pos, int warp,
                        const float (&v)[kTileJ], float lane_max) {
    const int lane = lane_id();
    int cnt = e.st_cnt[r];
    float Lv = lane < cnt ? e.st_val[r * KP + lane] : -INFINITY;
    int Lp = lane < cnt ? e.st_pos[r * KP + lane] : 0x7fffffff;
    float tv = -INFINITY;
    int tp = 0x7fffffff;
    float theta0 = -INFINITY;
    if (cnt == KP) {
        tv = __shfl_sync(0xffffffffu, Lv, KP - 1);
        tp = __shfl_sync(0xffffffffu, Lp, KP - 1);
        if (!__any_sync(0xffffffffu, lane_max >= tv)) return;   // nothing can enter
    } else {
        theta0 = warp_kth_largest(lane_max, KP);
    }
    bool cand[kTileJ];
    unsigned msk[kTileJ];
    int total = 0;
#pragma unroll
    for (int j = 0; j < kTileJ; ++j) {
        const int pj = base_pos + lane + 32 * j;
        cand[j] = v[j] != -INFINITY && v[j] >= theta0 && (cnt < KP || before(v[j], pj, tv, tp));
        msk[j] = __ballot_sync(0xffffffffu, cand[j]);
        total += __popc(msk[j]);
    }
    if (total == 0) return;
    float* sv = e.scr_v + warp * 32;
    int* sp = e.scr_p + warp * 32;
    for (int done = 0; done < total; done += 32) {
        int base = 0;
#pragma unroll
        for (int j = 0; j < kTileJ; ++j) {
            const int idx = base + __popc(msk[j] & ((1u << lane) - 1u)) - done;
            if (cand[j] && idx >= 0 && idx < 32) { sv[idx] = v[j]; sp[idx] = base_pos + lane + 32 * j; }
            base += __popc(msk[j]);
        }
        __syncwarp();
        const int nb = min(32, total - done);
        float bv = lane < nb ? sv[lane] : -INFINITY;
        int bp = lane < nb ? sp[lane] : 0x7fffffff;
        __syncwarp();
        warp_sort32(bv, bp);
        // top 32 of (list desc) u (batch desc): elementwise best against the
        // reversed batch gives a bitonic sequence; one bitonic merge sorts it
        const float rv = __shfl_sync(0xffffffffu, bv, 31 - lane);
        const int rp = __shfl_sync(0xffffffffu, bp, 31 - lane);
        if (before(rv, rp, Lv, Lp)) { Lv = rv; Lp = rp; }
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, Lv, j);
            const int op = __shfl_xor_sync(0xffffffffu, Lp, j);
            const bool keep_better = (lane & j) == 0;
            if (keep_better == before(ov, op, Lv, Lp)) { Lv = ov; Lp = op; }
        }
        cnt = min(cnt + nb, KP);
    }
    if (lane < cnt) { e.st_val[r * KP + lane] = Lv; e.st_pos[r * KP + lane] = Lp; }
    if (lane == 0) e.st_cnt[r] = cnt;
    __syncwarp();
    (void)tn;
}

// Fold one row's tile values into its sorted top-KP list (SLOTS*32 >= KP).
template <int SLOTS>
ES_DEV void fold_row(const EpiSmem& e, int r, int KP, int tn, int base_pos) {
    const int lane = lane_id();
    float v[kTileJ];
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < kTileJ; ++j) {
        const int p = lane + 32 * j;
        v[j] = p < tn ? e.tile[r * kTile + p] : -INFINITY;
        mx = fmaxf(mx, v[j]);
    }
    const float lane_max = mx;
    mx = warp_max(mx);
    if (tn <= 0) return;
    // load the list
    int cnt = e.st_cnt[r];
    TopList<SLOTS> L;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
        const int i = lane + 32 * s;
        L.v[s] = i < cnt ? e.st_val[r * KP + i] : -INFINITY;
        L.p[s] = i < cnt ? e.st_pos[r * KP + i] : 0x7fffffff;
    }
    __syncwarp();
    const int kl = (KP - 1) & 31, ks = (KP - 1) >> 5;   // holder of entry KP-1
    auto kth = [&](float& tv, int& tp) {
        float cv = L.v[0];
        int cp = L.p[0];
#pragma unroll
        for (int s = 1; s < SLOTS; ++s) if (s == ks) { cv = L.v[s]; cp = L.p[s]; }
        tv = __shfl_sync(0xffffffffu, cv, kl);
        tp = __shfl_sync(0xffffffffu, cp, kl);
    };
    float tv;
    int tp;
    kth(tv, tp);                      // (-inf, INT_MAX) while the list is not full
    float theta0 = -INFINITY;         // pre-threshold for a list that is not full
    if (cnt < KP && KP <= 32) theta0 = warp_kth_largest(lane_max, KP);
    if (cnt == KP && !(mx > tv)) {    // nothing in this tile can enter
        if (lane == 0) e.st_cnt[r] = cnt;
        return;
    }
#pragma unroll
    for (int j = 0; j < kTileJ; ++j) {
        const int pj = base_pos + lane + 32 * j;
        bool cand = v[j] != -INFINITY && v[j] >= theta0 && (cnt < KP ? true : before(v[j], pj, tv, tp));
        unsigned m = __ballot_sync(0xffffffffu, cand);
        while (m) {
            const int src = __ffs(m) - 1;
            m &= m - 1;
            const float x = __shfl_sync(0xffffffffu, v[j], src);
            const int xp = base_pos + src + 32 * j;
            if (cnt == KP && !before(x, xp, tv, tp)) continue;   // threshold rose meanwhile
            // rank of x in the list
            int at = 0;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s)
                at += __popc(__ballot_sync(0xffffffffu, (lane + 32 * s) < cnt && before(L.v[s], L.p[s], x, xp)));
            // shift entries at index >= at by one, insert at `at`
#pragma unroll
            for (int s = SLOTS - 1; s >= 0; --s) {
                float pv = __shfl_up_sync(0xffffffffu, L.v[s], 1);
                int pp = __shfl_up_sync(0xffffffffu, L.p[s], 1);
                if (s > 0) {
                    const float cv = __shfl_sync(0xffffffffu, L.v[s > 0 ? s - 1 : 0], 31);
                    const int cp = __shfl_sync(0xffffffffu, L.p[s > 0 ? s - 1 : 0], 31);
                    if (lane == 0) { pv = cv; pp = cp; }
                }
                const int i = lane + 32 * s;
                if (i > at) { L.v[s] = pv; L.p[s] = pp; }
                if (i == at) { L.v[s] = x; L.p[s] = xp; }
            }
            cnt = min(cnt + 1, KP);
            if (cnt == KP) kth(tv, tp);
        }
    }
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
        const int i = lane + 32 * s;
        if (i < cnt) { e.st_val[r * KP + i] = L.v[s]; e.st_pos[r * KP + i] = L.p[s]; }
    }
    if (lane == 0) e.st_cnt[r] = cnt;
    __syncwarp();
}

// Fold the current tile (tn valid positions starting at global position
// base_pos) into the state of rows r = warp, warp + n_warps, ...
ES_DEV void epi_tile(const EpiSmem& e, int n_h, int KP, int tn, int base_pos, int warp, int n_warps) {
    if (tn <= 0) return;
    const int lane = lane_id();
    for (int r = warp; r < n_h; r += n_warps) {
        float v[kTileJ];
        float lm = -INFINITY;
#pragma unroll
        for (int j = 0; j < kTileJ; ++j) {
            const int p = lane + 32 * j;
            v[j] = p < tn ? e.tile[r * kTile + p] : -INFINITY;
            lm = fmaxf(lm, v[j]);
        }
        fold_softmax(e, r, v, lm);
        if (KP <= 32) fold_topk32(e, r, KP, tn, base_pos, warp, v, lm);
        else if (KP <= 64) fold_row<2>(e, r, KP, tn, base_pos);
        else fold_row<3>(e, r, KP, tn, base_pos);
    }
}

// Write the CTA's state to the global partials (positions -> global ids).
// Only [0, cnt) is written: extras may already sit at [cnt, cnt + xcnt).
// Partials carry subset positions, not ids: the subset is sorted ascending, so
// position order is id order, and only the finalisation's few winners are
// translated (no dependent global loads in the LM-head tail).
ES_DEV void epi_store(const EpiSmem& e, const LmhPartials& P, int cta, int n_h_total, int h_row0,
                      int n_h, int KP, int LS, int warp, int n_warps) {
    for (int r = warp; r < n_h; r += n_warps) {
        const int cnt = e.st_cnt[r];
        const size_t o = ((size_t)cta * n_h_total + h_row0 + r);
        for (int i = lane_id(); i < cnt; i += 32) {
            P.val[o * LS + i] = e.st_val[r * KP + i];
            P.id[o * LS + i] = e.st_pos[r * KP + i];
        }
        // fixed-stride lists (LS > KP): the slots after the sorted entries and the
        // extras hold -inf, so the finalisation reads the row as one flat array
        if (LS > KP)
            for (int i = cnt + e.st_xcnt[r] + lane_id(); i < LS; i += 32) P.val[o * LS + i] = -INFINITY;
        const float ssum = warp_sum(e.st_ls[r * 32 + lane_id()]);
        if (lane_id() == 0) {
            P.cnt[part_st(P, cta, h_row0 + r)] = cnt;
            P.xcnt[part_st(P, cta, h_row0 + r)] = e.st_xcnt[r];
            P.m[part_st(P, cta, h_row0 + r)] = e.st_m[r];
            P.s[part_st(P, cta, h_row0 + r)] = ssum;
        }
    }
}

// The CTA's last tile: online softmax as usual, but instead of folding the
// survivors into the sorted list they are appended to the global partials as
// unsorted extras (the finalisation scans them). Survivors must beat the
// list's entry KP-1 -- any element of the CTA's top-KP does. Rows whose list
// is not full, or with more survivors than LS - KP slots, take the full fold.
ES_DEV void epi_tile_last(const EpiSmem& e, const LmhPartials& P, int cta, int n_h_total, int h_row0, int n_h,
                          int KP, int LS, int tn, int base_pos, int warp, int n_warps) {
    if (tn <= 0) return;
    const int lane = lane_id();
    for (int r = warp; r < n_h; r += n_warps) {
        float v[kTileJ];
        float lm = -INFINITY;
#pragma unroll
        for (int j = 0; j < kTileJ; ++j) {
            const int p = lane + 32 * j;
            v[j] = p < tn ? e.tile[r * kTile + p] : -INFINITY;
            lm = fmaxf(lm, v[j]);
        }
        fold_softmax(e, r, v, lm);
        const int cnt = e.st_cnt[r];
        if (KP <= 32 && cnt == 0 && LS > KP) {
            // the CTA's only tile: no sorted list to extend, so the values at or
            // above theta0 = the KP-th largest lane maximum (a superset of the
            // tile's top KP) go out unsorted when they fit the list
            // (a tile of at most LS positions goes out whole)
            const float th0 = tn <= LS ? -INFINITY : warp_kth_largest(lm, KP);
            bool cand[kTileJ];
            unsigned msk[kTileJ];
            int total = 0;
#pragma unroll
            for (int j = 0; j < kTileJ; ++j) {
                cand[j] = v[j] != -INFINITY && v[j] >= th0;
                msk[j] = __ballot_sync(0xffffffffu, cand[j]);
                total += __popc(msk[j]);
            }
            if (total <= LS) {
                // the list maximum goes to slot 0 (the finalisation ranks list heads)
                const float mv = warp_max(lm);
                int i_max = 0, base = 0;
                {
                    int b2 = 0;
                    bool found = false;
#pragma unroll
                    for (int j = 0; j < kTileJ; ++j) {
                        const unsigned hm = __ballot_sync(0xffffffffu, cand[j] && v[j] == mv);
                        if (!found && hm) {
                            const int ln = __ffs(hm) - 1;
                            i_max = b2 + __popc(msk[j] & ((1u << ln) - 1u));
                            found = true;
                        }
                        b2 += __popc(msk[j]);
                    }
                }
                const size_t o = ((size_t)cta * n_h_total + h_row0 + r);
#pragma unroll
                for (int j = 0; j < kTileJ; ++j) {
                    if (cand[j]) {
                        int idx = base + __popc(msk[j] & ((1u << lane) - 1u));
                        idx = idx == i_max ? 0 : (idx == 0 ? i_max : idx);
                        P.val[o * LS + idx] = v[j];
                        P.id[o * LS + idx] = base_pos + lane + 32 * j;
                    }
                    base += __popc(msk[j]);
                }
                if (lane == 0) e.st_xcnt[r] = total;
                __syncwarp();
                continue;
            }
        }
        if (KP > 32 || cnt < KP) {
            if (KP <= 32) fold_topk32(e, r, KP, tn, base_pos, warp, v, lm);
            else if (KP <= 64) fold_row<2>(e, r, KP, tn, base_pos);
            else fold_row<3>(e, r, KP, tn, base_pos);
            continue;
        }
        const float tv = e.st_val[r * KP + KP - 1];
        const int tp = e.st_pos[r * KP + KP - 1];
        bool cand[kTileJ];
        unsigned msk[kTileJ];
        int total = 0;
#pragma unroll
        for (int j = 0; j < kTileJ; ++j) {
            cand[j] = v[j] != -INFINITY && before(v[j], base_pos + lane + 32 * j, tv, tp);
            msk[j] = __ballot_sync(0xffffffffu, cand[j]);
            total += __popc(msk[j]);
        }
        if (total > LS - KP) {
            fold_topk32(e, r, KP, tn, base_pos, warp, v, lm);
            continue;
        }
        const size_t o = ((size_t)cta * n_h_total + h_row0 + r);
        int base = cnt;
#pragma unroll
        for (int j = 0; j < kTileJ; ++j) {
            if (cand[j]) {
                const int idx = base + __popc(msk[j] & ((1u << lane) - 1u));
                P.val[o * LS + idx] = v[j];
                P.id[o * LS + idx] = base_pos + lane + 32 * j;
            }
            base += __popc(msk[j]);
        }
        if (lane == 0) e.st_xcnt[r] = total;
        __syncwarp();
    }
}


// ---------------------------------------------------------------- buffered path
// KP <= 32 on the tensor-core kernel: no sorted list per row, but an unsorted
// buffer of at most kBuf (position, value) candidates and an admission bound
// (thv, thp): an element that is not before(thv, thp) under (value desc,
// position asc) cannot be among the CTA's best KP. The buffer always holds a
// superset of the CTA's best KP seen so far, and the finalisation selects from
// the flat lists exactly. Per tile and row the work is a ballot and an append;
// only the first tile pays a bound (the KP-th largest of the 32 lane maxima:
// KP distinct values at or above it), and only an overflowing buffer pays an
// exact rank-by-count compaction to its best KP (sorted; the bound becomes the
// KP-th entry).
// The buffer's best KP, sorted, into slots [0, KP) (cnt <= kBuf = 64): bitonic
// sort of each 32-slot half, one bitonic merge; returns the new bound.
ES_DEV void buf_compact_sorted(float* bv, int* bp, int cnt, int KP, float& thv, int& thp) {
    const int lane = lane_id();
    float x0 = lane < cnt ? bv[lane] : -INFINITY;
    int q0 = lane < cnt ? bp[lane] : 0x7fffffff;
    warp_sort32(x0, q0);
    if (cnt > 32) {
        float x1 = lane + 32 < cnt ? bv[lane + 32] : -INFINITY;
        int q1 = lane + 32 < cnt ? bp[lane + 32] : 0x7fffffff;
        warp_sort32(x1, q1);
        const float rv = __shfl_sync(0xffffffffu, x1, 31 - lane);
        const int rp = __shfl_sync(0xffffffffu, q1, 31 - lane);
        if (before(rv, rp, x0, q0)) { x0 = rv; q0 = rp; }
#pragma unroll
        for (int j = 16; j > 0; j >>= 1) {
            const float ov = __shfl_xor_sync(0xffffffffu, x0, j);
            const int op = __shfl_xor_sync(0xffffffffu, q0, j);
            if (((lane & j) == 0) == before(ov, op, x0, q0)) { x0 = ov; q0 = op; }
        }
    }
    __syncwarp();
    if (lane < KP) { bv[lane] = x0; bp[lane] = q0; }
    thv = __shfl_sync(0xffffffffu, x0, KP - 1);
    thp = __shfl_sync(0xffffffffu, q0, KP - 1);
    __syncwarp();
}

ES_DEV void fold_buf(const EpiSmem& e, int r, int KP, int tn, int base_pos, const float (&v)[kTileJ], float lm,
                     bool tighten, float* scr_v, int* scr_p) {
    const int lane = lane_id();
    int cnt = e.st_cnt[r];
    float thv = e.st_thv[r];
    int thp = e.st_thp[r];
    if (cnt == 0 && thv == -INFINITY) {
        const float t0 = warp_kth_largest(lm, KP);
        if (t0 > -INFINITY) { thv = t0; thp = 0x7fffffff; }
    }
    if (__any_sync(0xffffffffu, lm >= thv)) {
        bool cand[kTileJ];
        unsigned msk[kTileJ];
        int c = 0;
#pragma unroll
        for (int j = 0; j < kTileJ; ++j) {
            const int pj = tile_key(e, base_pos, lane + 32 * j);
            cand[j] = v[j] != -INFINITY && before(v[j], pj, thv, thp);
            msk[j] = __ballot_sync(0xffffffffu, cand[j]);
            c += __popc(msk[j]);
        }
        float* bv = e.st_val + (size_t)r * kBuf;
        int* bp = e.st_pos + (size_t)r * kBuf;
        if (cnt + c > kBuf && cnt > KP) {
            // make room: the buffer's best KP, then re-admit against the tighter bound
            buf_compact_sorted(bv, bp, cnt, KP, thv, thp);
            cnt = KP;
            c = 0;
#pragma unroll
            for (int j = 0; j < kTileJ; ++j) {
                cand[j] = cand[j] && before(v[j], tile_key(e, base_pos, lane + 32 * j), thv, thp);
                msk[j] = __ballot_sync(0xffffffffu, cand[j]);
                c += __popc(msk[j]);
            }
        }
        if (cnt + c <= kBuf) {
            int base = cnt;
#pragma unroll
            for (int j = 0; j < kTileJ; ++j) {
                if (cand[j]) {
                    const int idx = base + __popc(msk[j] & ((1u << lane) - 1u));
                    bv[idx] = v[j];
                    bp[idx] = tile_key(e, base_pos, lane + 32 * j);
                }
                base += __popc(msk[j]);
            }
            cnt += c;
        } else if (c > 0) {
            // more than kBuf - KP candidates against a buffer of at most KP: the sorted
            // buffer becomes a register list and the candidates are merged into it in
            // sorted batches of 32 (warp scratch), keeping the best 32
            float Lv = lane < cnt ? bv[lane] : -INFINITY;
            int Lp = lane < cnt ? bp[lane] : 0x7fffffff;
            warp_sort32(Lv, Lp);
            for (int done = 0; done < c; done += 32) {
                int base = 0;
#pragma unroll
                for (int j = 0; j < kTileJ; ++j) {
                    const int idx = base + __popc(msk[j] & ((1u << lane) - 1u)) - done;
                    if (cand[j] && idx >= 0 && idx < 32) { scr_v[idx] = v[j]; scr_p[idx] = tile_key(e, base_pos, lane + 32 * j); }
                    base += __popc(msk[j]);
                }
                __syncwarp();
                const int nb = min(32, c - done);
                float xv = lane < nb ? scr_v[lane] : -INFINITY;
                int xp = lane < nb ? scr_p[lane] : 0x7fffffff;
                __syncwarp();
                warp_sort32(xv, xp);
                const float rv = __shfl_sync(0xffffffffu, xv, 31 - lane);
                const int rp = __shfl_sync(0xffffffffu, xp, 31 - lane);
                if (before(rv, rp, Lv, Lp)) { Lv = rv; Lp = rp; }
#pragma unroll
                for (int j = 16; j > 0; j >>= 1) {
                    const float ov = __shfl_xor_sync(0xffffffffu, Lv, j);
                    const int op = __shfl_xor_sync(0xffffffffu, Lp, j);
                    if (((lane & j) == 0) == before(ov, op, Lv, Lp)) { Lv = ov; Lp = op; }
                }
            }
            if (lane < KP) { bv[lane] = Lv; bp[lane] = Lp; }
            thv = __shfl_sync(0xffffffffu, Lv, KP - 1);
            thp = __shfl_sync(0xffffffffu, Lp, KP - 1);
            cnt = KP;
            __syncwarp();
        }
        // between tiles (the next tile still streams): tighten the bound to the
        // CTA's current KP-th best so that later tiles admit few candidates
        if (tighten && cnt > KP) {
            buf_compact_sorted(bv, bp, cnt, KP, thv, thp);
            cnt = KP;
        }
    }
    __syncwarp();
    if (lane == 0) { e.st_cnt[r] = cnt; e.st_thv[r] = thv; e.st_thp[r] = thp; }
    __syncwarp();
}

ES_DEV void epi_tile_buf(const EpiSmem& e, int n_h, int KP, int tn, int base_pos, int warp, int n_warps,
                         bool tighten) {
    if (tn <= 0) return;
    const int lane = lane_id();
    for (int r = warp; r < n_h; r += n_warps) {
        float v[kTileJ];
        float lm = -INFINITY;
#pragma unroll
        for (int j = 0; j < kTileJ; ++j) {
            const int p = lane + 32 * j;
            v[j] = p < tn ? e.tile[r * kTile + p] : -INFINITY;
            lm = fmaxf(lm, v[j]);
        }
        fold_softmax(e, r, v, lm);
        fold_buf(e, r, KP, tn, base_pos, v, lm, tighten, e.scr_v + warp * 32, e.scr_p + warp * 32);
    }
}

// Buffered path store of one row: the buffer's entries, all "extras" (cnt = 0,
// xcnt entries), list stride LS; slots past xcnt are never read (no pads).
ES_DEV void store_row_buf(const EpiSmem& e, const LmhPartials& P, int cta, int n_h_total, int h_row0, int r, int LS) {
    const int lane = lane_id();
    const int cnt = e.st_cnt[r];
    const size_t o = ((size_t)cta * n_h_total + h_row0 + r);
    for (int i = lane; i < cnt; i += 32) {
        P.val[o * LS + i] = e.st_val[(size_t)r * kBuf + i];
        P.id[o * LS + i] = e.st_pos[(size_t)r * kBuf + i];
    }
    const float ssum = warp_sum(e.st_ls[r * 32 + lane]);
    if (lane == 0) {
        P.cnt[part_st(P, cta, h_row0 + r)] = 0;
        P.xcnt[part_st(P, cta, h_row0 + r)] = cnt;
        P.m[part_st(P, cta, h_row0 + r)] = e.st_m[r];
        P.s[part_st(P, cta, h_row0 + r)] = ssum;
    }
}

ES_DEV void epi_store_buf(const EpiSmem& e, const LmhPartials& P, int cta, int n_h_total, int h_row0, int n_h,
                          int warp, int n_warps, int LS) {
    for (int r = warp; r < n_h; r += n_warps) store_row_buf(e, P, cta, n_h_total, h_row0, r, LS);
}

// The CTA's last tile (all warps): fold, then store each row right away (the
// warp that folds a row writes its partial list -- no block-wide barrier).
ES_DEV void epi_tile_buf_last_store(const EpiSmem& e, const LmhPartials& P, int cta, int n_h_total, int h_row0,
                                    int n_h, int KP, int LS, int tn, int base_pos, int warp, int n_warps,
                                    long long* dtr = nullptr) {
    const int lane = lane_id();
    int it = 0;
    for (int r = warp; r < n_h; r += n_warps, ++it) {
        if (dtr && lane == 0 && it < 5) dtr[it * 4 + 0] = clock64();
        if (tn > 0) {
            float v[kTileJ];
            float lm = -INFINITY;
#pragma unroll
            for (int j = 0; j < kTileJ; ++j) {
                const int p = lane + 32 * j;
                v[j] = p < tn ? e.tile[r * kTile + p] : -INFINITY;
                lm = fmaxf(lm, v[j]);
            }
            fold_softmax(e, r, v, lm);
            if (dtr && lane == 0 && it < 5) dtr[it * 4 + 1] = clock64();
            fold_buf(e, r, KP, tn, base_pos, v, lm, false, e.scr_v + warp * 32, e.scr_p + warp * 32);
            if (dtr && lane == 0 && it < 5) dtr[it * 4 + 2] = clock64();
        }
        store_row_buf(e, P, cta, n_h_total, h_row0, r, LS);
        if (dtr && lane == 0 && it < 5) dtr[it * 4 + 3] = clock64();
    }
}

// ---------------------------------------------------------------- thread-parallel fold
// Buffered path (KP <= 32), tensor-core kernel. The warp-per-row fold above is a
// chain of shuffles and shared-memory round trips per row (~2,500 cycles); with
// 60 rows on 8-13 warps that chain is the exposed tail of the CTA's last tile.
// Here thread (r, g) owns positions [32 g, 32 g + 32) of row r -- kParG = 4
// adjacent lanes per row, so the row reductions are two xor shuffles:
//   softmax   tile maximum, m_new = max(m_old, it), sum of exp(z - m_new) plus
//             the rescaled old partial sums (the 32 per-row slots of st_ls);
//   bound     T = min over the 4 threads of each one's J-th largest value,
//             J = ceil(KP / 4): at least 4 J >= KP tile values are >= T, so T
//             bounds the row's KP-th best from below (ties at T admitted); the
//             tighter of T and the row's bound is kept;
//   admission candidates strictly before the bound are appended to the row's
//             buffer at a shared-memory atomic offset (st_xcnt).
// A row whose buffer would overflow keeps its count and is folded by the warp
// path (fold_buf) in phase 2, which also tightens rows between tiles and, on
// the last tile, stores the partial lists.
constexpr int kParG = 4;

ES_DEV float ex2_approx(float x) {   // 2^x, flush-to-zero (ex2 of -inf is +0)
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}


// (noinline, loops rolled: this code runs once per tile, so its instruction
// footprint -- not its issue count -- sets its cost; fully unrolled copies
// measured ~20k cycles per tile from instruction-cache misses alone)
template <int J>
ES_DEV void epi_par_phase1(const EpiSmem& e, int n_h, int tn, int base_pos, int tid, int nthr, bool last,
                           const LmhPartials& P, int cta, int n_h_total, int h_row0, int LS, long long* dtr) {
#define PTR_(i) do { if (dtr && lane == 0) dtr[i] = clock64(); } while (0)
    const int lane = lane_id();
    for (int base = tid - lane; base < n_h * kParG; base += nthr) {
        const int item = base + lane;
        const bool act = item < n_h * kParG;
        const int r = act ? item >> 2 : n_h - 1;   // idle lanes mirror a real row, write nothing
        const int g = item & (kParG - 1);
        const int rot = item & 7;                  // rotated float4 order: a quarter-warp hits 8 distinct bank groups
        const float* trow = e.tile + (size_t)r * kTile + g * 32;
        // the thread's 32 values are read from shared memory in three passes (bound,
        // softmax + admission, candidate writes) instead of being held in registers
        auto ld4 = [&](int j, float (&x)[4]) {
            const int q = (j + rot) & 7;
            const float4 f = *(const float4*)(trow + 4 * q);
            const int p = g * 32 + 4 * q;
            x[0] = p + 0 < tn ? f.x : -INFINITY;
            x[1] = p + 1 < tn ? f.y : -INFINITY;
            x[2] = p + 2 < tn ? f.z : -INFINITY;
            x[3] = p + 3 < tn ? f.w : -INFINITY;
        };
        PTR_(3);
        // row state, read by all four threads before any of them writes
        const float m_old = e.st_m[r];
        float thv = e.st_thv[r];
        int thp = e.st_thp[r];
        const int n_old = e.st_cnt[r];
        const float4 o0 = *(const float4*)&e.st_ls[r * 32 + g * 8];
        const float4 o1 = *(const float4*)&e.st_ls[r * 32 + g * 8 + 4];
        __syncwarp();
        // pass 1: maximum; on a row's first tile (no bound yet) also this thread's
        // J-th largest (branch-free insertion into a sorted top-J)
        float lm = -INFINITY, t = -INFINITY;
        if (thv == -INFINITY) {   // uniform over the row's four lanes
            float top[J];
#pragma unroll
            for (int i = 0; i < J; ++i) top[i] = -INFINITY;
#pragma unroll 2
            for (int j = 0; j < 8; ++j) {
                float x4[4];
                ld4(j, x4);
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float x = x4[c];
                    lm = fmaxf(lm, x);
#pragma unroll
                    for (int s2 = 0; s2 < J; ++s2) {
                        const float hi = fmaxf(top[s2], x);
                        x = fminf(top[s2], x);
                        top[s2] = hi;
                    }
                }
            }
            t = top[J - 1];
        } else {
#pragma unroll 4
            for (int j = 0; j < 8; ++j) {
                float x4[4];
                ld4(j, x4);
                lm = fmaxf(fmaxf(lm, fmaxf(x4[0], x4[1])), fmaxf(x4[2], x4[3]));
            }
        }
        t = fminf(t, __shfl_xor_sync(0xffffffffu, t, 1));
        t = fminf(t, __shfl_xor_sync(0xffffffffu, t, 2));
        if (t > thv) { thv = t; thp = 0x7fffffff; }
        float rm = fmaxf(lm, __shfl_xor_sync(0xffffffffu, lm, 1));
        rm = fmaxf(rm, __shfl_xor_sync(0xffffffffu, rm, 2));
        const float m_new = fmaxf(m_old, rm);
        PTR_(0);
        // pass 2, branch-free: sum of 2^((z - m) log2 e) (ex2 of -inf is 0, so masked
        // positions drop out) and admission (strictly before the bound)
        const float mb = m_new == -INFINITY ? 0.0f : m_new * 1.4426950408889634f;
        float sum0 = 0.0f, sum1 = 0.0f;
        unsigned cm = 0u, em = 0u;
#pragma unroll 4
        for (int j = 0; j < 8; ++j) {
            float x4[4];
            ld4(j, x4);
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float ex = ex2_approx(fmaf(x4[c], 1.4426950408889634f, -mb));
                if (c & 1) sum1 += ex; else sum0 += ex;
                // (bitwise, not short-circuit: no branch per value); values equal to the
                // bound are admitted by key below (rare)
                cm |= (unsigned)(x4[c] > thv) << (4 * j + c);
                em |= ((unsigned)(x4[c] == thv) & (unsigned)(x4[c] != -INFINITY)) << (4 * j + c);
            }
        }
        while (em) {
            const int i = __ffs(em) - 1;
            em &= em - 1u;
            if (tile_key(e, base_pos, g * 32 + 4 * (((i >> 2) + rot) & 7) + (i & 3)) < thp) cm |= 1u << i;
        }
        float sum = sum0 + sum1;
        PTR_(1);
        const float so = ((o0.x + o0.y) + (o0.z + o0.w)) + ((o1.x + o1.y) + (o1.z + o1.w));
        if (so != 0.0f) sum += so * ex2_approx((m_old - m_new) * 1.4426950408889634f);
        if (act) {
            *(float4*)&e.st_ls[r * 32 + g * 8] = make_float4(sum, 0.0f, 0.0f, 0.0f);
            *(float4*)&e.st_ls[r * 32 + g * 8 + 4] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
            if (g == 0) { e.st_m[r] = m_new; e.st_thv[r] = thv; e.st_thp[r] = thp; }
        }
        if (last) {   // the row's softmax state goes straight to the partials
            float tot = sum + __shfl_xor_sync(0xffffffffu, sum, 1);
            tot += __shfl_xor_sync(0xffffffffu, tot, 2);
            if (act && g == 0) {
                const size_t o = (size_t)cta * n_h_total + h_row0 + r;
                P.m[part_st(P, cta, h_row0 + r)] = m_new;
                P.s[part_st(P, cta, h_row0 + r)] = tot;
            }
        }
        PTR_(2);
        // pass 3 (candidates only): offsets within the row's group of kParG adjacent lanes by
        // two shuffles (no atomics); on the CTA's last tile the candidates go straight into the
        // row's global list behind the buffer's n_old entries, which the group copies too, and
        // the list's count is final here -- no second phase unless a row overflows
        const int nc = act ? __popc(cm) : 0;
        int pre = nc;   // inclusive prefix over the group
        {
            int t = __shfl_up_sync(0xffffffffu, pre, 1);
            if (g >= 1) pre += t;
            t = __shfl_up_sync(0xffffffffu, pre, 2);
            if (g >= 2) pre += t;
        }
        const int gtot = __shfl_sync(0xffffffffu, pre, lane | (kParG - 1));
        const int cap = last ? LS : kBuf;
        const bool fits = n_old + gtot <= cap;   // else the row overflows: phase 2 folds it (fold_buf)
        if (act && g == 0) {
            e.st_xcnt[r] = gtot;
            if (!fits) e.st_flag[0] = 1;
            if (last && fits) {
                const size_t o = (size_t)cta * n_h_total + h_row0 + r;
                P.cnt[part_st(P, cta, h_row0 + r)] = 0;
                P.xcnt[part_st(P, cta, h_row0 + r)] = n_old + gtot;
            }
        }
        if (act && fits) {
            const size_t go = ((size_t)cta * n_h_total + h_row0 + r) * LS;
            float* bv = last ? P.val + go : e.st_val + (size_t)r * kBuf;
            int* bp = last ? P.id + go : e.st_pos + (size_t)r * kBuf;
            int at = n_old + pre - nc;
            while (cm) {
                const int i = __ffs(cm) - 1;
                cm &= cm - 1u;
                const int pl = g * 32 + 4 * (((i >> 2) + rot) & 7) + (i & 3);
                bv[at] = trow[pl - g * 32];
                bp[at] = tile_key(e, base_pos, pl);
                ++at;
            }
            if (last)   // the buffer's entries into slots [0, n_old)
                for (int i = g; i < n_old; i += kParG) {
                    bv[i] = e.st_val[(size_t)r * kBuf + i];
                    bp[i] = e.st_pos[(size_t)r * kBuf + i];
                }
        }
    }
}

ES_DEV void epi_par_phase1_any(const EpiSmem& e, int n_h, int KP, int tn, int base_pos, int tid, int nthr,
                               bool last, const LmhPartials& P, int cta, int n_h_total, int h_row0, int LS,
                               long long* dtr = nullptr) {
    // J = ceil(KP / 4) would be exact; three instantiations keep the code small
    // (a larger J is still a valid bound, only a looser one)
    if (KP <= 12) epi_par_phase1<3>(e, n_h, tn, base_pos, tid, nthr, last, P, cta, n_h_total, h_row0, LS, dtr);
    else if (KP <= 20) epi_par_phase1<5>(e, n_h, tn, base_pos, tid, nthr, last, P, cta, n_h_total, h_row0, LS, dtr);
    else epi_par_phase1<8>(e, n_h, tn, base_pos, tid, nthr, last, P, cta, n_h_total, h_row0, LS, dtr);
}

// Phase 2 (after a barrier over the group of nthr threads, named barrier bar):
//   2a only if phase 1 raised the block flag: overflowed rows (their candidates
//      were not written) take the warp fold (fold_buf) -- on the last tile this
//      is all phase 2 does (phase 1 wrote the lists);
//   2b between tiles, one thread per row commits the appended count;
//   2c between tiles, one warp per row compacts a buffer above KP entries to its
//      best KP (the bound becomes its KP-th entry) -- hidden behind streaming.
// On the last tile the global list is the buffer's entries followed by the
// tile's candidates (stride LS = 128 > kBuf, so a last tile cannot overflow in
// practice; no pads: the finalisation reads xcnt entries; its maximum is m).
ES_DEV void epi_par_phase2(const EpiSmem& e, int n_h, int KP, int tn, int base_pos, int tid, int nthr, int bar,
                           bool last, const LmhPartials& P, int cta, int n_h_total, int h_row0, int LS,
                           long long* ovf = nullptr) {
    const int lane = lane_id(), warp = tid >> 5, n_warps = nthr >> 5;
    const int cap = last ? LS : kBuf;
    if (e.st_flag[0]) {   // uniform (set in phase 1, read after the caller's barrier): overflowed rows
        for (int r = warp; r < n_h; r += n_warps) {
            const int add = e.st_xcnt[r];
            if (add == 0 || e.st_cnt[r] + add <= cap) continue;
            if (ovf && lane == 0) atomicAdd((unsigned long long*)ovf, 1ull);
            float v[kTileJ];
            float lm = -INFINITY;
#pragma unroll
            for (int j = 0; j < kTileJ; ++j) {
                const int p = lane + 32 * j;
                v[j] = p < tn ? e.tile[r * kTile + p] : -INFINITY;
                lm = fmaxf(lm, v[j]);
            }
            // (the buffer still holds only the earlier tiles' entries: fold the tile into it)
            fold_buf(e, r, KP, tn, base_pos, v, lm, !last, e.scr_v + warp * 32, e.scr_p + warp * 32);
            if (last) {   // the list: the buffer's entries
                const size_t o = (size_t)cta * n_h_total + h_row0 + r;
                const int cnt = e.st_cnt[r];
                for (int i = lane; i < cnt; i += 32) {
                    P.val[o * LS + i] = e.st_val[(size_t)r * kBuf + i];
                    P.id[o * LS + i] = e.st_pos[(size_t)r * kBuf + i];
                }
                if (lane == 0) { P.cnt[part_st(P, cta, h_row0 + r)] = 0; P.xcnt[part_st(P, cta, h_row0 + r)] = cnt; }
            }
            __syncwarp();
            if (lane == 0) e.st_xcnt[r] = 0;
            __syncwarp();
        }
        named_bar_sync(bar, nthr);
        if (tid == 0) e.st_flag[0] = 0;
    }
    if (last) return;
    for (int r = tid; r < n_h; r += nthr) {   // commit the appended counts
        e.st_cnt[r] += e.st_xcnt[r];
        e.st_xcnt[r] = 0;
    }
    named_bar_sync(bar, nthr);
    // between tiles (the next tile still streams): compact buffers above KP entries to their
    // best KP, the bound becomes the KP-th entry
    for (int r = warp; r < n_h; r += n_warps) {
        const int cnt = e.st_cnt[r];
        if (cnt > KP) {
            float thv;
            int thp;
            buf_compact_sorted(e.st_val + (size_t)r * kBuf, e.st_pos + (size_t)r * kBuf, cnt, KP, thv, thp);
            if (lane == 0) { e.st_cnt[r] = KP; e.st_thv[r] = thv; e.st_thp[r] = thp; }
            __syncwarp();
        }
    }
}

}  // namespace es
