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
// against the current tile, which the strict comparison below implements.
#pragma once
#include "common.cuh"
#include "kernels.cuh"

namespace es {

constexpr int kTile = 128;

struct EpiSmem {
    float* tile;     // [n_h][kTile]
    float* st_val;   // [n_h][KP]
    int* st_pos;     // [n_h][KP]
    int* st_cnt;     // [n_h]
    float* st_m;     // [n_h]
    float* st_s;     // [n_h]
    float* scr_val;  // [n_warps][KP]
    int* scr_pos;    // [n_warps][KP]
};

ES_DEV size_t epi_smem_bytes(int n_h, int KP, int n_warps) {
    return (size_t)n_h * kTile * 4 + (size_t)n_h * KP * 8 + (size_t)n_h * 12 + (size_t)n_warps * KP * 8;
}

ES_DEV EpiSmem epi_carve(unsigned char* p, int n_h, int KP, int n_warps) {
    EpiSmem e;
    e.tile = (float*)p;        p += (size_t)n_h * kTile * 4;
    e.st_val = (float*)p;      p += (size_t)n_h * KP * 4;
    e.st_pos = (int*)p;        p += (size_t)n_h * KP * 4;
    e.st_cnt = (int*)p;        p += (size_t)n_h * 4;
    e.st_m = (float*)p;        p += (size_t)n_h * 4;
    e.st_s = (float*)p;        p += (size_t)n_h * 4;
    e.scr_val = (float*)p;     p += (size_t)n_warps * KP * 4;
    e.scr_pos = (int*)p;
    return e;
}

ES_DEV void epi_init(const EpiSmem& e, int n_h) {
    for (int r = threadIdx.x; r < n_h; r += blockDim.x) {
        e.st_cnt[r] = 0;
        e.st_m[r] = -INFINITY;
        e.st_s[r] = 0.0f;
    }
}

// local best of the lane's kTile/32 values under (value desc, pos asc)
ES_DEV void lane_best(const float (&v)[kTile / 32], int base_pos, int lane, float& bv, int& bp) {
    bv = -INFINITY;
    bp = 0x7fffffff;
#pragma unroll
    for (int j = 0; j < kTile / 32; ++j) {
        int p = base_pos + lane + 32 * j;
        if (v[j] != -INFINITY && before(v[j], p, bv, bp)) { bv = v[j]; bp = p; }
    }
}

// Fold the current tile (tn valid positions starting at global position
// base_pos) into the state of rows r = warp, warp + n_warps, ...
ES_DEV void epi_tile(const EpiSmem& e, int n_h, int KP, int tn, int base_pos, int warp, int n_warps) {
    const int lane = lane_id();
    float* sv = e.scr_val + warp * KP;
    int* sp = e.scr_pos + warp * KP;
    for (int r = warp; r < n_h; r += n_warps) {
        float v[kTile / 32];
        float mx = -INFINITY;
#pragma unroll
        for (int j = 0; j < kTile / 32; ++j) {
            int p = lane + 32 * j;
            v[j] = p < tn ? e.tile[r * kTile + p] : -INFINITY;
            mx = fmaxf(mx, v[j]);
        }
        mx = warp_max(mx);
        if (tn <= 0) continue;
        // online softmax
        const float m_old = e.st_m[r];
        const float m_new = fmaxf(m_old, mx);
        float acc = 0.0f;
#pragma unroll
        for (int j = 0; j < kTile / 32; ++j)
            if (v[j] != -INFINITY) acc += expf(v[j] - m_new);
        acc = warp_sum(acc);
        // top-KP merge
        const int cnt = e.st_cnt[r];
        const float theta = cnt == KP ? e.st_val[r * KP + KP - 1] : -INFINITY;
        __syncwarp();
        if (lane == 0) {
            e.st_s[r] = e.st_s[r] * (m_old == -INFINITY ? 0.0f : expf(m_old - m_new)) + acc;
            e.st_m[r] = m_new;
        }
        if (!(mx > theta) && cnt == KP) { __syncwarp(); continue; }
        float bv; int bp;
        lane_best(v, base_pos, lane, bv, bp);
        warp_argbest(bv, bp);
        int a = 0, produced = 0;
        while (produced < KP) {
            const bool tile_ok = bp != 0x7fffffff;
            const bool old_ok = a < cnt;
            if (!tile_ok && !old_ok) break;
            const float ov = old_ok ? e.st_val[r * KP + a] : -INFINITY;
            const int op = old_ok ? e.st_pos[r * KP + a] : 0x7fffffff;
            if (tile_ok && (!old_ok || before(bv, bp, ov, op))) {
                if (lane == 0) { sv[produced] = bv; sp[produced] = bp; }
                const int lp = bp - base_pos;        // remove it from the tile
                if ((lp & 31) == lane) {
#pragma unroll
                    for (int j = 0; j < kTile / 32; ++j) if (j == (lp >> 5)) v[j] = -INFINITY;
                }
                lane_best(v, base_pos, lane, bv, bp);
                warp_argbest(bv, bp);
            } else {
                if (lane == 0) { sv[produced] = ov; sp[produced] = op; }
                ++a;
            }
            ++produced;
        }
        __syncwarp();
        for (int i = lane; i < produced; i += 32) {
            e.st_val[r * KP + i] = sv[i];
            e.st_pos[r * KP + i] = sp[i];
        }
        if (lane == 0) e.st_cnt[r] = produced;
        __syncwarp();
    }
}

// Write the CTA's state to the global partials (positions -> global ids).
ES_DEV void epi_store(const EpiSmem& e, const LmhPartials& P, int cta, int n_h_total, int h_row0,
                      int n_h, int KP, const int32_t* subset) {
    for (int r = warp_id(); r < n_h; r += blockDim.x / 32) {
        const int cnt = e.st_cnt[r];
        const size_t o = ((size_t)cta * n_h_total + h_row0 + r);
        for (int i = lane_id(); i < KP; i += 32) {
            P.val[o * KP + i] = i < cnt ? e.st_val[r * KP + i] : -INFINITY;
            P.id[o * KP + i] = i < cnt ? subset[e.st_pos[r * KP + i]] : -1;
        }
        if (lane_id() == 0) {
            P.cnt[o] = cnt;
            P.m[o] = e.st_m[r];
            P.s[o] = e.st_s[r];
        }
    }
}

}  // namespace es
