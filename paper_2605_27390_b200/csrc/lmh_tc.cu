// lmh_tc.cu -- a5-a7 on the 5th-generation tensor cores for draft trees with
// n_h >= 5 (the paper's 60-node tree): at arithmetic
// intensity n_h flop/byte FFMA cannot keep pace with HBM, tcgen05 can.
//
//   z[r][j] = inv_temp * sum_c H[r][c] W[S_j][c]    (Eq. projection P:44-48,
//                                                    restricted to V_t)
//
// Swap-AB: the MMA's M dimension is 128 gathered vocabulary rows of W[S]
// (A, K-major), N is the tree width padded to a multiple of 16 (B = H,
// K-major), the fp32 accumulator D[128 x N] lives in TMEM.
//
// Persistent, warp-specialised CTA per SM (13 warps):
//   warps 0-3  producers: 16-byte cp.async of the gathered W rows into a
//           128B-swizzled smem stage (swizzle applied in the address), one
//           cp.async.mbarrier.arrive.noinc per thread (rows past a tile's end
//           skipped); H by one 2D TMA tile per stage.
//   warp 4  TMEM allocator + MMA issuer (one elected thread):
//           4 x tcgen05.mma.cta_group::1.kind::f16 (K = 16) per stage,
//           tcgen05.commit frees the stage; double-buffered accumulators.
//   warps 5-12 epilogue: tcgen05.ld 32x32b -> scale -> smem tile -> the
//           shared online-softmax + candidate-buffer fold (lmh_epilogue.cuh)
//           while the producers and MMA already stream the next tile; the
//           CTA's last tile is folded (and its rows stored) by all 13 warps.
// Segment mode (ragged head): CTAs serve (row group, position range) segments.
#include <algorithm>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"
#include "lmh_epilogue.cuh"

namespace es {

// W-operand producer: 4 warps of 16-byte cp.async (LDGSTS) with the 128B
// swizzle applied in the address, one mbarrier arrival per thread
// (cp.async.mbarrier.arrive.noinc). A TMA tile::gather4 producer (one warp,
// round-1 history) measured issue-bound at ~1.6 TB/s for 128-byte row pieces;
// LDGSTS streams the same gathered rows at HBM rate.
constexpr int kProdWarps = 4;
constexpr int kTcMmaWarp = kProdWarps;
constexpr int kTcEpiWarp0 = kProdWarps + 1;
constexpr int kTcEpiWarps = 8;
constexpr int kTcWarps = kProdWarps + 1 + kTcEpiWarps;
constexpr int kBlockK = 64;        // bf16 columns per stage = one 128-byte swizzle atom row
constexpr int kTileM = 128;
constexpr int kLastTile = 128;    // rows of a short last tile (128 = no split; see the launch)

#define TC_TRACE(slot) do { if (a.trace) a.trace[(size_t)blockIdx.x * 8 + (slot)] = gtime(); } while (0)


// ------------------------------------------------------------------ kernel
struct TcParams {
    int n_pad;       // N: tree rows padded to a multiple of 16 (<= 128)
    int stages;
    int nkb;         // d / 64
    uint32_t tmem_cols;
    int last_tile;   // rows of a CTA's short last tile (ranges longer than one tile)
    int dyn_tile;    // two-list mode: rows per second-list tile (EVOSPEC_DYN_TILE)
    int dyn_stride;  // two-list mode: CTA rank stride of the second-list round robin
    int dyn_share;   // two-list mode: first-list share (16ths) of the CTAs expected to take a second-list tile
    size_t off_b, off_epi, off_bar, off_rows;  // smem carve offsets
};

ES_DEV int dyn_rank_of(int b, int stride, int grid) { return (int)(((long long)b * stride) % grid); }

// Two-list mode, early second list: producer warp 0 polls the union's flag (one
// poller per CTA) and hands the outcome to the other warps through shared memory.
// Returns the list's length, or -1 (wait for the union's end).
__device__ __noinline__ int lmh_list2_resolve(const int* flag, int n_max, int* s_n2, int warp, int lane) {
    int v;
    if (warp == 0) {
        int f = 0;
        if (lane == 0) {
            const long long t0 = globaltimer_ns();
            for (;;) {
                asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(flag) : "memory");
                if (f != 0) break;
                if (globaltimer_ns() - t0 > 200000000LL) __trap();   // (200 ms: the union never published)
                __nanosleep(256);
            }
        }
        f = __shfl_sync(0xffffffffu, f, 0);
        v = f > 0 ? min(f - 1, n_max) : -1;
        if (lane == 0) asm volatile("st.release.cta.shared.b32 [%0], %1;" ::"r"(smem_u32(s_n2)), "r"(v) : "memory");
    } else {
        for (;;) {
            asm volatile("ld.acquire.cta.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(s_n2)) : "memory");
            if (v != -2) break;
            __nanosleep(64);
        }
    }
    return v;
}

__global__ void __launch_bounds__(kTcWarps * 32, 1)
lmh_tc_kernel(const __grid_constant__ CUtensorMap tmap_w, const __grid_constant__ CUtensorMap tmap_h,
              LmhArgs a, TcParams tp) {
    extern __shared__ __align__(1024) unsigned char tc_sm[];
    // 1024-align the stage ring (SWIZZLE_128B atoms)
    unsigned char* base = tc_sm + ((1024u - (smem_u32(tc_sm) & 1023u)) & 1023u);   // stays a shared-window pointer (LDS/STS, not generic LD/ST)
    const int S = tp.stages, NP = tp.n_pad;
    // rows of this CTA: all n_h, or (segment mode) its segment's rows [h_row0, h_row0 + n_h)
    int n_h = a.n_h, h_row0 = 0, seg_b = -1, seg_c0 = 0, seg_m = 1;
    if (a.nseg > 0) {
        if (a.seg_cta) {
            pdl_wait();                              // the schedule comes from the previous kernel
            seg_b = 0;
            while (seg_b < a.nseg && a.seg_cta[seg_b + 1] <= (int)blockIdx.x) ++seg_b;
            if (seg_b < a.nseg) { seg_c0 = a.seg_cta[seg_b]; seg_m = a.seg_cta[seg_b + 1] - seg_c0; }
        } else {
            seg_b = blockIdx.x / a.seg_ctas;
            seg_c0 = seg_b * a.seg_ctas;
            seg_m = a.seg_ctas;
        }
        if (seg_b >= a.nseg || a.seg_h[seg_b + 1] == a.seg_h[seg_b]) return;   // idle: no segment, or no rows
        h_row0 = a.seg_h[seg_b];
        n_h = a.seg_h[seg_b + 1] - h_row0;
    }
    unsigned char* smA = base;                                   // [S][128][128 B]
    unsigned char* smB = base + tp.off_b;                        // [S][NP][128 B]
    const bool buffered = a.KP <= 32 && a.LS >= kBuf;   // unsorted candidate buffers (lmh_epilogue.cuh)
    // buffered lists carry vocabulary ids (keys) instead of subset positions (a.gid_keys)
    EpiSmem e = epi_carve(base + tp.off_epi, a.nseg > 0 ? a.seg_rows : n_h, buffered ? kBuf : a.KP, kTcWarps,
                          buffered && a.gid_keys);
    uint64_t* full = (uint64_t*)(base + tp.off_bar);             // [S]
    uint64_t* empty = full + S;                                  // [S]
    uint64_t* tfull = empty + S;                                 // [2]
    uint64_t* tempty = tfull + 2;                                // [2]
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
    // two-list mode, early list: its length (-1: wait for the union's end; -2: not known yet)
    int& s_n2 = *(int*)(tmem_slot + 1);

    const int warp = warp_id(), lane = lane_id();
    const int pcta = a.part_cta0 + (int)blockIdx.x;   // this CTA's partial list / state index
    // clock64 details of CTA 0's last tile (EVOSPEC_TRACE; profiling aid)
    long long* const DTR = a.trace && blockIdx.x == 0 ? a.trace + 2 * kNumSMs * 8 + 48 : nullptr;
    if (DTR && threadIdx.x == 0) { DTR[48] = 0; DTR[49] = 0; }
    pdl_trigger();
    // setup that needs nothing from the previous kernel overlaps its tail (PDL)
    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_h) : "memory");
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], kProdWarps * 32 + 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], kTcEpiWarps * 32); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kTcMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(tp.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    epi_init(e, n_h);
    if (threadIdx.x == 0) s_n2 = -2;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // the subset (and n_S) come from the previous kernel on the stream; in two-list
    // mode the first list is an input: the wait comes before the second list only
    if (!a.list2) pdl_wait();
    int p0, p1;
    if (a.list2) {
        // the CTAs that will take a second-list tile (ranks < nd, for the list's capacity)
        // stream a smaller share of the first list: their second-list tile starts when
        // the union ends and costs a full K loop, so they should reach it earlier
        const int nd = tp.dyn_tile > 0 ? min((int)gridDim.x, (a.n_list2_max + tp.dyn_tile - 1) / tp.dyn_tile) : 0;
        const long long wt = (long long)nd * tp.dyn_share + 16LL * ((int)gridDim.x - nd);
        auto pre = [&](int b) -> long long {
            return (long long)min(b, nd) * tp.dyn_share + 16LL * max(0, b - nd);
        };
        const int rb = dyn_rank_of(blockIdx.x, tp.dyn_stride, gridDim.x);
        // ranks, not block ids, order the shares (rank r covers [pre(r), pre(r + 1)))
        p0 = (int)((long long)a.n1 * pre(rb) / wt);
        p1 = (int)((long long)a.n1 * pre(rb + 1) / wt);
    } else if (seg_b >= 0) {
        // the CTAs of a segment split its positions identically for every segment
        // with the same range, so concurrent row groups share W rows through L2
        int s0 = 0, s1;
        if (a.seg_pos) {
            s0 = a.seg_pos[seg_b];
            s1 = s0 + min(a.seg_pos[seg_b + 1] - s0, a.n_subset_max);
        } else {
            s1 = min(*a.n_subset_dev, a.n_subset_max);
        }
        const int n = max(0, s1 - s0), j = blockIdx.x - seg_c0;
        p0 = s0 + (int)((long long)n * j / seg_m);
        p1 = s0 + (int)((long long)n * (j + 1) / seg_m);
    } else {
        lmh_cta_range(a, p0, p1);
    }
    const int len = p1 - p0;
    // tiles: the CTA's range split evenly into <= 128-row tiles, except that a
    // range longer than one tile ends in a short tile of kLastTile rows -- only the
    // last tile's fold is exposed (the others overlap the next tile's streaming)
    const int last_len = len > kTileM ? min(tp.last_tile, len) : len;
    const int body = len - last_len;
    const int n_body = (body + kTileM - 1) / kTileM;
    const int n_tiles1 = n_body + (last_len > 0 ? 1 : 0);
    // two-list mode: this CTA's slice [q0, q1) of the second list (virtual positions
    // n1 + i), known only after griddepcontrol.wait -- every thread resolves it lazily
    // when its role reaches the end of the first list
    // The second list goes out in whole 128-row tiles, tile u of CTA b covering rows
    // [128 (b + G u), +128): its rows arrive only when the union ends, after the first
    // list's stream, and a few full tiles on a few CTAs stream far faster than a
    // sliver of it on every CTA (a short tile still pays all d / 64 stages of H).
    int nt2 = a.list2 ? -1 : 0, n2 = 0;
    bool early = false;   // the second list is the union's early copy (a.early_ids)
    const int32_t* l2p = a.list2;   // the second list's ids (a.list2, or a.early_ids once published)
    // the CTA's rank in the second-list round robin
    const int dyn_rank = dyn_rank_of(blockIdx.x, tp.dyn_stride, gridDim.x);
    auto ensure2 = [&]() {
        if (nt2 >= 0) return;
        if (a.early_flag) {   // (out of line: keeps the loops that call has_tile compact)
            const int v = lmh_list2_resolve(a.early_flag, a.n_list2_max, &s_n2, warp, lane);
            early = v >= 0;
            if (early) { n2 = v; l2p = a.early_ids; }
        }
        if (!early) {
            pdl_wait();
            n2 = max(0, min(*a.n_list2_dev, a.n_list2_max));
        }
        if (tp.dyn_tile == 0) {   // even split: this CTA's slice, one tile
            const int s0 = (int)((long long)n2 * blockIdx.x / gridDim.x);
            const int s1 = (int)((long long)n2 * (blockIdx.x + 1) / gridDim.x);
            nt2 = (s1 - s0 + kTileM - 1) / kTileM;
            return;
        }
        const int first = tp.dyn_tile * dyn_rank, step = tp.dyn_tile * (int)gridDim.x;
        nt2 = first < n2 ? (n2 - first + step - 1) / step : 0;
    };
    // (the early copy is read only after its flag: the first read of each line in this
    // kernel, so the read-only path fetches it from L2)
    auto id_at = [&](int vp) -> int32_t {
        return (a.list2 && vp >= a.n1) ? __ldg(&l2p[vp - a.n1]) : __ldg(&a.subset[vp]);
    };
    auto has_tile = [&](int t) -> bool {
        if (t < n_tiles1) return true;
        ensure2();
        return t < n_tiles1 + nt2;
    };

    if (threadIdx.x == 0) TC_TRACE(0);
    // thread-parallel fold for CTAs with two or more tiles; a single tile (small
    // subsets) keeps the warp fold, whose first-tile bound is tighter on short tiles
    const bool par = buffered && a.par_fold && (n_tiles1 >= 2 || a.list2);

    auto tile_range = [&](int t, int& t0, int& tn) {
        if (t >= n_tiles1) {   // two-list mode, second list
            if (tp.dyn_tile == 0) {   // even split of the CTA's slice into nt2 tiles
                const int s0 = (int)((long long)n2 * blockIdx.x / gridDim.x);
                const int s1 = (int)((long long)n2 * (blockIdx.x + 1) / gridDim.x);
                const int u = t - n_tiles1, len2 = s1 - s0;
                t0 = a.n1 + s0 + (int)((long long)len2 * u / nt2);
                tn = a.n1 + s0 + (int)((long long)len2 * (u + 1) / nt2) - t0;
                return;
            }
            const int r0 = tp.dyn_tile * (dyn_rank + (int)gridDim.x * (t - n_tiles1));   // whole tiles, round robin
            t0 = a.n1 + r0;
            tn = min(tp.dyn_tile, n2 - r0);
            return;
        }
        if (t < n_body) {
            t0 = p0 + (int)((long long)body * t / n_body);
            tn = p0 + (int)((long long)body * (t + 1) / n_body) - t0;
        } else {
            t0 = p0 + body;
            tn = last_len;
        }
    };

    if (warp < kProdWarps) {
        // ===== producers: W rows by 16-byte cp.async into the swizzled stage,
        // H by one 2D TMA tile (rows >= n_h zero-filled) per stage.
        // Thread (w, l) copies chunk l&7 of tile rows 16 i + 4 w + (l >> 3), i < 8:
        // one warp instruction moves 4 whole 128-byte row segments.
        const uint64_t pol_w = policy_evict_first(), pol_h = policy_evict_last();
        const int chunk = lane & 7;
        const size_t row_bytes = (size_t)a.d * 2;
        int stage = 0;
        uint32_t phase = 0;
        for (int t = 0;; ++t) {
            if (!has_tile(t)) break;
            int t0, tn;
            tile_range(t, t0, tn);
            const char* src[8];
            uint32_t dsto[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int row = 16 * i + 4 * warp + (lane >> 3);
                const int pos = t0 + (row < tn ? row : 0);
                src[i] = (const char*)a.W + (size_t)(id_at(pos) / a.R) * row_bytes + chunk * 16;
                dsto[i] = (uint32_t)(row * 128 + ((chunk ^ (row & 7)) << 4));
            }
            for (int kb = 0; kb < tp.nkb; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1);
                if (warp == 0 && lane == 0) {
                    mbar_arrive_expect_tx(&full[stage], (uint32_t)(NP * 128));
                    tma_load_2d(smB + (size_t)stage * NP * 128, &tmap_h, &full[stage], kb * kBlockK, h_row0, pol_h);
                }
                const uint32_t dA = smem_u32(smA + (size_t)stage * kTileM * 128);
#pragma unroll
                for (int i = 0; i < 8; ++i)   // rows past the tile's end are never read back
                    if (16 * i + 4 * warp + (lane >> 3) < tn) cp_async16(dA + dsto[i], src[i] + kb * 128, pol_w);
                cp_async_arrive_noinc(&full[stage]);
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
        }
        if (warp == 0 && lane == 0) TC_TRACE(1);
        (void)tmap_w;
    } else if (warp == kTcMmaWarp) {
        // ===== MMA issuer
        const uint32_t idesc = idesc_bf16(kTileM, NP);
        int stage = 0;
        uint32_t phase = 0;
        for (int t = 0; has_tile(t); ++t) {
            const int b = t & 1;
            const uint32_t use = (uint32_t)(t >> 1);
            if (t >= 2) mbar_wait(&tempty[b], (use - 1) & 1);
            tc_fence_after();
            const uint32_t tmem_d = tmem_base + (uint32_t)(b * NP);
            for (int kb = 0; kb < tp.nkb; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t aaddr = smem_u32(smA + (size_t)stage * kTileM * 128);
                    const uint32_t baddr = smem_u32(smB + (size_t)stage * NP * 128);
#pragma unroll
                    for (int k = 0; k < kBlockK / 16; ++k)
                        umma_bf16(tmem_d, umma_desc_sw128(aaddr + k * 32), umma_desc_sw128(baddr + k * 32), idesc,
                                  (kb | k) != 0);
                    umma_commit(&empty[stage]);
                    if (kb == tp.nkb - 1) umma_commit(&tfull[b]);
                }
                __syncwarp();
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
        }
        if (lane == 0) TC_TRACE(2);
    }
    // ===== epilogue: the 8 epilogue warps take every tile's accumulator out of TMEM
    // (lane quadrant = warp % 4; the two warps of a quadrant split the columns) and fold
    // the middle tiles; the CTA's last tile -- the exposed tail -- is folded by all 13
    // warps: the producers and the MMA warp join this loop at that tile, so the middle
    // and last tiles run ONE copy of the fold code (code run once per launch comes in
    // cold, ~2.6 cycles per instruction, tools/ubench/icache.cu; this copy is warm from
    // the middle tiles)
    const bool epi = warp >= kTcEpiWarp0;
    const int ew = warp - kTcEpiWarp0;          // 0..7 (epilogue warps)
    const int quad = warp & 3;
    const int half = ew >> 2;
    const int row = quad * 32 + lane;           // tile row (TMEM lane)
    const int nthr = kTcEpiWarps * 32;
    int t_first = 0;
    if (!epi) {
        if (a.list2) ensure2();
        const int nt = n_tiles1 + nt2;
        t_first = (nt > 0 && par) ? nt - 1 : 0x7fffffff;
    }
    for (int t = t_first; t != 0x7fffffff && has_tile(t); ++t) {
        int t0, tn;
        tile_range(t, t0, tn);
        // two-list mode: whether the last first-list tile is the CTA's last is known once the
        // union has published the second list (early, or at its end): a CTA without a
        // second-list tile folds it as its last tile, with all warps
        const bool last_t = !has_tile(t + 1);
        if (epi) {
            const int b = t & 1;
            // the tile's keys (vocabulary ids), loaded while the accumulator fills
            int key = 0x7fffffff;
            if (e.tile_id && half == 0 && row < tn) key = id_at(t0 + row);
            mbar_wait(&tfull[b], (uint32_t)(t >> 1) & 1);
            if (ew == 0 && lane == 0 && t < 2) TC_TRACE(3 + 2 * t);
            if (DTR && ew == 0 && lane == 0 && last_t) DTR[40] = clock64();
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(b * NP);
            for (int c0 = half * 16; c0 < NP; c0 += 32) {
                float v[16];
                tmem_ld16(taddr + c0, v);
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (c0 + j < n_h) e.tile[(c0 + j) * kTile + row] = v[j] * a.inv_temp;
            }
            if (e.tile_id && half == 0) e.tile_id[row] = key;
            tc_fence_before();
            mbar_arrive(&tempty[b]);
            if (DTR && ew == 0 && lane == 0 && last_t) DTR[41] = clock64();
            named_bar_sync(1, nthr);
            if (DTR && ew == 0 && lane == 0 && last_t) DTR[42] = clock64();
            if (a.logits_out) {
                for (int r = ew; r < n_h; r += kTcEpiWarps)
                    for (int p = lane; p < tn; p += 32)
                        a.logits_out[(size_t)r * a.n_subset_max + t0 + p] = e.tile[r * kTile + p];
            }
            if (last_t && !par) break;   // folded by all warps after the loop
        }
        if (par) {
            // middle tile: the epilogue warps (barrier 1); last tile: all warps (barrier 2)
            const int ftid = last_t ? (int)threadIdx.x : ew * 32 + lane;
            const int fn = last_t ? kTcWarps * 32 : nthr;
            const int bar = last_t ? 2 : 1;
            if (last_t) named_bar_sync(2, fn);
            if (DTR && last_t && warp == kTcEpiWarp0 && lane == 0) DTR[43] = clock64();
            epi_par_phase1_any(e, n_h, a.KP, tn, t0, ftid, fn, last_t, a.part, pcta, a.n_h, h_row0, a.LS,
                               DTR && last_t && warp == kTcEpiWarp0 ? DTR + 50 : nullptr);
            if (DTR && last_t && warp == kTcEpiWarp0 && lane == 0) DTR[44] = clock64();
            if (DTR && last_t && lane == 0) DTR[20 + warp] = clock64();   // (each warp's phase-1 end)
            named_bar_sync(bar, fn);
            epi_par_phase2(e, n_h, a.KP, tn, t0, ftid, fn, bar, last_t, a.part, pcta, a.n_h, h_row0, a.LS,
                           a.trace ? a.trace + kTraceOvf + (last_t ? 0 : kNumSMs) + blockIdx.x : nullptr);
            if (DTR && last_t && warp == kTcEpiWarp0 && lane == 0) DTR[46] = clock64();
            if (warp == kTcEpiWarp0 && lane == 0 && t < 2) TC_TRACE(4 + 2 * t);
            if (last_t) break;
        } else if (buffered) {
            epi_tile_buf(e, n_h, a.KP, tn, t0, ew, kTcEpiWarps, true);
            if (ew == 0 && lane == 0 && t < 2) TC_TRACE(4 + 2 * t);
        } else {
            epi_tile(e, n_h, a.KP, tn, t0, ew, kTcEpiWarps);
            if (ew == 0 && lane == 0 && t < 2) TC_TRACE(4 + 2 * t);
        }
        named_bar_sync(1, nthr);
    }
    if (a.list2) ensure2();
    const int n_tiles = n_tiles1 + nt2;
    const bool store_after = a.list2 && nt2 == 0 && !par;   // (two-list mode, no second-list tile)
    if (n_tiles > 0 && !store_after && !par) {
        // the last tile without the thread-parallel fold (single-tile CTAs, sorted lists):
        // all 13 warps split its rows
        int t0, tn;
        tile_range(n_tiles - 1, t0, tn);
        named_bar_sync(2, kTcWarps * 32);
        if (buffered) {
            epi_tile_buf_last_store(e, a.part, pcta, a.n_h, h_row0, n_h, a.KP, a.LS, tn, t0, warp, kTcWarps,
                                    warp == kTcEpiWarp0 ? DTR : nullptr);
        } else {
            epi_tile_last(e, a.part, pcta, a.n_h, h_row0, n_h, a.KP, a.LS, tn, t0, warp, kTcWarps);
        }
        if (warp == kTcEpiWarp0 && lane == 0 && n_tiles - 1 < 2) TC_TRACE(4 + 2 * (n_tiles - 1));
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (buffered) {
        if (n_tiles == 0 || store_after) epi_store_buf(e, a.part, pcta, a.n_h, h_row0, n_h, warp, kTcWarps, a.LS);
        // (otherwise the last tile's fold stored every row)
    } else {
        epi_store(e, a.part, pcta, a.n_h, h_row0, n_h, a.KP, a.LS, warp, kTcWarps);
    }
    if (threadIdx.x == 0) TC_TRACE(7);
    if (warp == kTcMmaWarp)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(tp.tmem_cols));
}

// ------------------------------------------------------------------ host
int lmh_tc_grid() { return kNumSMs; }
static int lmh_tc_grid(const LmhArgs& a) { return a.grid > 0 ? a.grid : kNumSMs; }

bool lmh_tc_supported(const LmhArgs& a) {
    const int rows = a.nseg > 0 ? a.seg_rows : a.n_h;
    return a.w_dtype == 0 && a.h_dtype == 0 && a.d % kBlockK == 0 && rows >= 1 && rows <= kTcMaxRows &&
           a.n_w_rows <= 0x7fffffff && (a.nseg == 0 || (a.nseg <= lmh_tc_grid() && a.KP <= 32));
}

cudaError_t launch_lmh_tc(const LmhArgs& a, cudaStream_t st) {
    TcParams tp{};
    const int rows = a.nseg > 0 ? a.seg_rows : a.n_h;
    tp.n_pad = ((rows + 15) / 16) * 16;
    tp.nkb = a.d / kBlockK;
    tp.last_tile = kLastTile;
    tp.dyn_tile = 112;   // (second-list tile rows: 4,096 dynamic rows on 37 CTAs; step 245.6 -> 244.9 us vs 128)
    tp.dyn_stride = 1;   // (scattering the second-list CTAs over the chip measured equal)
    // half a share (llama draft step: those CTAs stream one first-list tile, the others
    // two; measured r2 with the step timeline: 16/16 277.5 us, 12 282.0, 8 264.8, 6 286.7,
    // 4 286.4 -- below 8 the other CTAs' ranges grow a third tile)
    tp.dyn_share = 8;
    if (const char* e = getenv("EVOSPEC_DYN_TILE")) tp.dyn_tile = atoi(e) <= 0 ? 0 : std::max(16, std::min(kTileM, atoi(e)));
    uint32_t cols = 2 * tp.n_pad, c = 32;
    while (c < cols) c <<= 1;
    tp.tmem_cols = c;
    const size_t stage_a = (size_t)kTileM * 128, stage_b = (size_t)tp.n_pad * 128;
    const size_t epi = epi_smem_bytes(rows, (a.KP <= 32 && a.LS >= kBuf) ? kBuf : a.KP, kTcWarps);
    const size_t fixed = epi + 2 * 128 * 4 + 64 * 8 + 1024 /*align slack*/ + 256;
    const size_t budget = 227 * 1024;
    int S = (int)((budget - fixed) / (stage_a + stage_b));
    S = std::min(S, 8);
    if (const char* e = getenv("EVOSPEC_TC_SMAX")) S = std::max(2, std::min(S, atoi(e)));   // (experiment)
    if (S < 2) return cudaErrorInvalidConfiguration;
    tp.stages = S;
    tp.off_b = (size_t)S * stage_a;
    tp.off_epi = tp.off_b + (size_t)S * stage_b;
    tp.off_bar = (tp.off_epi + epi + 15) & ~(size_t)15;
    tp.off_rows = tp.off_bar + (size_t)(2 * S + 4) * 8 + 16;
    const size_t smem = tp.off_rows + 2 * 128 * 4 + 1024;
    CUtensorMap mw{}, mh;   // W rows are gathered by cp.async: no W map is needed
    if (!cached_map(&mh, a.H, (uint64_t)a.d, (uint64_t)a.n_h, kBlockK, (uint32_t)tp.n_pad,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B))
        return cudaErrorInvalidValue;
    cudaError_t e = ensure_smem(lmh_tc_kernel, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(lmh_tc_kernel, dim3(lmh_tc_grid(a)), dim3(kTcWarps * 32), smem, st, mw, mh, a, tp);
}

}  // namespace es
