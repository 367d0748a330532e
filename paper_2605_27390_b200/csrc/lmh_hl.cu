// lmh_hl.cu -- a5-a7 (gathered LM head, online softmax, per-CTA top-k lists) on
// the 5th-generation tensor cores with the draft-tree rows on the TMEM lanes:
//
//   z[r][j] = inv_temp * sum_c H[r][c] W[S_j][c]     (Eq. projection P:44-48,
//                                                     restricted to V_t)
//
// MMA orientation: A = H (M = 128: rows 0..n_h-1 are the tree rows, n_h <= 64;
// lanes 64..127 compute on whatever follows the H block in shared memory and are
// never read), B = the gathered W rows of one tile (N = tile rows padded to 16,
// <= 256), both K-major with the 128-byte swizzle; the fp32 accumulator D[128 x N]
// sits in TMEM with H row r on lane r, double-buffered (2 x 256 columns).
// An epilogue thread therefore owns one H row's logits of 64 consecutive
// subset positions: the online softmax and the top-k candidates need no
// shuffles and no shared-memory tile.
//
// Tiles: each CTA owns a contiguous share of the subset positions, split into
// <= 256-row tiles; H is streamed once per tile (per CTA at n_S <= 256 * 148).
// A ring slot holds one or more K-blocks (64 columns) of H and of the tile's W
// rows: short tiles pack several K-blocks per slot, so the bytes in flight per
// SM stay the same when a tile is mostly H.
//
// Warp roles (14 warps; a warp reads the TMEM lanes 32 (w % 4) .. + 31):
//   w % 4 in {0, 1}  (0,1,4,5,8,9,12,13)  epilogue: quadrant w % 4 (rows), column
//                    quarter w / 4 of the 256-column accumulator
//   2, 3, 6, 7       W producers: 16-byte cp.async into the swizzled slot, one
//                    cp.async.mbarrier.arrive.noinc per thread and slot
//   10               TMEM allocation + MMA issue (one thread)
//   11               H by 2D TMA (one K-block box per K-block of a slot)
//
// Epilogue per tile and row (4 threads x 64 columns):
//   - softmax: the row maximum over the 4 threads (shared memory), then the
//     thread's sum of 2^((z - m) log2 e) and the rescaled running sum;
//   - candidates: a lower bound B of the row's KP-th best in this tile (KP =
//     k + 8: the KP-th largest of the 32 or 64 group maxima -- at least KP
//     distinct entries are >= B), values >= B (and > the running bound of
//     earlier tiles) are appended to the row's buffer (<= 64 entries); a row
//     that would overflow takes an exact KP-th-value search by bisection on the
//     monotone float key (rare: massive ties);
//   - between tiles a buffer above KP entries is cut to its exact top KP
//     (ranks by counting) and its KP-th entry becomes the running bound; after
//     the last tile the buffer's exact top KP are written sorted to the CTA's
//     partial list (stride kHlLS), with the row's (m, s) -- the finalisation
//     (finalize32.cuh, sorted-list mode) merges the CTAs' lists.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace es {

constexpr int kHlWarps = 14;
constexpr int kHlThreads = kHlWarps * 32;
constexpr int kHlMmaWarp = 10;
constexpr int kHlTmaWarp = 11;
constexpr int kHlEpiThreads = 256;
constexpr int kHlRows = 64;          // H rows (TMEM lanes 0..63)
constexpr int kHlTile = 256;         // W rows per tile (MMA N <= 256)
constexpr int kHlCap = 64;           // candidate buffer per row
constexpr int kHlCapS = kHlCap + 1;  // its row stride (conflict-free column reads)
constexpr int kHlGS = 65;            // group-maxima row stride (conflict-free scalar access across rows)
constexpr int kHlHBytes = kHlRows * 128;   // H K-block: 64 rows x 128 B
constexpr int kHlMaxSlots = 16;
constexpr int kHlRB = (kHlRows + kHlWarps - 1) / kHlWarps;   // rows per warp in the last-tile phase (5)
constexpr int kHlZS = 260;           // staged last-tile logits: row stride (16-byte rows, conflict-free float4)
constexpr int kHlBar = 1;            // named barrier of the 256 epilogue threads
constexpr float kL2E = 1.4426950408889634f;

ES_DEV float ex2f(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
ES_DEV float key_to_float(uint32_t k) { return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k); }
// 16 floats sorted descending in registers (bitonic network, branch-free)
ES_DEV void bitonic_desc16(float (&v)[16]) {
#pragma unroll
    for (int k = 2; k <= 16; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const float a = v[i], b = v[l];
                    const bool desc = (i & k) == 0;
                    v[i] = desc ? fmaxf(a, b) : fminf(a, b);
                    v[l] = desc ? fminf(a, b) : fmaxf(a, b);
                }
            }
}
// 32 floats sorted descending in registers (bitonic network, branch-free)
ES_DEV void bitonic_desc32(float (&v)[32]) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const float a = v[i], b = v[l];
                    const bool desc = (i & k) == 0;
                    v[i] = desc ? fmaxf(a, b) : fminf(a, b);
                    v[l] = desc ? fminf(a, b) : fmaxf(a, b);
                }
            }
}
ES_DEV void hl_bar() { named_bar_sync(kHlBar, kHlEpiThreads); }
// per-CTA globaltimer stamps (EVOSPEC_TRACE; profiling aid): [cta][8]
#define HL_TRACE(slot) do { if (a.trace) a.trace[(size_t)blockIdx.x * 8 + (slot)] = gtime(); } while (0)
// clock64 stamps of CTA 0, warp 0, lane 0 (epilogue steps of each tile, last tile wins)
#define HL_G0(i) do { if (a.trace && blockIdx.x == 0) a.trace[2 * 148 * 8 + 48 + 16 + (i)] = gtime(); } while (0)
#define HL_CLK(i) do { if (a.trace && blockIdx.x == 0 && warp == 0 && lane == 0) a.trace[2 * 148 * 8 + 48 + (i)] = clock64(); } while (0)

// 64 consecutive accumulator columns of this warp's 32 lanes (two x32 loads and
// the wait in one asm statement, so no use of the registers precedes the wait)
ES_DEV void tmem_ld64(uint32_t taddr, float (&v)[64]) {
    uint32_t r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%64];\n"
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%65];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
          "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
          "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
          "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
          "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr), "r"(taddr + 32u)
        : "memory");
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 consecutive accumulator columns of this warp's 32 lanes (load and wait in one
// asm statement, so no use of the registers precedes the wait)
ES_DEV void tmem_ld16w(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// chunks at taddr a and b (16 columns each) into v[0..15], v[16..31], one wait
ES_DEV void tmem_ld16x2w(uint32_t ta, uint32_t tb, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n"
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(ta), "r"(tb)
        : "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Column of element j (0..63) of epilogue thread cq: the thread's 4 chunks of 16
// interleave with the other threads' (64 c + 16 cq), so every thread holds about
// tn / 4 valid columns whatever the tile length
ES_DEV int hl_col(int cq, int j) { return 64 * (j >> 4) + 16 * cq + (j & 15); }
ES_DEV void hl_load64(uint32_t taddr0, int cq, float (&z)[64]) {
    float t[16];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        tmem_ld16w(taddr0 + 64 * c + 16 * cq, t);
#pragma unroll
        for (int j = 0; j < 16; ++j) z[16 * c + j] = t[j];
    }
}

// Overflow of a row's candidate buffer (rare: massive ties): the exact KP-th value
// T of the candidates (this tile's admitted values + the buffer) by bisection on
// the monotone float key, then the buffer := the KP best (ties by position: the
// buffer's entries, then the columns in order). Executed by all 256 epilogue
// threads (named barriers); rows without overflow (ov false) only take the
// barriers. The logits are re-read from TMEM (the accumulator is still held).
__device__ __noinline__ void hl_overflow(uint32_t taddr0, bool rv, bool ov, int tn, float inv_temp, float B,
                                         float Br, int KP, int n_old, int t0, int r, int cq, float* bv, int* bp,
                                         int* t_c, int* t_x, int* st_n, float* b_run) {
    float z[64];
    hl_load64(taddr0, cq, z);
#pragma unroll
    for (int j = 0; j < 64; ++j) z[j] = (rv && hl_col(cq, j) < tn) ? z[j] * inv_temp : -INFINITY;
    uint32_t mlo = 0u, mhi = 0u;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        mlo |= (uint32_t)(z[j] >= B && z[j] > Br) << j;
        mhi |= (uint32_t)(z[32 + j] >= B && z[32 + j] > Br) << j;
    }
    uint32_t lo = 0u, hi = 0xffffffffu;
#pragma unroll 1
    for (int it = 0; it < 32; ++it) {
        int* tcx = t_c + ((it + 1) & 1) * kHlRows * 4;
        const uint32_t mid = lo + (uint32_t)(((uint64_t)hi - lo + 1) >> 1);
        int c = 0;
        if (ov && lo < hi) {
#pragma unroll
            for (int j = 0; j < 64; ++j) c += ((((j < 32 ? mlo : mhi) >> (j & 31)) & 1u) && float_key(z[j]) >= mid);
            if (cq == 0)
                for (int i = 0; i < n_old; ++i) c += float_key(bv[i]) >= mid;
        }
        tcx[r * 4 + cq] = c;
        hl_bar();
        if (ov && lo < hi) {
            const int4 v = *(const int4*)&tcx[r * 4];
            if (v.x + v.y + v.z + v.w >= KP) lo = mid;
            else hi = mid - 1;
        }
    }
    const uint32_t T = lo;
    int gt = 0, eq = 0, bgt = 0, beq = 0;
    if (ov) {
#pragma unroll
        for (int j = 0; j < 64; ++j) {
            if ((((j < 32 ? mlo : mhi) >> (j & 31)) & 1u)) {
                const uint32_t k = float_key(z[j]);
                gt += k > T;
                eq += k == T;
            }
        }
        if (cq == 0)
            for (int i = 0; i < n_old; ++i) {
                const uint32_t k = float_key(bv[i]);
                bgt += k > T;
                beq += k == T;
            }
    }
    hl_bar();   // (the bisection's last reads of t_c precede its reuse)
    t_c[r * 4 + cq] = gt + bgt;
    t_c[kHlRows * 4 + r * 4 + cq] = eq + beq;
    hl_bar();
    int take = 0, sel = 0;
    if (ov) {
        const int4 g4v = *(const int4*)&t_c[r * 4];
        const int4 e4v = *(const int4*)&t_c[kHlRows * 4 + r * 4];
        const int need = KP - (g4v.x + g4v.y + g4v.z + g4v.w);
        const int pre_eq = (cq > 0 ? e4v.x : 0) + (cq > 1 ? e4v.y : 0) + (cq > 2 ? e4v.z : 0);
        take = min(max(need - pre_eq, 0), eq + beq);
        if (cq == 0) {   // the buffer, compacted in place (its ties first)
            int nb = 0;
            for (int i = 0; i < n_old; ++i) {
                const uint32_t k = float_key(bv[i]);
                if (k > T || (k == T && take > 0)) {
                    if (k == T) --take;
                    bv[nb] = bv[i];
                    bp[nb] = bp[i];
                    ++nb;
                }
            }
            st_n[r] = nb;
        }
        sel = gt + min(take, eq);
    }
    t_x[kHlRows * 4 + r * 4 + cq] = sel;
    hl_bar();
    if (ov) {
        const int4 sx = *(const int4*)&t_x[kHlRows * 4 + r * 4];
        int o = st_n[r] + (cq > 0 ? sx.x : 0) + (cq > 1 ? sx.y : 0) + (cq > 2 ? sx.z : 0);
#pragma unroll
        for (int j = 0; j < 64; ++j) {
            if ((((j < 32 ? mlo : mhi) >> (j & 31)) & 1u)) {
                const uint32_t k = float_key(z[j]);
                if (k > T || (k == T && take > 0)) {
                    if (k == T) --take;
                    bv[o] = z[j];
                    bp[o] = t0 + hl_col(cq, j);
                    ++o;
                }
            }
        }
    }
    hl_bar();
    if (ov && cq == 0) {
        st_n[r] = KP;
        b_run[r] = key_to_float(T);
    }
}

// debug output of this thread's 64 logits (re-read from TMEM)
__device__ __noinline__ void hl_logits_out(uint32_t taddr0, int tn, int cq, float inv_temp, float* out) {
    float z[64];
    hl_load64(taddr0, cq, z);
#pragma unroll
    for (int j = 0; j < 64; ++j)
        if (hl_col(cq, j) < tn) out[hl_col(cq, j)] = z[j] * inv_temp;
}

// Exact warp-level selection of a row's best KP when the candidates overflow its
// buffer (rare: massive ties). Candidates: the buffer's [0, n_old) (earlier tiles:
// smaller positions) and this tile's values >= B and > Br (the staged row zrow,
// column lane + 32 j).
// T = the KP-th largest key by bisection on the monotone float key (warp sums); the
// selection: every key > T, then the ties in position order (the buffer's by their
// positions, then the tile's by column). Writes KP entries to rbv / rbp [0, KP).
__device__ __noinline__ void hl_warp_select(const float* zrow, float B, float Br, float* rbv, int* rbp, int n_old,
                                            int t0, int KP, int lane) {
    float v[8];
    uint32_t bal[8];
    for (int j = 0; j < 8; ++j) {
        v[j] = zrow[lane + 32 * j];
        bal[j] = __ballot_sync(0xffffffffu, v[j] >= B && v[j] > Br);
    }
    const bool hb0 = lane < n_old, hb1 = lane + 32 < n_old;
    const float bv0 = hb0 ? rbv[lane] : -INFINITY, bv1 = hb1 ? rbv[lane + 32] : -INFINITY;
    const int bp0 = hb0 ? rbp[lane] : INT_MAX, bp1 = hb1 ? rbp[lane + 32] : INT_MAX;
    const uint32_t kb0 = float_key(bv0), kb1 = float_key(bv1);
    uint32_t kt[8];
    bool ht[8];
    for (int j = 0; j < 8; ++j) { ht[j] = (bal[j] >> lane) & 1u; kt[j] = float_key(v[j]); }
    uint32_t lo = 0u, hi = 0xffffffffu;
    while (lo < hi) {   // (uniform: the counts are warp sums)
        const uint32_t mid = lo + (uint32_t)(((uint64_t)hi - lo + 1) >> 1);
        int c = (hb0 && kb0 >= mid) + (hb1 && kb1 >= mid);
        for (int j = 0; j < 8; ++j) c += ht[j] && kt[j] >= mid;
        if (warp_sum_i(c) >= KP) lo = mid;
        else hi = mid - 1;
    }
    const uint32_t T = lo;
    int gt = (hb0 && kb0 > T) + (hb1 && kb1 > T);
    for (int j = 0; j < 8; ++j) gt += ht[j] && kt[j] > T;
    const int need = KP - warp_sum_i(gt);
    // ties of the buffer, ranked by position among themselves
    const bool tb0 = hb0 && kb0 == T, tb1 = hb1 && kb1 == T;
    int rb0 = 0, rb1 = 0;
    for (int w = 0; w < 2; ++w)
        for (int l = 0; l < 32; ++l) {
            const bool ts = __shfl_sync(0xffffffffu, w ? tb1 : tb0, l);
            const int ps = __shfl_sync(0xffffffffu, w ? bp1 : bp0, l);
            rb0 += ts && ps < bp0;
            rb1 += ts && ps < bp1;
        }
    const int nbt = warp_sum_i(tb0 + tb1);
    const uint32_t lt = (1u << lane) - 1u;
    bool sel[10];
    sel[0] = hb0 && (kb0 > T || (tb0 && rb0 < need));
    sel[1] = hb1 && (kb1 > T || (tb1 && rb1 < need));
    int tpre = 0;
    for (int j = 0; j < 8; ++j) {
        const uint32_t tt = __ballot_sync(0xffffffffu, ht[j] && kt[j] == T);
        const bool tie = (tt >> lane) & 1u;
        sel[2 + j] = ht[j] && (kt[j] > T || (tie && nbt + tpre + __popc(tt & lt) < need));
        tpre += __popc(tt);
    }
    __syncwarp();   // (every lane read its buffer entries above)
    int pos = 0;
    for (int q = 0; q < 10; ++q) {
        const uint32_t sb = __ballot_sync(0xffffffffu, sel[q]);
        if (sel[q]) {
            const int sl = pos + __popc(sb & lt);
            rbv[sl] = q == 0 ? bv0 : q == 1 ? bv1 : v[q - 2];
            rbp[sl] = q == 0 ? bp0 : q == 1 ? bp1 : t0 + lane + 32 * (q - 2);
        }
        pos += __popc(sb);
    }
    __syncwarp();
}

struct HlParams {
    int slot_bytes;   // ring slot (multiple of 1024): one K-block of H + W rows of the largest tile
    int slots;
    int nkb;          // d / 64
    int bh;           // H rows per TMA box (n_h padded to 8)
    int off_epi, off_bar;
};

// epilogue shared memory (floats / ints)
__host__ __device__ constexpr int hl_epi_bytes() {
    return 4 * (2 * kHlRows * kHlCapS      // buf_v, buf_p
                + kHlRows * kHlGS          // gmax
                + 6 * kHlRows * 4          // t_m, t_s, t_c[2], t_x[2]
                + 6 * kHlRows + 8);        // st_m, st_s, st_n, ctr, b_run, ovf, flag, last tile
}

__global__ void __launch_bounds__(kHlThreads, 1)
lmh_hl_kernel(const __grid_constant__ CUtensorMap tmap_h, LmhArgs a, HlParams hp) {
    extern __shared__ __align__(1024) unsigned char hl_sm[];
    unsigned char* base = hl_sm + ((1024u - (smem_u32(hl_sm) & 1023u)) & 1023u);   // shared-window pointer
    const int S = hp.slots;
    uint64_t* full = (uint64_t*)(base + hp.off_bar);
    uint64_t* empty = full + S;
    uint64_t* tfull = empty + S;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);
    float* buf_v = (float*)(base + hp.off_epi);            // [64][kHlCapS]
    int* buf_p = (int*)(buf_v + kHlRows * kHlCapS);        // [64][kHlCapS] (virtual) subset positions
    float* gmax = (float*)(buf_p + kHlRows * kHlCapS);     // [64][kHlGS]
    float* t_m = gmax + kHlRows * kHlGS;                   // [64][4] per-thread tile maxima
    float* t_s = t_m + kHlRows * 4;                        // [64][4] per-thread exp sums
    int* t_c = (int*)(t_s + kHlRows * 4);                  // [2][64][4] counts
    int* t_x = t_c + 2 * kHlRows * 4;                      // [2][64][4] counts
    float* st_m = (float*)(t_x + 2 * kHlRows * 4);         // running row maximum
    float* st_s = st_m + kHlRows;                          // running sum of e^(z - st_m)
    int* st_n = (int*)(st_s + kHlRows);                    // buffer fill
    int* ctr = st_n + kHlRows;                             // this tile's append counter
    float* b_run = (float*)(ctr + kHlRows);                // running bound (strict)
    int* ovf = (int*)(b_run + kHlRows);                    // row overflow
    int* any_ovf = ovf + kHlRows;
    int* fin_tile = any_ovf + 1;                           // [3] the last tile's t0, tn, positions seen

    const int warp = warp_id(), lane = lane_id();
    pdl_trigger();
    if (threadIdx.x == 0) HL_TRACE(0);
    if (threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap_h) : "memory");
        for (int s = 0; s < S; ++s) { mbar_init(&full[s], 4 * 32 + 1); mbar_init(&empty[s], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kHlMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(2 * kHlTile));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    if (threadIdx.x == 0) HL_G0(0);

    // ---- the CTA's tile schedule (every role evaluates it identically)
    // one-list mode: the subset (and n_S) come from the previous kernel. Two-list
    // mode (draft_step overlap): the first list is an input, streamed before
    // griddepcontrol.wait; the second list's share is resolved lazily after it.
    const bool two = a.list2 != nullptr;
    if (!two) pdl_wait();
    if (threadIdx.x == 0) HL_G0(1);
    const int G = gridDim.x, bid = blockIdx.x;
    int p0, p1;
    if (two) {
        p0 = (int)((long long)a.n1 * bid / G);
        p1 = (int)((long long)a.n1 * (bid + 1) / G);
    } else {
        lmh_cta_range(a, p0, p1);
    }
    const int len1 = p1 - p0;
    const int nt1 = (len1 + kHlTile - 1) / kHlTile;
    int nt2 = two ? -1 : 0, q0 = 0, len2 = 0;
    auto ensure2 = [&]() {
        if (nt2 >= 0) return;
        pdl_wait();
        const int n2 = max(0, min(*(volatile const int*)a.n_list2_dev, a.n_list2_max));
        q0 = (int)((long long)n2 * bid / G);
        len2 = (int)((long long)n2 * (bid + 1) / G) - q0;
        nt2 = (len2 + kHlTile - 1) / kHlTile;
    };
    auto has_tile = [&](int t) -> bool {
        if (t < nt1) return true;
        if (!two) return false;
        ensure2();
        return t < nt1 + nt2;
    };
    auto tile_range = [&](int t, int& t0, int& tn) {
        if (t < nt1) {
            t0 = p0 + (int)((long long)len1 * t / nt1);
            tn = p0 + (int)((long long)len1 * (t + 1) / nt1) - t0;
        } else {
            const int u = t - nt1;
            t0 = a.n1 + q0 + (int)((long long)len2 * u / nt2);
            tn = a.n1 + q0 + (int)((long long)len2 * (u + 1) / nt2) - t0;
        }
    };
    // K-blocks per slot for a tile of tn rows (unit: H block + the tile's W rows)
    // (the producer copies whole 16-row groups: rows past the tile end repeat its last row)
    auto tile_unit = [&](int tn) { return kHlHBytes + ((tn + 15) >> 4) * 2048; };
    auto tile_kps = [&](int tn) { return max(1, min(hp.nkb, hp.slot_bytes / tile_unit(tn))); };

    if ((warp & 3) >= 2 && warp < 8) {
        // ===== W producers: thread (pw, lane) copies chunk lane & 7 of the tile rows
        // 16 i + 4 pw + (lane >> 3): one warp instruction moves 4 whole 128-byte rows
        const int pw = ((warp >> 2) << 1) | (warp & 1);
        const uint64_t pol_w = policy_evict_first();   // W is read once: keep L2 for H and the lists
        const int chunk = lane & 7, rsub = 4 * pw + (lane >> 3);
        const size_t row_bytes = (size_t)a.d * 2;
        int stage = 0;
        uint32_t phase = 0;
        for (int t = 0; has_tile(t); ++t) {
            int t0, tn;
            tile_range(t, t0, tn);
            const int unit = tile_unit(tn), kps = tile_kps(tn);
            // row groups of 16 (warp-uniform count); rows past the tile's end re-copy its
            // last row into smem rows whose accumulator columns are masked
            const int ng = (tn + 15) >> 4;
            const char* src[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const int row = min(16 * i + rsub, tn - 1);
                src[i] = (const char*)a.W + (size_t)(lmh_id_at(a, t0 + row) / a.R) * row_bytes + chunk * 16;
            }
            const uint32_t doff = kHlHBytes + rsub * 128 + ((chunk ^ (rsub & 7)) << 4);   // row 16 i + rsub: + 2048 i
            for (int kb0 = 0; kb0 < hp.nkb; kb0 += kps) {
                mbar_wait(&empty[stage], phase ^ 1);
                const uint32_t sb = smem_u32(base + (size_t)stage * hp.slot_bytes) + doff;
                const int nk = min(kps, hp.nkb - kb0);
                for (int j = 0; j < nk; ++j) {
                    const uint32_t dW = sb + j * unit;
                    const int ko = (kb0 + j) * 128;
                    if (ng == 16) {   // full 256-row tile: no predicates in the issue stream
#pragma unroll
                        for (int i = 0; i < 16; ++i) cp_async16(dW + i * 2048, src[i] + ko, pol_w);
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i)
                            if (i < ng) cp_async16(dW + i * 2048, src[i] + ko, pol_w);
                    }
                }
                if (warp == 2 && lane == 0 && t == 0 && (kb0 == 0 || kb0 == 8 || kb0 == 32)) HL_G0(2 + (kb0 == 8) + 2 * (kb0 == 32));
                cp_async_arrive_noinc(&full[stage]);
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
        }
        if (warp == 2 && lane == 0) HL_TRACE(1);
    } else if (warp == kHlTmaWarp) {
        // ===== H: one 2D TMA box (64 columns x bh rows, rows >= n_h zero-filled) per K-block
        if (lane == 0) {
            const uint64_t pol_h = policy_evict_last();
            int stage = 0;
            uint32_t phase = 0;
            for (int t = 0; has_tile(t); ++t) {
                int t0, tn;
                tile_range(t, t0, tn);
                const int unit = tile_unit(tn), kps = tile_kps(tn);
                for (int kb0 = 0; kb0 < hp.nkb; kb0 += kps) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    const int nk = min(kps, hp.nkb - kb0);
                    mbar_arrive_expect_tx(&full[stage], (uint32_t)(nk * hp.bh * 128));
                    unsigned char* sb = base + (size_t)stage * hp.slot_bytes;
                    for (int j = 0; j < nk; ++j) tma_load_2d(sb + j * unit, &tmap_h, &full[stage], (kb0 + j) * 64, 0, pol_h);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == kHlMmaWarp) {
        // ===== MMA issuer: 4 x tcgen05.mma (K = 16) per K-block, commit per slot
        int stage = 0;
        uint32_t phase = 0;
        for (int t = 0; has_tile(t); ++t) {
            int t0, tn;
            tile_range(t, t0, tn);
            const int unit = tile_unit(tn), kps = tile_kps(tn);
            const uint32_t idesc = idesc_bf16(128, (tn + 15) & ~15);
            const int b = t & 1;
            if (t >= 2) mbar_wait(&tempty[b], (uint32_t)((t >> 1) - 1) & 1);
            tc_fence_after();
            const uint32_t tmem_d = tmem_base + (uint32_t)(b * kHlTile);
            for (int kb0 = 0; kb0 < hp.nkb; kb0 += kps) {
                mbar_wait(&full[stage], phase);
                if (lane == 0 && t == 0 && (kb0 == 0 || kb0 == 8 || kb0 == 32)) HL_G0(5 + (kb0 == 8) + 2 * (kb0 == 32));
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t sb = smem_u32(base + (size_t)stage * hp.slot_bytes);
                    const int nk = min(kps, hp.nkb - kb0);
                    for (int j = 0; j < nk; ++j) {
                        const uint32_t aa = sb + j * unit, ba = aa + kHlHBytes;
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            umma_bf16(tmem_d, umma_desc_sw128(aa + k * 32), umma_desc_sw128(ba + k * 32), idesc,
                                      (uint32_t)((kb0 + j) | k));
                    }
                    umma_commit(&empty[stage]);
                    if (kb0 + kps >= hp.nkb) umma_commit(&tfull[b]);
                }
                __syncwarp();
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
        }
        if (lane == 0) HL_TRACE(2);
    } else if ((warp & 3) < 2) {
        // ===== epilogue: row r = 32 (w % 4) + lane, columns [64 cq, 64 cq + 64) of the tile.
        // The code runs once per tile, so it is paid for by its footprint (instruction
        // fetch), not its issue count: every pass is a rolled loop over 4 chunks of 16
        // columns re-read from TMEM (tcgen05.ld 32x32b.x16), nothing is unrolled 64-wide.
        const int qd = warp & 3, cq = warp >> 2;
        const int r = 32 * qd + lane;
        const bool rv = r < a.n_h;
        const int KP = a.KP;
        float* bv = buf_v + r * kHlCapS;
        int* bp = buf_p + r * kHlCapS;
        float* gr = gmax + r * kHlGS;
        if (cq == 0) {
            st_m[r] = -INFINITY; st_s[r] = 0.0f; st_n[r] = 0; b_run[r] = -INFINITY; ovf[r] = 0;
            if (r == 0) *any_ovf = 0;
        }
        hl_bar();
        int seen = 0;   // subset positions of this CTA so far (entries beyond the list were dropped)
        int t;
        // (`dry`: a dry run of the tile epilogue on the idle accumulator before tile 0,
        // to warm the instruction cache, was measured without gain and removed; the
        // side-effect masks it needed remain as constants)
        for (t = 0; has_tile(t); ++t) {
            constexpr bool dry = false;
            int t0 = 0, tn = kHlTile;
            if (!dry) {
                tile_range(t, t0, tn);
                seen += tn;
            }
            const int b = dry ? 1 : (t & 1);
            // (two-list mode: resolving the next tile may wait for the union here)
            const bool last = !dry && !has_tile(t + 1);
            if (!dry) {
                mbar_wait_sleep(&tfull[b], (uint32_t)(t >> 1) & 1, 200);
                if (warp == 0 && lane == 0) HL_TRACE(t == 0 ? 3 : 5);
                HL_CLK(0);
            }
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(32 * qd) << 16) + (uint32_t)(b * kHlTile);
            const float it = a.inv_temp;
            if (last) {
                // the CTA's last tile: its logits go to shared memory (the ring is idle
                // now) and all 14 warps finish its rows below, one warp per row
                float z[64];
                hl_load64(taddr, cq, z);
                float* zr = (float*)base + r * kHlZS;
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        float4 w;
                        const int col = 64 * c + 16 * cq + 4 * q;
                        w.x = (rv && col + 0 < tn) ? z[16 * c + 4 * q + 0] * it : -INFINITY;
                        w.y = (rv && col + 1 < tn) ? z[16 * c + 4 * q + 1] * it : -INFINITY;
                        w.z = (rv && col + 2 < tn) ? z[16 * c + 4 * q + 2] * it : -INFINITY;
                        w.w = (rv && col + 3 < tn) ? z[16 * c + 4 * q + 3] * it : -INFINITY;
                        *(float4*)&zr[col] = w;
                    }
                if (a.logits_out)   // debug output (out of line: re-read from TMEM; the whole warp loads)
                    hl_logits_out(taddr, rv ? tn : 0, cq, it, a.logits_out + (size_t)(rv ? r : 0) * a.n_subset_max + t0);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&tempty[b]);
                if (warp == 0 && lane == 0) { fin_tile[0] = t0; fin_tile[1] = tn; fin_tile[2] = seen; }
                HL_CLK(1);
                break;
            }
            // ---- pass A: the thread's 64 logits in one TMEM round trip (a load costs ~1000
            // cycles with 8 warps loading, measured), its maximum, exp sum and 16
            // four-column group maxima, of which it publishes the 8 largest (sorted)
            float z[64];
            hl_load64(taddr, cq, z);
#pragma unroll
            for (int j = 0; j < 64; ++j) z[j] = (rv && hl_col(cq, j) < tn) ? z[j] * it : -INFINITY;
            if (!dry) HL_CLK(10);
            float g[16];
#pragma unroll
            for (int u = 0; u < 16; ++u)
                g[u] = fmaxf(fmaxf(z[4 * u], z[4 * u + 1]), fmaxf(z[4 * u + 2], z[4 * u + 3]));
            float tm = g[0];
#pragma unroll
            for (int u = 1; u < 16; ++u) tm = fmaxf(tm, g[u]);
            float ts = 0.0f;
            if (tm != -INFINITY) {
                const float mb = tm * kL2E;
                float e0 = 0.0f, e1 = 0.0f, e2 = 0.0f, e3 = 0.0f;
#pragma unroll
                for (int j = 0; j < 64; j += 4) {
                    e0 += ex2f(fmaf(z[j], kL2E, -mb));
                    e1 += ex2f(fmaf(z[j + 1], kL2E, -mb));
                    e2 += ex2f(fmaf(z[j + 2], kL2E, -mb));
                    e3 += ex2f(fmaf(z[j + 3], kL2E, -mb));
                }
                ts = (e0 + e1) + (e2 + e3);
            }
            if (!dry) HL_CLK(12);
            bitonic_desc16(g);
            if (!dry) HL_CLK(13);
#pragma unroll
            for (int u = 0; u < 8; ++u) gr[8 * cq + u] = g[u];
            if (cq == 0) gr[32] = -INFINITY;   // run-end sentinel of the merge below
            t_m[r * 4 + cq] = tm;
            t_s[r * 4 + cq] = ts;
            if (cq == 0) ctr[r] = st_n[r];   // the append counter
            HL_CLK(1);
            hl_bar();
            HL_CLK(2);
            const int n_old = st_n[r];
            // bound B: the KP-th largest of the 32 published group maxima (distinct groups:
            // at least KP values are >= B, so nothing below B is in the row's best KP),
            // by a KP-step merge of the 4 sorted runs (every thread of the row, no barrier)
            float B = -INFINITY;
            if (rv && n_old + tn > kHlCap) {
                // branch-free: the rows of a warp pop different runs; the run ends are
                // -inf sentinels (gr[32])
                int i0 = 0, i1 = 8, i2 = 16, i3 = 24;
                float h0 = gr[0], h1 = gr[8], h2 = gr[16], h3 = gr[24];
#pragma unroll 1
                for (int k = 0; k < KP; ++k) {
                    const float m = fmaxf(fmaxf(h0, h1), fmaxf(h2, h3));
                    B = m;
                    const bool s0 = h0 == m, s1 = !s0 && h1 == m, s2 = !s0 && !s1 && h2 == m;
                    const bool s3 = !s0 && !s1 && !s2;
                    const int lim = s0 ? 8 : s1 ? 16 : s2 ? 24 : 32;
                    const int ni = (s0 ? i0 : s1 ? i1 : s2 ? i2 : i3) + 1;
                    const float nv = gr[ni < lim ? ni : 32];
                    i0 = s0 ? ni : i0; h0 = s0 ? nv : h0;
                    i1 = s1 ? ni : i1; h1 = s1 ? nv : h1;
                    i2 = s2 ? ni : i2; h2 = s2 ? nv : h2;
                    i3 = s3 ? ni : i3; h3 = s3 ? nv : h3;
                }
            }
            const float Br = b_run[r];
            HL_CLK(3);
            // ---- pass B: admission (>= B, > the running bound); the row's slots reserved
            // with one shared atomic, values written if they fit (else: overflow)
            uint32_t mlo = 0u, mhi = 0u;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                mlo |= (uint32_t)(z[j] >= B && z[j] > Br) << j;
                mhi |= (uint32_t)(z[32 + j] >= B && z[32 + j] > Br) << j;
            }
            const int na = __popc(mlo) + __popc(mhi);
            if (na) {
                const int ob = atomicAdd(&ctr[r], na);
                if (ob + na <= kHlCap) {
                    const int o1 = ob + __popc(mlo);
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        if ((mlo >> j) & 1u) {
                            const int o = ob + __popc(mlo & ((1u << j) - 1u));
                            bv[o] = z[j];
                            bp[o] = t0 + hl_col(cq, j);
                        }
                        if ((mhi >> j) & 1u) {
                            const int o = o1 + __popc(mhi & ((1u << j) - 1u));
                            bv[o] = z[32 + j];
                            bp[o] = t0 + hl_col(cq, 32 + j);
                        }
                    }
                }
            }
            HL_CLK(6);
            hl_bar();
            const int tot = ctr[r];
            if (!dry && cq == 0 && rv && tot > kHlCap) { ovf[r] = 1; *any_ovf = 1; }
            hl_bar();
            if (a.logits_out && !dry)   // debug output (out of line: re-read from TMEM; the whole warp loads)
                hl_logits_out(taddr, rv ? tn : 0, cq, it, a.logits_out + (size_t)(rv ? r : 0) * a.n_subset_max + t0);
            if (*any_ovf)   // rare (ties): out of line, so the common path keeps its registers
                hl_overflow(taddr, rv, rv && ovf[r], tn, it, B, Br, KP, n_old, t0, r, cq, bv, bp, t_c, t_x,
                            st_n, b_run);
            tc_fence_before();
            __syncwarp();
            if (lane == 0 && !dry) mbar_arrive(&tempty[b]);   // the MMA may reuse this accumulator
            HL_CLK(7);
            // state update (one thread per row): merge the 4 threads' (max, sum), then the running pair
            if (cq == 0 && rv) {
                const float4 mv = *(const float4*)&t_m[r * 4];
                const float4 sv = *(const float4*)&t_s[r * 4];
                const float mt = fmaxf(fmaxf(mv.x, mv.y), fmaxf(mv.z, mv.w));
                auto term = [&](float mm, float ss) { return mm == -INFINITY ? 0.0f : ss * ex2f((mm - mt) * kL2E); };
                const float stile = (term(mv.x, sv.x) + term(mv.y, sv.y)) + (term(mv.z, sv.z) + term(mv.w, sv.w));
                const float mo = st_m[r], mn = fmaxf(mo, mt);
                const float so = mo == -INFINITY ? 0.0f : st_s[r] * ex2f((mo - mn) * kL2E);
                const float sn = mt == -INFINITY ? 0.0f : stile * ex2f((mt - mn) * kL2E);
                if (!dry) {
                    st_s[r] = so + sn;
                    st_m[r] = mn;
                    if (!ovf[r]) st_n[r] = tot;
                    ovf[r] = 0;
                }
            }
            hl_bar();
            if (warp == 0 && lane == 0 && t == 0) HL_TRACE(4);
            if (cq == 0 && r == 0) *any_ovf = 0;   // (every reader passed the barrier above)
            HL_CLK(8);
            const int n = st_n[r];
            if (!dry) {
                // a middle tile: cut the buffer to its exact top KP (ranked into the group-maxima rows,
                // then copied back); its KP-th entry bounds later tiles
                const bool cut = rv && n > KP;
                float* sv = gr;                   // [KP] values
                int* sp = (int*)(gr + 32);        // [KP] positions
                if (cut) {
                    for (int i = cq; i < n; i += 4) {
                        const float v = bv[i];
                        const int p = bp[i];
                        int rank = 0;
                        for (int j = 0; j < n; ++j) rank += before(bv[j], bp[j], v, p);
                        if (rank < KP) { sv[rank] = v; sp[rank] = p; }
                    }
                }
                hl_bar();
                if (cut)
                    for (int i = cq; i < KP; i += 4) { bv[i] = sv[i]; bp[i] = sp[i]; }
                hl_bar();
                if (cut && cq == 0) {
                    st_n[r] = KP;
                    b_run[r] = sv[KP - 1];
                }
            }
        }
    }
    // ===== the CTA's last tile, one warp per row (all 14 warps): its logits are staged
    // in shared memory by the epilogue warps (zs rows of kHlZS floats, -inf outside the
    // tile / the tree rows). Per row: the row maximum and exp sum (warp shuffles) merged
    // with the running pair of earlier tiles; the candidate bound B = the KP-th largest
    // of the 32 lane maxima (warp bitonic sort; >= KP distinct values are >= B); the
    // values >= B (and > the running bound) appended to the row's buffer by ballot
    // prefix; a buffer overflow (ties) takes the exact warp-level selection; the buffer
    // is written out as the CTA's list (unsorted, -inf padded: the finalisation's
    // buffered format cnt = 0, xcnt = n).
    __syncwarp();   // (role branches diverge inside a warp: reconverge before the aligned barrier)
    named_bar_sync(2, kHlThreads);
    HL_CLK(2);
    {
        const int KP = a.KP, LS = a.LS;
        const bool any = has_tile(0);
        const int ft0 = any ? fin_tile[0] : 0, ftn = any ? fin_tile[1] : 0, fseen = any ? fin_tile[2] : 0;
        const float* zs = (const float*)base;
        const int nrep = 1;
        for (int rep = 0; rep < nrep; ++rep) {
        if (rep == nrep - 1) HL_CLK(3);
        const bool wr = rep == nrep - 1;
        for (int rr = warp; rr < a.n_h; rr += kHlWarps) {
            const size_t o = (size_t)bid * a.n_h + rr;
            float* rbv = buf_v + rr * kHlCapS;
            int* rbp = buf_p + rr * kHlCapS;
            float mfin = -INFINITY, sfin = 0.0f;
            int n = 0;
            if (any) {
                float v[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) v[j] = zs[rr * kHlZS + lane + 32 * j];
                float lm = v[0];
#pragma unroll
                for (int j = 1; j < 8; ++j) lm = fmaxf(lm, v[j]);
                const float M = warp_max(lm);
                float sacc = 0.0f;
                if (M != -INFINITY) {
                    const float mb = M * kL2E;
#pragma unroll
                    for (int j = 0; j < 8; ++j) sacc += ex2f(fmaf(v[j], kL2E, -mb));
                }
                sacc = warp_sum(sacc);
                const float mo = st_m[rr], so = st_s[rr];
                mfin = fmaxf(mo, M);
                sfin = (mo == -INFINITY ? 0.0f : so * ex2f((mo - mfin) * kL2E)) +
                       (M == -INFINITY ? 0.0f : sacc * ex2f((M - mfin) * kL2E));
                const int n_old = st_n[rr];
                const float Br = b_run[rr];
                float B = -INFINITY;
                if (n_old + ftn > kHlCap) {   // the KP-th largest lane maximum (KP <= 32)
                    float x = lm;
#pragma unroll 1
                    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll 1
                        for (int j = k >> 1; j > 0; j >>= 1) {
                            const float y = __shfl_xor_sync(0xffffffffu, x, j);
                            x = (((lane & k) == 0) == ((lane & j) == 0)) ? fmaxf(x, y) : fminf(x, y);
                        }
                    B = __shfl_sync(0xffffffffu, x, KP - 1);
                }
                uint32_t bal[8];
                int cnt = 0;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    bal[j] = __ballot_sync(0xffffffffu, v[j] >= B && v[j] > Br);
                    cnt += __popc(bal[j]);
                }
                if (n_old + cnt <= kHlCap) {
                    int pos = n_old;
                    const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        if (wr && ((bal[j] >> lane) & 1u)) {
                            const int sl = pos + __popc(bal[j] & lt);
                            rbv[sl] = v[j];
                            rbp[sl] = ft0 + lane + 32 * j;
                        }
                        pos += __popc(bal[j]);
                    }
                    n = n_old + cnt;
                } else if (wr) {
                    hl_warp_select(zs + rr * kHlZS, B, Br, rbv, rbp, n_old, ft0, KP, lane);   // (rare: ties)
                    n = KP;
                }
                __syncwarp();
            }
            for (int i = lane; i < LS && wr; i += 32) {
                const bool h = i < n;
                a.part.val[o * LS + i] = h ? rbv[i] : -INFINITY;
                a.part.id[o * LS + i] = h ? rbp[i] : -1;
            }
            if (lane == 0 && wr) {
                a.part.m[o] = mfin;
                a.part.s[o] = sfin;
                a.part.cnt[o] = 0;
                a.part.xcnt[o] = n;
            }
        }
        }
        (void)fseen;
        if (warp == 0 && lane == 0) HL_TRACE(6);
        HL_CLK(9);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) HL_TRACE(7);
    if (warp == kHlMmaWarp)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(2 * kHlTile));
}

// ------------------------------------------------------------------ host
bool lmh_hl_supported(const LmhArgs& a) {
    return a.w_dtype == 0 && a.h_dtype == 0 && a.d % 64 == 0 && a.d >= 64 && a.n_h >= 1 && a.n_h <= kHlRows &&
           a.nseg == 0 && a.KP <= 32 && a.n_w_rows <= INT_MAX;
}

cudaError_t launch_lmh_hl(const LmhArgs& a, cudaStream_t st) {
    const int G = a.grid > 0 ? a.grid : kNumSMs;
    auto tile_rows = [&](long long n) {   // largest tile of an even split of n positions over G CTAs
        const long long per = (n + G - 1) / G;
        const long long nt = std::max(1LL, (per + kHlTile - 1) / kHlTile);
        return (int)((per + nt - 1) / nt);
    };
    int nw = a.list2 ? std::max(tile_rows(a.n1), tile_rows(a.n_list2_max)) : tile_rows(a.n_subset_max);
    nw = std::max(16, (nw + 15) & ~15);
    HlParams hp{};
    hp.nkb = a.d / 64;
    hp.bh = (a.n_h + 7) & ~7;
    const int unit = kHlHBytes + ((nw * 128 + 1023) & ~1023);   // one K-block of the largest tile
    const int epi = hl_epi_bytes();
    const int bar = (2 * kHlMaxSlots + 4) * 8 + 16;
    const int budget = 227 * 1024 - 1024 /*alignment slack*/ - epi - bar;
    // S slots of several K-blocks each: every slot costs a fixed handshake (~0.3-0.5 us
    // measured: the consumer's wait + MMA issue + commit), so a slot carries as many
    // K-blocks as the ring allows with S slots (EVOSPEC_HL_SLOTS, default 2)
    int S = 2;   // (3, 4 and 8 slots measured slower at 36,864 rows)
    while (S > 2 && budget / S < unit) --S;
    const int kps = std::max(1, std::min(hp.nkb, budget / S / unit));
    hp.slot_bytes = kps * unit;
    if (budget / hp.slot_bytes < S) S = budget / hp.slot_bytes;
    // the ring also holds the last tile's staged logits (64 rows x kHlZS floats)
    while (S * hp.slot_bytes < kHlRows * kHlZS * 4 && (S + 1) * hp.slot_bytes <= budget && S < kHlMaxSlots) ++S;
    if (S < 2 || S * hp.slot_bytes < kHlRows * kHlZS * 4) return cudaErrorInvalidConfiguration;
    hp.slots = S;
    hp.off_epi = S * hp.slot_bytes;   // (>= 8 KB after the ring: the M = 128 A operand reads past a slot's H block)
    hp.off_bar = (hp.off_epi + epi + 15) & ~15;
    const size_t smem = (size_t)hp.off_bar + (size_t)(2 * S + 4) * 8 + 16 + 1024;
    CUtensorMap mh;
    if (!cached_map(&mh, a.H, (uint64_t)a.d, (uint64_t)a.n_h, 64, (uint32_t)hp.bh, CU_TENSOR_MAP_L2_PROMOTION_L2_128B))
        return cudaErrorInvalidValue;
    cudaError_t e = ensure_smem(lmh_hl_kernel, smem);
    if (e != cudaSuccess) return e;
    return launch_pdl(lmh_hl_kernel, dim3(G), dim3(kHlThreads), smem, st, mh, a, hp);
}

}  // namespace es
