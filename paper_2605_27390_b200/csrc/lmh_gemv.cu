// lmh_gemv.cu -- a5-a7 for narrow draft trees (n_h <= 8) and fp32 heads:
// z[r][j] = inv_temp * sum_c H[r][c] W[S_j][c] with FFMA, fused with the
// online softmax / top-k epilogue. Bandwidth-bound: every gathered W row is
// read once with 16-byte streaming loads (Eq. projection P:44-48 restricted
// to V_t, alg:evospec P:364).
//
// CTA = 8 warps, persistent over a contiguous run of subset positions.
// A warp takes 8 subset rows at a time; lane l owns the 16-byte pieces
// l, l+32, ... of each row; H lives in shared memory lane-interleaved
// ([r][chunk][elem][lane], conflict-free) and is read once per 8 rows.
// The 8 x NH per-lane partial sums are reduce-scattered across the warp.
#include "common.cuh"
#include "kernels.cuh"
#include "lmh_epilogue.cuh"

namespace es {

constexpr int kGemvWarps = 8;
constexpr int kGemvRows = 8;   // rows per warp iteration

int lmh_gemv_grid() { return 2 * kNumSMs; }

// Reduce-scatter T per-lane values across the warp. Afterwards a lane holds
// max(1, T/32) consecutive complete sums starting at rs_index(lane).
template <int T>
ES_DEV void reduce_scatter(float (&v)[T], int lane) {
    int c = T;
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1) {
        if (c >= 2) {
            const int half = c >> 1;
            const bool upper = (lane & h) != 0;
#pragma unroll
            for (int i = 0; i < T / 2; ++i) {
                if (i < half) {
                    float send = upper ? v[i] : v[i + half];
                    float keep = upper ? v[i + half] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
                }
            }
            c = half;
        } else {
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], h);
        }
    }
}
template <int T>
ES_DEV int rs_index(int lane) {
    int c = T, idx = 0;
#pragma unroll
    for (int h = 16; h >= 1; h >>= 1)
        if (c >= 2) { const int half = c >> 1; if (lane & h) idx += half; c = half; }
    return idx;
}
template <int T>
ES_DEV bool rs_writer(int lane) { return T >= 32 ? true : (lane & (32 / T - 1)) == 0; }

template <int DT, int NH>
__global__ void __launch_bounds__(kGemvWarps * 32, 2)
lmh_gemv_kernel(LmhArgs a, int h_row0) {
    constexpr int ELEMS = DT == 0 ? 8 : 4;
    // rows per warp batch: 16 for a single tree row (one batch per 128-row tile: no
    // pipeline drain between batches, twice the loads in flight), else 8
    constexpr int ROWS = NH == 1 ? 16 : kGemvRows;
    constexpr int T = ROWS * NH;
    constexpr int NV = T >= 32 ? T / 32 : 1;
    extern __shared__ __align__(16) unsigned char g_sm[];
    const int d = a.d;
    const int n_chunks = (d + 32 * ELEMS - 1) / (32 * ELEMS);
    float* H_sm = (float*)g_sm;                              // [NH][n_chunks][ELEMS][32]
    EpiSmem e = epi_carve(g_sm + (size_t)NH * n_chunks * ELEMS * 32 * 4, NH, a.KP, kGemvWarps);
    const int lane = lane_id(), warp = warp_id();

    if (a.h_dtype == 0 && d % 8 == 0 && ELEMS == 8) {
        // bf16 H: one 16-byte load per (row, chunk, lane) -> its 8 elements (every CTA
        // stages H first, so this is a fixed cost of the launch: vectorised, no divisions)
        const int per_row = n_chunks * 32;
        for (int i = threadIdx.x; i < NH * per_row; i += blockDim.x) {
            const int r = i / per_row, rem = i - r * per_row;   // rem = ch * 32 + ln
            const int ch = rem >> 5, ln = rem & 31;
            const int c = ch * 32 * 8 + ln * 8;
            float f[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            if (c < d) unpack_bf16x8(__ldg((const uint4*)((const uint16_t*)a.H + (size_t)(h_row0 + r) * d + c)), f);
            float* dst = H_sm + ((size_t)(r * n_chunks + ch) * 8) * 32 + ln;
#pragma unroll
            for (int j = 0; j < 8; ++j) dst[j * 32] = f[j];
        }
    } else {
        for (int i = threadIdx.x; i < NH * n_chunks * ELEMS * 32; i += blockDim.x) {
            int r = i / (n_chunks * ELEMS * 32), rem = i % (n_chunks * ELEMS * 32);
            int ch = rem / (ELEMS * 32), j = (rem / 32) % ELEMS, ln = rem % 32;
            int c = ch * 32 * ELEMS + ln * ELEMS + j;
            float v = 0.0f;
            if (c < d) {
                size_t o = (size_t)(h_row0 + r) * d + c;
                v = a.h_dtype == 0 ? bf16_bits_to_f32(((const uint16_t*)a.H)[o]) : ((const float*)a.H)[o];
            }
            H_sm[i] = v;
        }
    }
    epi_init(e, NH);
    __syncthreads();

    int p0, p1;
    lmh_cta_range(a, p0, p1);
    const size_t row_bytes = (size_t)d * (DT == 0 ? 2 : 4);

    for (int tb = p0; tb < p1; tb += kTile) {
        const int tn = min(kTile, p1 - tb);
        // each warp: rows [tb + 16 w, tb + 16 w + 16) in batches of ROWS
        for (int bt = 0; bt < kTile / (kGemvWarps * ROWS); ++bt) {
            const int rbase = warp * (kTile / kGemvWarps) + bt * ROWS;   // tile-local
            const char* rowp[ROWS];
            bool ok[ROWS];
#pragma unroll
            for (int i = 0; i < ROWS; ++i) {
                const int p = rbase + i;
                ok[i] = p < tn;
                const int32_t id = ok[i] ? a.subset[tb + p] : 0;
                rowp[i] = (const char*)a.W + (size_t)(id / a.R) * row_bytes;
            }
            float acc[T];
#pragma unroll
            for (int i = 0; i < T; ++i) acc[i] = 0.0f;
#pragma unroll 2
            for (int ch = 0; ch < n_chunks; ++ch) {
                const int c0 = ch * 32 * ELEMS + lane * ELEMS;
                const bool cok = c0 < d;
                uint4 u[ROWS];
#pragma unroll
                for (int i = 0; i < ROWS; ++i)
                    u[i] = (ok[i] && cok) ? ld_stream(rowp[i] + (size_t)c0 * (DT == 0 ? 2 : 4))
                                          : make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int r = 0; r < NH; ++r) {
                    float hv[ELEMS];
#pragma unroll
                    for (int j = 0; j < ELEMS; ++j) hv[j] = H_sm[((r * n_chunks + ch) * ELEMS + j) * 32 + lane];
#pragma unroll
                    for (int i = 0; i < ROWS; ++i) {
                        float f[ELEMS];
                        if constexpr (DT == 0) {
                            float g[8];
                            unpack_bf16x8(u[i], g);
#pragma unroll
                            for (int j = 0; j < 8; ++j) f[j] = g[j];
                        } else {
                            f[0] = __uint_as_float(u[i].x); f[1] = __uint_as_float(u[i].y);
                            f[2] = __uint_as_float(u[i].z); f[3] = __uint_as_float(u[i].w);
                        }
                        float s = acc[i * NH + r];
#pragma unroll
                        for (int j = 0; j < ELEMS; ++j) s = fmaf(f[j], hv[j], s);
                        acc[i * NH + r] = s;
                    }
                }
            }
            reduce_scatter<T>(acc, lane);
            if (rs_writer<T>(lane)) {
                const int idx0 = rs_index<T>(lane);
#pragma unroll
                for (int q = 0; q < NV; ++q) {
                    const int idx = idx0 + q;
                    const int i = idx / NH, r = idx % NH;
                    const float z = acc[q] * a.inv_temp;
                    e.tile[r * kTile + rbase + i] = z;
                    if (a.logits_out && rbase + i < tn)
                        a.logits_out[(size_t)(h_row0 + r) * a.n_subset_max + tb + rbase + i] = z;
                }
            }
        }
        __syncthreads();
        epi_tile(e, NH, a.KP, tn, tb, warp, kGemvWarps);
        __syncthreads();
    }
    epi_store(e, a.part, blockIdx.x, a.n_h, h_row0, NH, a.KP, a.LS, warp, kGemvWarps);
}

template <int DT, int NH>
static size_t smem_t(const LmhArgs& a) {
    const int elems = DT == 0 ? 8 : 4;
    const int n_chunks = (a.d + 32 * elems - 1) / (32 * elems);
    return (size_t)NH * n_chunks * elems * 32 * 4 + epi_smem_bytes(NH, a.KP, kGemvWarps);
}

template <int DT, int NH>
static void launch_t(const LmhArgs& a, int h_row0, cudaStream_t st) {
    const size_t smem = smem_t<DT, NH>(a);
    cudaFuncSetAttribute(lmh_gemv_kernel<DT, NH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    lmh_gemv_kernel<DT, NH><<<lmh_gemv_grid(), kGemvWarps * 32, smem, st>>>(a, h_row0);
}

// Largest group width NH in {8,4,2,1}, NH <= n_left, whose shared memory
// still lets two CTAs share an SM (<= 110 KB each).
int lmh_gemv_group_width(const LmhArgs& a, int n_left) {
    const size_t cap = 110 * 1024;
    auto fits = [&](int nh) {
        if (a.w_dtype == 0)
            return (nh == 4 ? smem_t<0, 4>(a) : nh == 2 ? smem_t<0, 2>(a) : smem_t<0, 1>(a)) <= cap;
        return (nh == 4 ? smem_t<1, 4>(a) : nh == 2 ? smem_t<1, 2>(a) : smem_t<1, 1>(a)) <= cap;
    };
    for (int nh = 4; nh > 1; nh >>= 1)   // NH = 8 exceeds the 128-register budget
        if (nh <= n_left && fits(nh)) return nh;
    return 1;
}

int launch_lmh_gemv(const LmhArgs& a, int h_row0, int n_h_grp, cudaStream_t st) {
    // each group launch covers exactly n_h_grp (in {8,4,2,1}) rows of H
    if (a.w_dtype == 0) {
        switch (n_h_grp) {
            case 4: launch_t<0, 4>(a, h_row0, st); break;
            case 2: launch_t<0, 2>(a, h_row0, st); break;
            default: launch_t<0, 1>(a, h_row0, st); break;
        }
    } else {
        switch (n_h_grp) {
            case 4: launch_t<1, 4>(a, h_row0, st); break;
            case 2: launch_t<1, 2>(a, h_row0, st); break;
            default: launch_t<1, 1>(a, h_row0, st); break;
        }
    }
    return lmh_gemv_grid();
}

}  // namespace es
