// sem.cu -- a2: semantic retrieval S_sem as an EXACT GPU scan.
//
// The paper retrieves the top-N MIPS neighbours of the target hidden state
// over the LM-head rows with HNSW (App. A.3). HNSW
// approximates the exact answer; on a B200 the exact scan q . E^T over all
// 128k rows is one HBM pass (~1 GB, ~160 us), so we compute the exact answer
// (reading C2 in DESIGN.md) and select the top-N by (score desc, id asc).
//
// Kernels:
//   sem_scan_kernel     s64[v] = sum_c q[c] E[v][c] in fp64 (bf16 x fp32 products
//                       are exact in fp64), one warp per 16-row chunk, 16-byte
//                       streaming loads, q held per lane from a lane-interleaved
//                       fp64 copy in shared memory.
//                       The scan also histograms the top 12 bits of the
//                       order-preserving fp32 key of every score.
//   topn_cand_kernel    cooperative radix select over the composite key
//                       (float_key(s), double_key(s), ~id). Pass 0 reuses the
//                       scan's histogram, so in the common case no grid-wide
//                       sync runs: every CTA finds the boundary bin b and emits
//                       all scores in bins >= b -- a candidate SUPERSET of the
//                       top-N of at most `cap` elements, carrying exact keys.
//                       Further passes (grid.sync) run only if that superset
//                       would not fit. The exact top-N, its order where the
//                       formation needs it, and the cap are resolved in the
//                       union kernel (union.cu) on those exact keys.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace es {

// ---------------------------------------------------------------- scan
// Block: kScanWarps warps; each warp owns a contiguous row range and walks it
// in chunks of 16 rows. Per chunk and per 256-column slab (bf16; 128 for
// fp32) each lane loads one 16-byte piece of each of the 16 rows.
template <int DT>  // element type of E: 0 bf16, 1 fp32
__global__ void __launch_bounds__(kScanWarps * 32, 1)
sem_scan_kernel(const void* __restrict__ E, int64_t n_rows, int d,
                const void* __restrict__ q, int q_dtype, uint32_t* __restrict__ hist12,
                double* __restrict__ s64, uint32_t* __restrict__ key32) {
    constexpr int ELEMS = DT == 0 ? 8 : 4;           // elements per 16 bytes
    constexpr int SLAB = 32 * ELEMS;                  // columns per slab
    extern __shared__ double q_sm[];                  // [n_slabs][ELEMS][32]
    __shared__ uint32_t hist_sm[kHistBins];           // top-12-bit histogram of key32
    const int n_slabs = (d + SLAB - 1) / SLAB;
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x) hist_sm[i] = 0;
    // stage q as fp64 in the lane-interleaved layout (exact: q is bf16/fp32)
    for (int i = threadIdx.x; i < n_slabs * SLAB; i += blockDim.x) {
        int s = i / SLAB, within = i % SLAB, lane = within / ELEMS, j = within % ELEMS;
        int c = s * SLAB + within;
        double v = 0.0;
        if (c < d) v = q_dtype == 0 ? (double)bf16_bits_to_f32(((const uint16_t*)q)[c])
                                    : (double)((const float*)q)[c];
        // bf16 E: q is pre-scaled by 2^896 (exact; |q| < 2^128 stays finite) so
        // that each E element can enter as the "raw" double whose fields are the
        // bf16 fields in place (value e * 2^-896, exact, no conversion unit):
        // the product q*e, hence every fma, is bit-identical to the unscaled one
        if (DT == 0) v *= 0x1p896;
        q_sm[(s * ELEMS + j) * 32 + lane] = v;
    }
    __syncthreads();

    const int lane = lane_id();
    const int64_t gw = (int64_t)blockIdx.x * kScanWarps + warp_id();
    const int64_t nw = (int64_t)gridDim.x * kScanWarps;
    const int64_t r0 = n_rows * gw / nw, r1 = n_rows * (gw + 1) / nw;
    const size_t row_bytes = (size_t)d * (DT == 0 ? 2 : 4);

    for (int64_t base = r0; base < r1; base += 16) {
        double acc[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) acc[r] = 0.0;
        for (int s = 0; s < n_slabs; ++s) {
            const int c0 = s * SLAB + lane * ELEMS;
            const bool col_ok = c0 < d;
            uint4 u[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                int64_t row = base + r;
                if (col_ok && row < r1)
                    u[r] = ld_stream((const char*)E + row * row_bytes + (size_t)c0 * (DT == 0 ? 2 : 4));
                else
                    u[r] = make_uint4(0, 0, 0, 0);
            }
            double qv[ELEMS];
#pragma unroll
            for (int j = 0; j < ELEMS; ++j) qv[j] = q_sm[(s * ELEMS + j) * 32 + lane];
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                if constexpr (DT == 0) {
                    const uint32_t w4[4] = {u[r].x, u[r].y, u[r].z, u[r].w};
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        // sign | exp | mant of a bf16 moved to the double's field positions:
                        // arithmetic >> 3 puts exp at [27:20], mant at [19:13]; the mask
                        // keeps the sign at bit 31 (bf16 zero / denormal map exactly too)
                        const uint32_t lo = (uint32_t)((int32_t)(w4[j] << 16) >> 3) & 0x8FFFE000u;
                        const uint32_t hi = (uint32_t)((int32_t)w4[j] >> 3) & 0x8FFFE000u;
                        acc[r] = fma(__hiloint2double((int)lo, 0), qv[2 * j], acc[r]);
                        acc[r] = fma(__hiloint2double((int)hi, 0), qv[2 * j + 1], acc[r]);
                    }
                } else {
                    float f[4] = {__uint_as_float(u[r].x), __uint_as_float(u[r].y),
                                  __uint_as_float(u[r].z), __uint_as_float(u[r].w)};
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[r] = fma((double)f[j], qv[j], acc[r]);
                }
            }
        }
        // reduce-scatter 16 rows over 32 lanes: lane l ends with row (l & 15)
#pragma unroll
        for (int h = 8; h >= 1; h >>= 1) {
            const bool upper = (lane & h) != 0;
#pragma unroll
            for (int i = 0; i < h; ++i) {
                double send = upper ? acc[i] : acc[i + h];
                double keep = upper ? acc[i + h] : acc[i];
                acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, h);
            }
        }
        double tot = acc[0] + __shfl_xor_sync(0xffffffffu, acc[0], 16);
        int64_t row = base + (lane & 15);
        uint32_t digit = 0xFFFFFFFFu;
        if (lane < 16 && row < r1) {
            const uint32_t k = float_key((float)tot);
            s64[row] = tot;
            key32[row] = k;
            digit = k >> 20;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, digit);
        if (digit != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist_sm[digit], (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kHistBins; i += blockDim.x)
        if (hist_sm[i]) atomicAdd(&hist12[i], hist_sm[i]);
}

void launch_sem_scan(const void* E, int e_dtype, int64_t n_rows, int d, const void* q, int q_dtype,
                     double* s64, uint32_t* key32, uint32_t* hist12, cudaStream_t st) {
    cudaMemsetAsync(hist12, 0, kHistBins * sizeof(uint32_t), st);
    const int elems = e_dtype == 0 ? 8 : 4;
    const int n_slabs = (d + 32 * elems - 1) / (32 * elems);
    const size_t smem = (size_t)n_slabs * 32 * elems * sizeof(double);
    if (e_dtype == 0) {
        cudaFuncSetAttribute(sem_scan_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        sem_scan_kernel<0><<<kNumSMs, kScanWarps * 32, smem, st>>>(E, n_rows, d, q, q_dtype, hist12, s64, key32);
    } else {
        cudaFuncSetAttribute(sem_scan_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        sem_scan_kernel<1><<<kNumSMs, kScanWarps * 32, smem, st>>>(E, n_rows, d, q, q_dtype, hist12, s64, key32);
    }
}

// ---------------------------------------------------------------- select
struct SelWords { uint32_t w[4]; };

ES_DEV SelWords sel_words(double s, int32_t id) {
    SelWords k;
    k.w[0] = float_key((float)s);
    uint64_t dk = double_key(s);
    k.w[1] = (uint32_t)(dk >> 32);
    k.w[2] = (uint32_t)dk;
    k.w[3] = 0xFFFFFFFFu - (uint32_t)id;   // lower id ranks higher
    return k;
}

struct SelState {
    uint32_t pmask[4], pval[4];
    int remaining;
    int done;
};

ES_DEV bool sel_matches(const SelWords& k, const SelState& st) {
#pragma unroll
    for (int w = 0; w < 4; ++w)
        if ((k.w[w] & st.pmask[w]) != st.pval[w]) return false;
    return true;
}
// composite-prefix >= selected prefix
ES_DEV bool sel_selected(const SelWords& k, const SelState& st) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        uint32_t a = k.w[w] & st.pmask[w];
        if (a != st.pval[w]) return a > st.pval[w];
    }
    return true;
}

// digit schedule: word 0 (fp32 key) 12/10/10 bits -- pass 0 matches the
// scan's 4096-bin histogram; words 1-3: 11/11/10 bits.
ES_DEV void pass_digit(int pass, int& word, int& shift, int& nbits) {
    word = pass / 3;
    const int part = pass % 3;
    if (word == 0) { shift = part == 0 ? 20 : (part == 1 ? 10 : 0); nbits = part == 0 ? 12 : 10; }
    else { shift = part == 0 ? 21 : (part == 1 ? 10 : 0); nbits = part == 2 ? 10 : 11; }
}

__global__ void __launch_bounds__(kSelThreads, 1)
topn_cand_kernel(const double* __restrict__ s64, const int32_t* __restrict__ ids, int64_t n,
                 int id_mul, int id_add, int N, int cap, const uint32_t* __restrict__ hist_pre,
                 uint32_t* __restrict__ hist_g, int* __restrict__ out_count, double* __restrict__ out_s,
                 int32_t* __restrict__ out_id) {
    cg::grid_group grid = cg::this_grid();
    __shared__ uint32_t hist[kHistBins];
    __shared__ uint32_t warp_sum_s[kSelThreads / 32];
    __shared__ SelState st;
    __shared__ int found_bin, found_above;

    const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
    auto id_of = [&](int64_t i) -> int32_t { return ids ? ids[i] : (int32_t)(i * id_mul + id_add); };
    const int lane = lane_id(), wid = warp_id();

    if (threadIdx.x == 0) {
        for (int w = 0; w < 4; ++w) { st.pmask[w] = 0; st.pval[w] = 0; }
        st.remaining = N < 0 ? 0 : N;
        st.done = (N >= n) || (N <= 0);
    }
    __syncthreads();

    for (int pass = 0; pass < 12 && !st.done; ++pass) {
        int word, shift, nbits;
        pass_digit(pass, word, shift, nbits);
        const uint32_t dmask = (1u << nbits) - 1u;
        const uint32_t* hp;
        if (pass == 0 && hist_pre) {
            hp = hist_pre;
        } else {
            for (int b = threadIdx.x; b < kHistBins; b += blockDim.x) hist[b] = 0;
            __syncthreads();
            SelState my = st;
            for (int64_t b0 = lo; b0 < hi; b0 += blockDim.x) {   // uniform trip count per warp
                const int64_t i = b0 + threadIdx.x;
                uint32_t digit = 0xFFFFFFFFu;
                if (i < hi && id_of(i) >= 0) {
                    SelWords k = sel_words(s64[i], id_of(i));
                    if (sel_matches(k, my)) digit = (k.w[word] >> shift) & dmask;
                }
                const unsigned peers = __match_any_sync(0xffffffffu, digit);
                if (digit != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&hist[digit], (uint32_t)__popc(peers));
            }
            __syncthreads();
            uint32_t* hw = hist_g + (size_t)pass * kHistBins;
            for (int b = threadIdx.x; b < (1 << nbits); b += blockDim.x)
                if (hist[b]) atomicAdd(&hw[b], hist[b]);
            grid.sync();
            hp = hw;
        }
        // every CTA: the bin (descending) where the running count reaches `remaining`;
        // thread t owns bins [8t, 8t+8)
        constexpr int BPT = kHistBins / kSelThreads;
        uint32_t c[BPT], tot = 0;
        const int t = threadIdx.x;
#pragma unroll
        for (int j = 0; j < BPT; ++j) {
            const int b = BPT * t + j;
            c[j] = b < (1 << nbits) ? __ldcg(&hp[b]) : 0u;
            tot += c[j];
        }
        uint32_t inc = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t v = __shfl_down_sync(0xffffffffu, inc, o);
            if (lane + o < 32) inc += v;
        }
        if (lane == 0) warp_sum_s[wid] = inc;
        __syncthreads();
        uint32_t above_w = 0;
        for (int w2 = wid + 1; w2 < kSelThreads / 32; ++w2) above_w += warp_sum_s[w2];
        const uint32_t rem = (uint32_t)st.remaining;
        uint32_t run = above_w + inc - tot;   // count in bins above this thread's range
#pragma unroll
        for (int j = BPT - 1; j >= 0; --j) {
            if (run < rem && run + c[j] >= rem) { found_bin = BPT * t + j; found_above = (int)run; }
            run += c[j];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int b = found_bin;
            const uint32_t in_bin = __ldcg(&hp[b]);
            const long long superset = (long long)(N - st.remaining) + found_above + in_bin;
            st.remaining -= found_above;
            st.pmask[word] |= dmask << shift;
            st.pval[word] |= ((uint32_t)b) << shift;
            // exact, or a candidate superset (everything in bins >= b) that fits
            if ((uint32_t)st.remaining == in_bin || superset <= cap) st.done = 1;
        }
        __syncthreads();
    }
    // compaction: warp-aggregated appends of (double_key(s), id)
    SelState my = st;
    const bool take_all = (N >= n);
    for (int64_t b0 = lo; b0 < hi; b0 += blockDim.x) {
        const int64_t i = b0 + threadIdx.x;
        bool sel = false;
        double s = 0.0;
        int32_t id = 0;
        if (i < hi) {
            s = s64[i];
            id = id_of(i);
            sel = id >= 0 && (take_all || (N > 0 && sel_selected(sel_words(s, id), my)));
        }
        const unsigned m = __ballot_sync(0xffffffffu, sel);
        int base = 0;
        if (lane == 0 && m) base = atomicAdd(out_count, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        const int o = base + __popc(m & ((1u << lane) - 1u));
        if (sel && o < cap) { out_s[o] = s; out_id[o] = id; }
    }
}

cudaError_t launch_topn_cand(const double* s64, const int32_t* ids, int64_t n, int id_mul, int id_add,
                             int N, int cap, const uint32_t* hist_pre, uint32_t* hist_g, int* out_count,
                             double* out_s, int32_t* out_id, cudaStream_t st) {
    cudaMemsetAsync(hist_g, 0, 12 * kHistBins * sizeof(uint32_t), st);
    cudaMemsetAsync(out_count, 0, sizeof(int), st);
    int grid = kNumSMs;
    if (n < (int64_t)grid * 64) grid = (int)((n + 63) / 64);
    if (grid < 1) grid = 1;
    void* args[] = {(void*)&s64, (void*)&ids, (void*)&n, (void*)&id_mul, (void*)&id_add, (void*)&N, (void*)&cap,
                    (void*)&hist_pre, (void*)&hist_g, (void*)&out_count, (void*)&out_s, (void*)&out_id};
    return cudaLaunchCooperativeKernel((void*)topn_cand_kernel, grid, kSelThreads, args, 0, st);
}

}  // namespace es
