// union.cu -- a3/a4: statistical expansion, runtime candidate formation,
// budget cap and the sorted union  V_t = V_static u dyn  (Eq. vocab_union
// P:88-93; formation App. A.3; budget |V_t \ V_static| <= N_dyn,
// Eq. optimization; cap order S:260; readings C4-C9).
//
// One CTA: the semantic candidates (an exact-keyed superset of S_sem from
// sem.cu), the answer as a V-bit membership bitmap (16 KB at V = 128k) and
// the graph lists all live in shared memory:
//   1. static ids -> bitmap;
//   2. S_sem = exact top-N_sem of the candidates (block radix select on
//      (double_key(s), ~id));
//   3. the ordered prefix S_sem[:n_graph_sem_seeds] (select + rank);
//      G = dedupe(seeds ++ that prefix); S_graph = the first per_seed CSR
//      successors of each g in G, in G order;
//   4. formation: seeds, then the first (budget) NEW ids of S_sem in S_sem
//      order (= exact top-budget of the new ones), then S_graph and S_ctx
//      walked 32 ids at a time (match.any first-occurrence) until N_dyn ids
//      are taken -- the same set the sequential walk of the definition takes;
//   5. block-wide popcount scan of the bitmap writes the sorted ids (and this
//      shard's slice v mod R == r).
// Two-list draft step (early_flag != null): right after the selections the
// new seeds and the semantic part are also written, unsorted, to early_ids; if
// they fill N_dyn the dynamic list is complete (steps 3-4's graph and context
// walks add nothing) and its length + 1 is release-stored to *early_flag, else
// -1 -- the LM head (lmh_tc.cu) starts its dynamic tiles on that, ~11 us
// before this kernel's end.
#include "common.cuh"
#include "kernels.cuh"

namespace es {

static constexpr int kMaxG = 128;

ES_DEV int block_excl_scan(int v, int* warp_tot, int& total) {
    const int lane = lane_id(), wid = warp_id(), nw = blockDim.x / 32;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_tot[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        int w = lane < nw ? warp_tot[lane] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < nw) warp_tot[lane] = wi - w;  // exclusive
        if (lane == nw - 1) warp_tot[32] = wi;
    }
    __syncthreads();
    int res = warp_tot[wid] + inc - v;
    total = warp_tot[32];
    __syncthreads();
    return res;
}

// ------------------------------------------------------------ S_ctx (C5)
// ids of ctx with count >= min_count, ordered (count desc, id asc), first n_max.
__global__ void __launch_bounds__(kUnionThreads, 1)
ctx_select_kernel(const int32_t* __restrict__ ctx, int n_ctx, int V, int min_count, int n_max,
                  int32_t* __restrict__ out, int* __restrict__ out_n, int* flags) {
    extern __shared__ unsigned char cs_sm[];
    int P = 1;
    while (P < n_ctx) P <<= 1;
    uint32_t* a = (uint32_t*)cs_sm;                        // [P]
    unsigned long long* key = (unsigned long long*)(a + P);  // [P]
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        uint32_t v = 0xFFFFFFFFu;
        if (i < n_ctx) {
            int32_t c = ctx[i];
            if (c < 0 || c >= V) { atomicOr(flags, kFlagBadIds); c = -1; }
            v = c < 0 ? 0xFFFFFFFFu : (uint32_t)c;
        }
        a[i] = v;
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    bool asc = (i & k) == 0;
                    uint32_t x = a[i], y = a[ixj];
                    if ((x > y) == asc) { a[i] = y; a[ixj] = x; }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < P; i += blockDim.x) {
        unsigned long long kk = 0;
        uint32_t v = a[i];
        if (v != 0xFFFFFFFFu && (i == 0 || a[i - 1] != v)) {
            int e = i;
            while (e < P && a[e] == v) ++e;
            int cnt = e - i;
            if (cnt >= min_count) kk = ((unsigned long long)cnt << 32) | (0xFFFFFFFFull - v);
        }
        key[i] = kk;
    }
    __syncthreads();
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < P; i += blockDim.x) {
                int ixj = i ^ j;
                if (ixj > i) {
                    bool desc = (i & k) == 0;
                    unsigned long long x = key[i], y = key[ixj];
                    if ((x < y) == desc) { key[i] = y; key[ixj] = x; }
                }
            }
            __syncthreads();
        }
    __shared__ int n_out;
    if (threadIdx.x == 0) n_out = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < min(P, n_max); i += blockDim.x) {
        unsigned long long kk = key[i];
        if (kk != 0) {
            out[i] = (int32_t)(0xFFFFFFFFull - (kk & 0xFFFFFFFFull));
            atomicAdd(&n_out, 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) *out_n = n_out;  // nonzero keys are a prefix after the sort
}

void launch_ctx_select(const int32_t* ctx, int n_ctx, int V, int min_count, int n_max,
                       int32_t* out, int* out_n, int* flags, cudaStream_t st) {
    int P = 1;
    while (P < n_ctx) P <<= 1;
    size_t smem = (size_t)P * (4 + 8);
    cudaFuncSetAttribute(ctx_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ctx_select_kernel<<<1, kUnionThreads, smem, st>>>(ctx, n_ctx, V, min_count, n_max, out, out_n, flags);
}

// ------------------------------------------------------------ union
// Block-wide exact top-M under (key desc, id asc) among the candidates whose
// flag has any bit of A; marks them with bit S. Radix select on the composite
// (64-bit order key, ~id) with 10-bit digits (one histogram bin per thread),
// starting at the highest bit in which the active keys differ, so two or
// three passes settle ~10k fp64 scores; the ~id digits run only when the
// boundary holds equal keys. Exits as soon as the boundary bin is taken whole.
struct BSel {
    uint64_t kmask, kval;
    uint32_t imask, ival;
    int remaining, done, found_bin, found_above;
    uint64_t kmin, kmax;
};

ES_DEV bool bmatch(uint64_t k, int32_t id, const BSel& st) {
    return (k & st.kmask) == st.kval && ((0xFFFFFFFFu - (uint32_t)id) & st.imask) == st.ival;
}
ES_DEV bool bselected(uint64_t k, int32_t id, const BSel& st) {
    const uint64_t a = k & st.kmask;
    if (a != st.kval) return a > st.kval;
    return ((0xFFFFFFFFu - (uint32_t)id) & st.imask) >= st.ival;
}

ES_DEV int block_count(int v, int* warp_tot) {
    int total;
    block_excl_scan(v, warp_tot, total);
    return total;
}

ES_DEV uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o); v = w < v ? w : v; }
    return v;
}
ES_DEV uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o); v = w > v ? w : v; }
    return v;
}

constexpr int kSelBins = 1024;   // == kUnionThreads: one bin per thread in the scan

ES_DEV void block_topM(const uint64_t* ck, const int32_t* cid, uint8_t* cf, int n, uint8_t A, uint8_t S, int M,
                       uint32_t* hist, BSel& st, int* warp_tot) {
    const int tid = threadIdx.x, T = blockDim.x, lane = lane_id();
    int c = 0;
    uint64_t kmin = ~0ull, kmax = 0ull;
    for (int i = tid; i < n; i += T)
        if (cf[i] & A) { ++c; kmin = min(kmin, ck[i]); kmax = max(kmax, ck[i]); }
    kmin = warp_min_u64(kmin);
    kmax = warp_max_u64(kmax);
    if (tid == 0) { st.kmin = ~0ull; st.kmax = 0ull; }
    const int cnt = block_count(c, warp_tot);   // syncs: st initialised before the atomics below
    if (lane == 0 && kmin <= kmax) { atomicMin((unsigned long long*)&st.kmin, kmin); atomicMax((unsigned long long*)&st.kmax, kmax); }
    if (M >= cnt || M <= 0) {
        if (M > 0)
            for (int i = tid; i < n; i += T)
                if (cf[i] & A) cf[i] |= S;
        __syncthreads();
        return;
    }
    __syncthreads();
    if (tid == 0) {
        st.kmask = 0; st.kval = 0; st.imask = 0; st.ival = 0;
        st.remaining = M;
        st.done = 0;
    }
    __syncthreads();
    const uint64_t diff = st.kmin ^ st.kmax;
    int kbit = diff ? 63 - __clzll((long long)diff) : -1;   // highest differing key bit
    int ibit = 31;
    for (int pass = 0; pass < 16; ++pass) {
        if (st.done || (kbit < 0 && ibit < 0)) break;
        const bool on_key = kbit >= 0;
        const int hi = on_key ? kbit : ibit;
        const int width = hi + 1 < 10 ? hi + 1 : 10;
        const int lo = hi - width + 1;
        const uint32_t dmask = (1u << width) - 1u;
        for (int b = tid; b < kSelBins; b += T) hist[b] = 0;
        __syncthreads();
        const BSel my = st;
        // digits spread over ~1k bins (range-normalised), so plain smem atomics
        for (int i = tid; i < n; i += T)
            if ((cf[i] & A) && bmatch(ck[i], cid[i], my))
                atomicAdd(&hist[on_key ? (uint32_t)(ck[i] >> lo) & dmask
                                        : ((0xFFFFFFFFu - (uint32_t)cid[i]) >> lo) & dmask], 1u);
        __syncthreads();
        // thread t owns bin (kSelBins-1-t): an exclusive scan over t counts the bins above it
        const int bin = kSelBins - 1 - tid;
        const uint32_t hb = tid < kSelBins ? hist[bin] : 0u;
        int total;
        const int above = block_excl_scan((int)hb, warp_tot, total);
        if (tid < kSelBins && above < my.remaining && above + (int)hb >= my.remaining) {
            st.found_bin = bin;
            st.found_above = above;
        }
        __syncthreads();
        if (tid == 0) {
            const int b = st.found_bin;
            st.remaining -= st.found_above;
            if (on_key) { st.kmask |= (uint64_t)dmask << lo; st.kval |= (uint64_t)b << lo; }
            else { st.imask |= dmask << lo; st.ival |= (uint32_t)b << lo; }
            if ((uint32_t)st.remaining == hist[b]) st.done = 1;
        }
        __syncthreads();
        if (on_key) kbit = lo - 1; else ibit = lo - 1;
    }
    const BSel my = st;
    for (int i = tid; i < n; i += T)
        if ((cf[i] & A) && bselected(ck[i], cid[i], my)) cf[i] |= S;
    __syncthreads();
}

// K exact top-M selections at once (K <= 3): selection j takes the M[j] best
// (key desc, id asc) of the candidates whose flag has a bit of A[j] and marks
// them with S[j]. Key-linear binning: selection j keeps a window of keys
// [base, base + wspan] that holds its boundary; a pass histograms the active
// keys of every live window into kSelBins equal-width bins (one read of the
// candidates feeds the K histograms, one K-wide block scan finds the K
// boundary bins) and narrows the window to the boundary bin. The keys of
// fp64 scores spread over their range, so one pass usually leaves a boundary
// bin of a few dozen candidates: those are ranked exactly by counting under
// (key desc, id asc) and the first `remaining` taken. A boundary bin of more
// than kRankCap candidates that is a single key (equal scores) goes to
// block_topM, whose ~id digits settle it.
template <int K>
ES_DEV void block_scan_multi(const int (&v)[K], int* warp_tot /*[K][33]*/, int (&excl)[K]) {
    const int lane = lane_id(), wid = warp_id(), nw = blockDim.x / 32;
    int inc[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        inc[j] = v[j];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc[j], o);
            if (lane >= o) inc[j] += t;
        }
        if (lane == 31) warp_tot[j * 33 + wid] = inc[j];
    }
    __syncthreads();
    if (wid < K) {
        const int w = lane < nw ? warp_tot[wid * 33 + lane] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < nw) warp_tot[wid * 33 + lane] = wi - w;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < K; ++j) excl[j] = warp_tot[j * 33 + wid] + inc[j] - v[j];
    __syncthreads();
}

constexpr int kRankCap = kSelBins;   // the rank lists reuse the selection's histogram
enum : int { kWLive = 0, kWWhole = 1, kWRank = 2, kWFallback = 3, kWAll = 4, kWNone = 5 };
struct WSel {
    uint64_t kmin, kmax, base, wspan;
    int shift, bin, above, remaining, mode, gn;
};

template <int K>
ES_DEV void block_topM_multi(const uint64_t* ck, const int32_t* cid, uint8_t* cf, int n, const uint8_t (&A)[K],
                             const uint8_t (&S)[K], const int (&M)[K], uint32_t* hist /*[K][kSelBins]*/,
                             WSel* ws /*[K]*/, BSel* bs /*[K]*/, int* warp_tot /*[K][33]*/, long long* tr = nullptr,
                             const int* pre_c = nullptr, const uint64_t* pre_lo = nullptr,
                             const uint64_t* pre_hi = nullptr) {
    const int tid = threadIdx.x, T = blockDim.x, lane = lane_id();
    auto stamp = [&](int i) {
        if (tr && tid == 0 && i < 16) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); tr[i] = t_; }
    };
    stamp(0);
    int c[K];
    uint64_t kmin[K], kmax[K];
#pragma unroll
    for (int j = 0; j < K; ++j) { c[j] = 0; kmin[j] = ~0ull; kmax[j] = 0ull; }
    if (pre_c) {   // this thread's statistics, gathered by the caller while loading
#pragma unroll
        for (int j = 0; j < K; ++j) { c[j] = pre_c[j]; kmin[j] = pre_lo[j]; kmax[j] = pre_hi[j]; }
    } else {
        for (int i = tid; i < n; i += T) {
            const uint8_t f = cf[i];
            const uint64_t k = ck[i];
#pragma unroll
            for (int j = 0; j < K; ++j)
                if (f & A[j]) { ++c[j]; kmin[j] = min(kmin[j], k); kmax[j] = max(kmax[j], k); }
        }
    }
    stamp(10);
    if (tid < K) ws[tid].gn = 0;
    {
        int ex[K];
        block_scan_multi<K>(c, warp_tot, ex);   // (syncs: ws initialised before the atomics)
        // totals: the last thread's exclusive prefix plus its own count
        if (tid == T - 1)
#pragma unroll
            for (int j = 0; j < K; ++j) warp_tot[j * 33 + 32] = ex[j] + c[j];
    }
    // key range: warp reductions, then one warp per selection over the warps' results
    // (64-bit shared atomics are CAS loops: 32 warps on one address serialise)
    uint64_t* red = (uint64_t*)hist;   // [2][K][32] (the histograms are free until the passes)
    const int wid = warp_id(), nw = T / 32;
#pragma unroll
    for (int j = 0; j < K; ++j) {
        kmin[j] = warp_min_u64(kmin[j]);
        kmax[j] = warp_max_u64(kmax[j]);
        if (lane == 0) { red[j * 32 + wid] = kmin[j]; red[(K + j) * 32 + wid] = kmax[j]; }
    }
    __syncthreads();
    if (wid < K) {
        const uint64_t lo = warp_min_u64(lane < nw ? red[wid * 32 + lane] : ~0ull);
        const uint64_t hi = warp_max_u64(lane < nw ? red[(K + wid) * 32 + lane] : 0ull);
        if (lane == 0) { ws[wid].kmin = lo; ws[wid].kmax = hi; }
    }
    __syncthreads();
    if (tid < K) {
        WSel& w = ws[tid];
        const int cnt = warp_tot[tid * 33 + 32];
        w.remaining = M[tid];
        if (M[tid] <= 0) w.mode = kWNone;
        else if (M[tid] >= cnt) w.mode = kWAll;
        else {
            w.mode = kWLive;
            w.base = w.kmin;
            w.wspan = w.kmax - w.kmin;
            const int bl = w.wspan ? 64 - __clzll((long long)w.wspan) : 0;
            w.shift = bl > 10 ? bl - 10 : 0;    // (wspan >> shift) < kSelBins
        }
    }
    __syncthreads();
    stamp(11);
    for (int pass = 0; pass < 8; ++pass) {
        WSel my[K];
        bool live[K];
        bool any = false;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            my[j] = ws[j];
            live[j] = my[j].mode == kWLive;
            any |= live[j];
        }
        if (!any) break;
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (live[j]) for (int b = tid; b < kSelBins; b += T) hist[j * kSelBins + b] = 0;
        __syncthreads();
        // equal-width bins over the window: ~n / kSelBins per bin, plain smem atomics
        for (int i = tid; i < n; i += T) {
            const uint8_t f = cf[i];
            const uint64_t k = ck[i];
#pragma unroll
            for (int j = 0; j < K; ++j)
                if (live[j] && (f & A[j]) && k - my[j].base <= my[j].wspan)   // (k < base wraps: outside)
                    atomicAdd(&hist[j * kSelBins + (int)((k - my[j].base) >> my[j].shift)], 1u);
        }
        __syncthreads();
        if (pass == 0) stamp(12);
        // thread t owns bin (kSelBins-1-t): an exclusive scan over t counts the bins above it
        const int bin = kSelBins - 1 - tid;
        int hb[K], above[K];
#pragma unroll
        for (int j = 0; j < K; ++j) hb[j] = (live[j] && tid < kSelBins) ? (int)hist[j * kSelBins + bin] : 0;
        block_scan_multi<K>(hb, warp_tot, above);
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (live[j] && tid < kSelBins && above[j] < my[j].remaining && above[j] + hb[j] >= my[j].remaining) {
                ws[j].bin = bin;
                ws[j].above = above[j];
            }
        __syncthreads();
        if (tid < K && live[tid]) {
            WSel& w = ws[tid];
            w.remaining -= w.above;
            const uint32_t h = hist[tid * kSelBins + w.bin];
            if ((uint32_t)w.remaining == h) w.mode = kWWhole;
            else if (h <= (uint32_t)kRankCap) w.mode = kWRank;
            else if (w.shift == 0) w.mode = kWFallback;
            else {   // narrow to the boundary bin
                w.base += (uint64_t)w.bin << w.shift;
                w.wspan = (1ull << w.shift) - 1ull;
                w.shift = w.shift > 10 ? w.shift - 10 : 0;
            }
        }
        __syncthreads();
        stamp(1 + pass);
    }
    // marking: everything above the boundary bin (and the bin itself when taken
    // whole); the boundary bins to be ranked are gathered into the histograms.
    // Per selection: selected iff key >= hi; ranked iff lo <= key < hi.
    WSel my[K];
    uint8_t a_eff[K];
    uint64_t klo[K], khi[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        my[j] = ws[j];
        a_eff[j] = (my[j].mode == kWNone || my[j].mode == kWFallback) ? 0 : A[j];
        if (my[j].mode == kWAll) { klo[j] = 0; khi[j] = 0; }
        else {
            klo[j] = my[j].base + ((uint64_t)my[j].bin << my[j].shift);
            const uint64_t up = (uint64_t)(my[j].bin + 1) << my[j].shift;
            khi[j] = my[j].base + (up > my[j].wspan ? my[j].wspan + 1 : up);
            if (my[j].mode == kWWhole) khi[j] = klo[j];
            if (my[j].mode != kWRank) klo[j] = khi[j];
        }
    }
    for (int i = tid; i < n; i += T) {
        const uint8_t f = cf[i];
        const uint64_t k = ck[i];
        uint8_t add = 0;
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if (!(f & a_eff[j])) continue;
            if (k >= khi[j]) add |= S[j];
            else if (k >= klo[j]) hist[j * kSelBins + atomicAdd(&ws[j].gn, 1)] = i;
        }
        if (add) cf[i] = f | add;
    }
    __syncthreads();
    stamp(13);
    // the boundary bins: rank each member among its bin's members by counting
    int tot = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) tot += my[j].mode == kWRank ? ws[j].gn : 0;
    for (int p = tid; p < tot; p += T) {
        int j = 0, start = 0, cnt = 0, rem = 0, acc = 0;
        unsigned int sb = 0;
#pragma unroll
        for (int q = 0; q < K; ++q) {   // (statically indexed: no local-memory copies of my[])
            const int g = my[q].mode == kWRank ? ws[q].gn : 0;
            if (p >= acc && p < acc + g) { j = q; start = acc; cnt = g; rem = my[q].remaining; sb = S[q]; }
            acc += g;
        }
        const uint32_t* list = hist + j * kSelBins;
        const int a = (int)list[p - start];
        const uint64_t ka = ck[a];
        const int32_t ia = cid[a];
        int rank = 0;
        for (int q = 0; q < cnt; ++q) {
            const int b = (int)list[q];
            rank += before(ck[b], cid[b], ka, ia) ? 1 : 0;
        }
        if (rank < rem)   // cf bytes of other members are written concurrently: word atomics
            atomicOr((unsigned int*)(cf + (a & ~3)), sb << (8 * (a & 3)));
    }
    __syncthreads();
    stamp(14);
#pragma unroll
    for (int j = 0; j < K; ++j)
        if (my[j].mode == kWFallback) block_topM(ck, cid, cf, n, A[j], S[j], M[j], hist, bs[j], warp_tot);
}
enum : uint8_t { kCand = 1, kSem = 2, kGs = 4, kNew = 8, kTake = 16 };

__global__ void __launch_bounds__(kUnionThreads, 1)
union_kernel(int V, const int32_t* __restrict__ static_ids, int n_static,
             const int32_t* __restrict__ seeds, int n_seed,
             const double* __restrict__ cand_s, const int32_t* __restrict__ cand_id,
             const int* __restrict__ n_cand_dev, int cap, int n_sem,
             const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
             const int32_t* __restrict__ ctx_sel, const int* __restrict__ n_ctx_sel_dev,
             int n_graph_sem_seeds, int per_seed, int n_dyn, int R, int r,
             int32_t* __restrict__ out_ids, int32_t* __restrict__ out_n,
             int32_t* __restrict__ out_local, int32_t* __restrict__ out_local_n,
             int32_t* __restrict__ sem_out, int* __restrict__ sem_out_n, int debug, int* flags,
             long long* __restrict__ trace, const int32_t* __restrict__ dyn_base, uint32_t* __restrict__ clear_hist,
             uint32_t* __restrict__ emit_bits, uint32_t* __restrict__ sbits, int32_t* __restrict__ early_ids,
             int* __restrict__ early_flag) {
    extern __shared__ __align__(16) unsigned char u_sm[];
    const int nwords = (V + 31) / 32;
    uint64_t* ck = (uint64_t*)u_sm;                          // [cap]
    int32_t* cid = (int32_t*)(ck + cap);                     // [cap]
    uint32_t* bits = (uint32_t*)(cid + cap);                 // [nwords]
    int32_t* G = (int32_t*)(bits + nwords);                  // [kMaxG]
    int32_t* goff = G + kMaxG;                               // [kMaxG + 1]
    int32_t* gs = goff + kMaxG + 1;                          // [kMaxG] ordered S_sem prefix
    int32_t* graph = gs + kMaxG;                             // [kMaxG * per_seed]
    uint8_t* cf = (uint8_t*)(graph + kMaxG * per_seed);      // [cap]
    __shared__ int warp_tot[3 * 33];
    __shared__ __align__(16) uint32_t hist[3 * kSelBins];
    __shared__ BSel bsel[3];
    __shared__ WSel wsel[3];
    __shared__ int nG_s, bad_s, taken_s, ngs_s, sem_n_s, early_n_s;

    const int tid = threadIdx.x, lane = lane_id(), T = blockDim.x;
    // (the finalisation after the LM head resets the early-list flag; cleared here too,
    // ahead of the trigger, in case a step ended without it)
    if (early_flag && tid == 0) *(volatile int*)early_flag = 0;
    pdl_trigger();
    if (trace) { if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[0] = t_; } }
    if (tid == 0) { bad_s = 0; sem_n_s = 0; early_n_s = 0; }
    const unsigned lt_mask = (1u << lane) - 1u;
    // rec: the new members' ids at their formation positions (the seeds, for the early list)
    auto walk = [&](const int32_t* src, int len, int taken, int32_t* rec) -> int {
        for (int base = 0; base < len && taken < n_dyn; base += 32) {
            const int idx = base + lane;
            int32_t c = idx < len ? src[idx] : -1;
            const bool valid = c >= 0 && c < V;
            if (idx < len && !valid) bad_s = 1;
            if (!valid) c = -1 - lane;            // distinct non-matching sentinel
            const unsigned peers = __match_any_sync(0xffffffffu, c);
            const bool first = valid && ((__ffs(peers) - 1) == lane);
            const bool cand = first && !((bits[c < 0 ? 0 : (c >> 5)] >> (c & 31)) & 1u);
            const unsigned bal = __ballot_sync(0xffffffffu, cand);
            const int bf = __popc(bal & lt_mask);
            if (cand && taken + bf < n_dyn) {
                atomicOr(&bits[c >> 5], 1u << (c & 31));
                if (rec) rec[taken + bf] = c;
            }
            taken += min(__popc(bal), n_dyn - taken);
            __syncwarp();
        }
        return taken;
    };
    pdl_wait();
    if (trace) { if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[40] = t_; } }
    // 1. static members: the bitmap static_bits_kernel built ahead of the scan (an
    //    earlier kernel on the stream: complete once the predecessor is)
    {
        const uint4* s4 = (const uint4*)sbits;
        uint4* b4 = (uint4*)bits;
        const int n4 = nwords >> 2;
        for (int w = tid; w < n4; w += T) b4[w] = __ldcg(&s4[w]);
        for (int w = (n4 << 2) + tid; w < nwords; w += T) bits[w] = __ldcg(&sbits[w]);
    }
    __syncthreads();
    if (trace) { if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[41] = t_; } }
    // formation starts with the seeds (C6): warp 0 walks them
    if (warp_id() == 0) {
        const int t = walk(seeds, n_seed, 0, early_ids);
        if (lane == 0) taken_s = t;
    }
    // the selection has consumed the scan's histogram: leave it zero for the next build
    if (clear_hist)
        for (int i = tid; i < kHistBins; i += T) clear_hist[i] = 0;
    const int n_cand_raw = *n_cand_dev;
    const int n_cand = min(n_cand_raw, cap);
    __syncthreads();   // the seeds walk (warp 0) has set its bits: kNew is decided while loading
    if (trace) { if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[42] = t_; } }
    // per-thread statistics of the three selections below (count, key range), gathered
    // while loading: kCand (selections 0 and 2) and kNew (selection 1)
    int st_c[2] = {0, 0};
    uint64_t st_lo[2] = {~0ull, ~0ull}, st_hi[2] = {0ull, 0ull};
    for (int i0 = 0; i0 < n_cand; i0 += 4 * T) {           // 4 independent loads in flight
        double sv[4];
        int32_t iv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * T + tid;
            sv[u] = i < n_cand ? __ldcg(&cand_s[i]) : 0.0;
            iv[u] = i < n_cand ? __ldcg(&cand_id[i]) : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int i = i0 + u * T + tid;
            if (i >= n_cand) continue;
            const uint64_t key = double_key(sv[u]);
            ck[i] = key;
            cid[i] = iv[u];
            uint8_t f = 0;
            if (iv[u] >= 0 && iv[u] < V) {
                f = kCand;
                ++st_c[0]; st_lo[0] = min(st_lo[0], key); st_hi[0] = max(st_hi[0], key);
                if (!((bits[iv[u] >> 5] >> (iv[u] & 31)) & 1u)) {   // not static, not a seed
                    f |= kNew;
                    ++st_c[1]; st_lo[1] = min(st_lo[1], key); st_hi[1] = max(st_hi[1], key);
                }
            }
            cf[i] = f;
        }
    }
    if (trace) { if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[43] = t_; } }
    __syncthreads();
    if (trace) { __syncthreads(); if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[1] = t_; } }
    // 2.-3. three exact selections in one set of radix passes (block_topM_multi):
    //   S_sem      = the n_sem best candidates                          (kSem)
    //   T_b        = the `budget` best NEW candidates (not static, not a seed) (kTake)
    //   S_sem[:ngs] = the ngs best candidates (graph seeds, ordered below) (kGs)
    // The new members of S_sem are a prefix of the new candidates in (key desc,
    // id asc) order, so "the first `budget` new ids of S_sem in S_sem order"
    // (the formation's semantic part) is T_b intersected with S_sem.
    const int taken0 = taken_s;
    const int budget = n_dyn - taken0;
    const int ngs = min(n_graph_sem_seeds, min(n_sem, kMaxG));
    if (tid == 0) ngs_s = 0;
    __syncthreads();
    {
        const uint8_t A[3] = {kCand, kNew, kCand};
        const uint8_t S[3] = {kSem, kTake, kGs};
        const int M[3] = {n_sem, budget, ngs};
        const int pc[3] = {st_c[0], st_c[1], st_c[0]};
        const uint64_t plo[3] = {st_lo[0], st_lo[1], st_lo[0]}, phi[3] = {st_hi[0], st_hi[1], st_hi[0]};
        block_topM_multi<3>(ck, cid, cf, n_cand, A, S, M, hist, wsel, bsel, warp_tot, trace ? trace + 24 : nullptr, pc, plo,
                            phi);
        if (trace && tid == 0) trace[23] = n_cand;   // (stamps 24..39: the selection's phases)
    }
    // the formation's semantic part (step 5 below): T_b ∩ S_sem, the new members of S_sem
    // in S_sem order up to the budget, marked in the bitmap. Two-list draft step
    // (early_flag, lmh_tc.cu): also appended after the new seeds to early_ids; when the
    // seeds and the semantic part fill the budget, the graph and context walks add
    // nothing and the dynamic list is complete now -- its length is published (release)
    // ahead of the sorted list that follows at the kernel's end; otherwise the head is
    // told to wait for the end (flag -1)
    int c_take = 0;
    for (int base = 0; base < n_cand; base += T) {
        const int i = base + tid;
        const bool in = i < n_cand && (cf[i] & kTake) && (cf[i] & kSem);
        if (in) { atomicOr(&bits[cid[i] >> 5], 1u << (cid[i] & 31)); ++c_take; }
        if (early_flag) {
            const unsigned m = __ballot_sync(0xffffffffu, in);
            int o = 0;
            if (lane == 0 && m) o = atomicAdd(&early_n_s, __popc(m));
            o = __shfl_sync(0xffffffffu, o, 0) + __popc(m & lt_mask);
            if (in) early_ids[taken0 + o] = cid[i];
        }
    }
    if (early_flag) __threadfence();
    const int took = block_count(c_take, warp_tot);   // (syncs: every append fenced before the flag)
    if (early_flag && tid == 0) {
        const int f = taken0 + took >= n_dyn ? taken0 + took + 1 : -1;
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(early_flag), "r"(f) : "memory");
    }
    if (sem_out) {
        for (int base = 0; base < n_cand; base += T) {      // one smem atomic per warp
            const int i = base + tid;
            const bool in = i < n_cand && (cf[i] & kSem);
            const unsigned m = __ballot_sync(0xffffffffu, in);
            int o = 0;
            if (lane == 0 && m) o = atomicAdd(&sem_n_s, __popc(m));
            o = __shfl_sync(0xffffffffu, o, 0) + __popc(m & ((1u << lane) - 1u));
            if (in) sem_out[o] = cid[i];
        }
    }
    if (trace) { __syncthreads(); if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[2] = t_; } }
    // the ngs graph seeds in S_sem order: gathered, ranked exactly by counting
    for (int i = tid; i < n_cand; i += T)
        if (cf[i] & kGs) {
            const int slot = atomicAdd(&ngs_s, 1);
            if (slot < kMaxG) graph[slot] = i;      // graph[] as scratch: candidate index
        }
    __syncthreads();
    const int ngs_pool = min(ngs_s, kMaxG);
    for (int a2 = tid; a2 < ngs_pool; a2 += T) {
        const int ia = graph[a2];
        int rank = 0;
        for (int b2 = 0; b2 < ngs_pool; ++b2) {
            const int ib = graph[b2];
            rank += before(ck[ib], cid[ib], ck[ia], cid[ia]) ? 1 : 0;   // (key desc, id asc)
        }
        if (rank < ngs) gs[rank] = cid[ia];
    }
    const int ngs_found = min(ngs, ngs_pool);
    __syncthreads();
    if (trace) { __syncthreads(); if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[3] = t_; } }
    // 4. G = dedupe(seeds ++ S_sem[:ngs]) and S_graph (warp 0)
    if (warp_id() == 0) {
        const int nc = min(n_seed + ngs_found, kMaxG);
        for (int i = lane; i < nc; i += 32) {
            int32_t g = i < n_seed ? seeds[i] : gs[i - n_seed];
            if (g < 0 || g >= V) { bad_s = 1; g = -1; }
            graph[i] = g;
        }
        __syncwarp();
        int nG = 0;
        for (int base = 0; base < nc; base += 32) {
            const int i = base + lane;
            const int32_t g = i < nc ? graph[i] : -1;
            bool keep = g >= 0;
            for (int j = 0; j < i && keep; ++j) keep = graph[j] != g;   // first occurrence
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) G[nG + __popc(bal & ((1u << lane) - 1u))] = g;
            nG += __popc(bal);
        }
        __syncwarp();
        int carry = 0;
        for (int base = 0; base < nG; base += 32) {
            const int j = base + lane;
            int c = 0;
            if (j < nG && row_ptr) c = min(row_ptr[G[j] + 1] - row_ptr[G[j]], per_seed);
            int inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            if (j < nG) goff[j] = carry + inc - c;
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) { goff[nG] = carry; nG_s = nG; }
    }
    __syncthreads();
    const int nG = nG_s;
    const int n_graph = goff[nG];
    if (row_ptr)
        for (int j = warp_id(); j < nG; j += T / 32) {
            const int cnt = goff[j + 1] - goff[j];
            const int base = row_ptr[G[j]];
            for (int e = lane; e < cnt; e += 32) graph[goff[j] + e] = col[base + e];
        }
    __syncthreads();

    if (trace) { __syncthreads(); if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[4] = t_; } }
    // dynamic-list mode: this thread's static words of its compaction range (below),
    // loaded now so their round trip overlaps the formation
    const int w0 = (int)((long long)nwords * tid / T), w1 = (int)((long long)nwords * (tid + 1) / T);
    const bool sreg = dyn_base && !emit_bits && nwords <= 8 * T;   // (w1 - w0 <= 8)
    uint32_t sw[8];
    const int base_pre = sreg ? *dyn_base : 0;
    if (sreg) {
#pragma unroll
        for (int j = 0; j < 8; ++j) sw[j] = w0 + j < w1 ? __ldcg(&sbits[w0 + j]) : 0u;
    }
    // 5. formation: seeds ++ S_sem ++ S_graph ++ S_ctx, first occurrence, skip
    //    members (static or taken), stop at N_dyn. The seeds were walked before
    //    the wait; the S_sem part is T_b and S_sem (selected above); graph and
    //    ctx are walked by warp 0 in 32-wide windows.
    // (T_b ∩ S_sem was marked above)
    if (warp_id() == 0) {
        const int n_ctx_sel = ctx_sel ? *n_ctx_sel_dev : 0;
        int t = taken0 + took;
        if (t < n_dyn) t = walk(graph, n_graph, t, nullptr);
        if (t < n_dyn) t = walk(ctx_sel, n_ctx_sel, t, nullptr);
    }
    __syncthreads();

    if (trace) { __syncthreads(); if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[5] = t_; } }
    // batched mode (dyn_base != null): the output is the sorted DYNAMIC list only,
    // written at out_ids + *dyn_base, and *out_n = *dyn_base + its length
    // (out_n = offsets + b + 1 for sequence b, dyn_base = offsets + b)
    int base_off = 0;
    if (sreg) {   // own words only (the compaction below reads only its own range): no barrier
        base_off = base_pre;
        out_ids += base_off;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (w0 + j < w1) { bits[w0 + j] &= ~sw[j]; sbits[w0 + j] = 0; }
    } else {
        if (dyn_base) {
            for (int w = tid; w < nwords; w += T) bits[w] &= ~__ldcg(&sbits[w]);
            base_off = *dyn_base;
            out_ids += base_off;
        }
        // the static bitmap is consumed: leave it zero for the next build's static_bits_kernel
        for (int w = tid; w < nwords; w += T) sbits[w] = 0;
        __syncthreads();
    }
    if (emit_bits) {
        // single shard, full output: the sorted ids are written by the multi-CTA
        // emit kernel from the bitmap (union_emit_kernel)
        for (int w = tid; w < nwords; w += T) emit_bits[w] = bits[w];
        if (tid == 0) {
            if (sem_out_n) *sem_out_n = sem_n_s;
            if (bad_s) atomicOr(flags, kFlagBadIds);
            if (n_cand_raw > cap) atomicOr(flags, kFlagSelectOverflow);
        }
        if (trace) { __syncthreads(); if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[6] = t_; } }
        return;
    }
    // 6. compaction. Thread t owns words [t*nwords/T, (t+1)*nwords/T); a block
    //    scan of the popcounts gives each thread's output offset. The sorted
    //    ids are staged in shared memory (the candidate arrays are dead by now)
    //    and copied out coalesced; the shard slice (v mod R == r) is filtered
    //    from the staged copy. Outputs larger than the staging area fall back to
    //    direct per-thread stores.
    int cnt = 0;
    for (int w = w0; w < w1; ++w) cnt += __popc(bits[w]);
    int total = 0, total_local = 0;
    int off = block_excl_scan(cnt, warp_tot, total);
    int32_t* stage = (int32_t*)u_sm;                          // aliases ck/cid: 3*cap int32
    // (a dynamic list alone -- a few thousand ids -- goes straight out: each thread's ids
    // are contiguous and follow its left neighbour's, no staging barrier)
    const bool staged = total <= 3 * cap && !(sreg && !out_local);
    int32_t* dst = staged ? stage : out_ids;
    for (int w = w0; w < w1; ++w)
        for (uint32_t bb = bits[w]; bb; bb &= bb - 1) dst[off++] = w * 32 + __ffs(bb) - 1;
    if (staged || out_local) __syncthreads();
    if (staged)
        for (int i = tid; i < total; i += T) out_ids[i] = stage[i];
    if (out_local) {
        if (R == 1) {
            if (staged)
                for (int i = tid; i < total; i += T) out_local[i] = stage[i];
            else
                for (int i = tid; i < total; i += T) out_local[i] = out_ids[i];   // own writes: visible after the sync
            total_local = total;
        } else {
            const int32_t* srcv = staged ? stage : out_ids;
            const int i0 = (int)((long long)total * tid / T), i1 = (int)((long long)total * (tid + 1) / T);
            int cl = 0;
            for (int i = i0; i < i1; ++i) cl += (srcv[i] % R) == r;
            int offl = block_excl_scan(cl, warp_tot, total_local);
            for (int i = i0; i < i1; ++i)
                if ((srcv[i] % R) == r) out_local[offl++] = srcv[i];
        }
    }
    if (tid == 0) {
        *out_n = base_off + total;
        if (out_local_n) *out_local_n = total_local;
        if (sem_out_n) *sem_out_n = sem_n_s;
        if (bad_s) atomicOr(flags, kFlagBadIds);
        if (total > (dyn_base ? 0 : n_static) + n_dyn) atomicOr(flags, kFlagBudget);
        if (n_cand_raw > cap) atomicOr(flags, kFlagSelectOverflow);
    }
    if (trace) { __syncthreads(); if (threadIdx.x == 0) { long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); trace[6] = t_; } }
}

// Sorted ids from the union bitmap, 32 words (1024 ids) per CTA: a CTA's
// output offset is the popcount of all words before its chunk (each CTA sums
// them from L2 itself: no inter-CTA chain), warp 0 scans its 32 words and
// writes the ids. The last CTA writes n_S and the budget check.
constexpr int kEmitThreads = 128;

__global__ void __launch_bounds__(kEmitThreads)
union_emit_kernel(const uint32_t* __restrict__ bits, int nwords, int32_t* __restrict__ out_ids,
                  int32_t* __restrict__ out_n, int32_t* __restrict__ out_local, int32_t* __restrict__ out_local_n,
                  int budget_max, int* flags) {
    pdl_trigger();
    pdl_wait();
    __shared__ int wsum[kEmitThreads / 32];
    const int tid = threadIdx.x, lane = lane_id(), warp = warp_id();
    const int w0 = blockIdx.x * 32, w1 = min(nwords, w0 + 32);
    int c = 0;
#pragma unroll 4
    for (int w = tid; w < w0; w += kEmitThreads) c += __popc(__ldcg(&bits[w]));
    c = warp_sum_i(c);
    if (lane == 0) wsum[warp] = c;
    __syncthreads();
    if (warp != 0) return;
    int prefix = 0;
#pragma unroll
    for (int i = 0; i < kEmitThreads / 32; ++i) prefix += wsum[i];
    const int w = w0 + lane;
    const uint32_t x = w < w1 ? __ldcg(&bits[w]) : 0u;
    const int pc = __popc(x);
    int inc = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    int off = prefix + inc - pc;
    for (uint32_t bb = x; bb; bb &= bb - 1) {
        const int32_t id = w * 32 + __ffs(bb) - 1;
        out_ids[off] = id;
        if (out_local) out_local[off] = id;
        ++off;
    }
    if (blockIdx.x == gridDim.x - 1 && lane == 31) {
        const int total = prefix + inc;
        *out_n = total;
        if (out_local_n) *out_local_n = total;
        if (total > budget_max) atomicOr(flags, kFlagBudget);
    }
}

void launch_union_emit(const uint32_t* bits, int V, int32_t* out_ids, int32_t* out_n, int32_t* out_local,
                       int32_t* out_local_n, int budget_max, int* flags, cudaStream_t st) {
    const int nwords = (V + 31) / 32;
    launch_pdl(union_emit_kernel, dim3((nwords + 31) / 32), dim3(kEmitThreads), 0, st, bits, nwords, out_ids, out_n,
               out_local, out_local_n, budget_max, flags);
}

static size_t union_fixed_bytes(int V, int per_seed) {
    const int nwords = (V + 31) / 32;
    return (size_t)nwords * 4 + (size_t)(3 * kMaxG + 1) * 4 + (size_t)kMaxG * per_seed * 4 + 64;
}

// Largest candidate superset the union kernel can hold in shared memory.
int union_cand_cap(int V, int per_seed) {
    const size_t budget = 212 * 1024;   // + ~12.6 KB static (three selection histograms)
    const size_t fixed = union_fixed_bytes(V, per_seed);
    if (fixed >= budget) return 0;
    return (int)((budget - fixed) / 13) & ~15;
}

void launch_union(int V, const int32_t* static_ids, int n_static, const int32_t* seeds, int n_seed,
                  const double* cand_s, const int32_t* cand_id, const int* n_cand_dev, int cap, int n_sem,
                  const int32_t* row_ptr, const int32_t* col,
                  const int32_t* ctx_sel, const int* n_ctx_sel_dev,
                  int n_graph_sem_seeds, int per_seed, int n_dyn, int R, int r,
                  int32_t* out_ids, int32_t* out_n, int32_t* out_local, int32_t* out_local_n,
                  int32_t* sem_out, int* sem_out_n, int debug, int* flags, cudaStream_t st, long long* trace,
                  const int32_t* dyn_base, uint32_t* clear_hist, uint32_t* emit_bits, uint32_t* sbits,
                  int32_t* early_ids, int* early_flag) {
    const size_t smem = (size_t)cap * 13 + union_fixed_bytes(V, per_seed) + 16;
    cudaFuncSetAttribute(union_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    launch_pdl(union_kernel, dim3(1), dim3(kUnionThreads), smem, st, V, static_ids, n_static, seeds, n_seed, cand_s, cand_id, n_cand_dev,
                                                  cap, n_sem, row_ptr, col, ctx_sel, n_ctx_sel_dev, n_graph_sem_seeds,
                                                  per_seed, n_dyn, R, r, out_ids, out_n, out_local, out_local_n,
                                                  sem_out, sem_out_n, debug, flags, trace, dyn_base, clear_hist, emit_bits,
                                                  sbits, early_ids, early_flag);
}

// a4 static core -> the V-bit membership bitmap the union starts from (sbits: zero
// on entry -- the union kernel zeroes it after use). Launched ahead of the scan,
// which overlaps it (PDL) and waits for it before completing. Range-checked (and,
// with debug, order-checked) like the union's own inputs.
__global__ void __launch_bounds__(256)
static_bits_kernel(const int32_t* __restrict__ static_ids, int n_static, int V, int debug,
                   uint32_t* __restrict__ sbits, int* __restrict__ flags) {
    pdl_trigger();
    bool bad = false;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_static; i += gridDim.x * blockDim.x) {
        const int32_t v = __ldg(&static_ids[i]);
        if (v < 0 || v >= V) { bad = true; continue; }
        if (debug && i > 0 && __ldg(&static_ids[i - 1]) >= v) bad = true;
        atomicOr(&sbits[v >> 5], 1u << (v & 31));
    }
    if (bad && flags) atomicOr(flags, kFlagBadIds);
}

void launch_static_bits(const int32_t* static_ids, int n_static, int V, int debug, uint32_t* sbits, int* flags,
                        cudaStream_t st) {
    const int grid = std::max(1, std::min(32, (n_static + 1023) / 1024));
    static_bits_kernel<<<grid, 256, 0, st>>>(static_ids, n_static, V, debug, sbits, flags);
}

}  // namespace es
