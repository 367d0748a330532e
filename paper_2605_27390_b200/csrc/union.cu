// union.cu -- a3/a4: statistical expansion, runtime candidate formation,
// budget cap and the sorted union  V_t = V_static u dyn  (Eq. vocab_union
// P:88-93; formation App. A.3; budget |V_t \ V_static| <= N_dyn,
// Eq. optimization; cap order S:260; readings C4-C9).
//
// One CTA: the candidate list is at most a few thousand ids and the answer
// is a V-bit membership bitmap in shared memory (16 KB at V = 128k), so a
// single SM does the whole step in a few microseconds:
//   1. static ids -> bitmap;
//   2. G = dedupe(seeds ++ S_sem[:n_graph_sem_seeds]); S_graph = the first
//      per_seed CSR successors of each g in G, in G order;
//   3. one warp walks  seeds ++ S_sem ++ S_graph ++ S_ctx  32 ids at a time:
//      an id is taken iff it is not yet a member (static or already taken)
//      and is the first occurrence inside its 32-wide window (match.any),
//      until N_dyn ids are taken -- exactly the sequential first-occurrence
//      walk of the definition;
//   4. block-wide popcount scan of the bitmap writes the sorted ids (and this
//      shard's slice v mod R == r).
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
__global__ void __launch_bounds__(kUnionThreads, 1)
union_kernel(int V, const int32_t* __restrict__ static_ids, int n_static,
             const int32_t* __restrict__ seeds, int n_seed,
             const int32_t* __restrict__ sem, const int* __restrict__ n_sem_dev, int n_sem_max,
             const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
             const int32_t* __restrict__ ctx_sel, const int* __restrict__ n_ctx_sel_dev,
             int n_graph_sem_seeds, int per_seed, int n_dyn, int R, int r,
             int32_t* __restrict__ out_ids, int32_t* __restrict__ out_n,
             int32_t* __restrict__ out_local, int32_t* __restrict__ out_local_n,
             int debug, int* flags) {
    extern __shared__ unsigned char u_sm[];
    const int nwords = (V + 31) / 32;
    uint32_t* bits = (uint32_t*)u_sm;                       // [nwords]
    int32_t* G = (int32_t*)(bits + nwords);                  // [kMaxG]
    int32_t* goff = G + kMaxG;                               // [kMaxG + 1]
    int32_t* graph = goff + kMaxG + 1;                       // [kMaxG * per_seed]
    __shared__ int warp_tot[33];
    __shared__ int nG_s, bad_s, taken_s;

    const int tid = threadIdx.x, lane = lane_id();
    for (int w = tid; w < nwords; w += blockDim.x) bits[w] = 0;
    if (tid == 0) bad_s = 0;
    __syncthreads();
    // 1. static members
    for (int i0 = 0; i0 < n_static; i0 += 8 * blockDim.x) {   // 8 independent loads in flight
        int32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x + tid;
            v[u] = i < n_static ? __ldg(&static_ids[i]) : -1;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = i0 + u * blockDim.x + tid;
            if (i >= n_static) continue;
            if (v[u] < 0 || v[u] >= V) { bad_s = 1; continue; }
            if (debug && i > 0 && static_ids[i - 1] >= v[u]) bad_s = 1;
            atomicOr(&bits[v[u] >> 5], 1u << (v[u] & 31));
        }
    }
    const int n_sem = min(*n_sem_dev, n_sem_max);
    const int n_ctx_sel = ctx_sel ? *n_ctx_sel_dev : 0;
    // 2. graph seeds G = dedupe(seeds ++ S_sem[:ngs]) and S_graph, warp 0 in parallel
    if (warp_id() == 0) {
        const int ngs = min(n_graph_sem_seeds, n_sem);
        const int nc = min(n_seed + ngs, kMaxG);
        for (int i = lane; i < nc; i += 32) {          // candidates -> graph[] as scratch
            int32_t g = i < n_seed ? seeds[i] : sem[i - n_seed];
            if (g < 0 || g >= V) { bad_s = 1; g = -1; }
            graph[i] = g;
        }
        __syncwarp();
        int nG = 0;
        for (int base = 0; base < nc; base += 32) {
            const int i = base + lane;
            int32_t g = i < nc ? graph[i] : -1;
            bool keep = g >= 0;
            for (int j = 0; j < i && keep; ++j) keep = graph[j] != g;   // first occurrence
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) G[nG + __popc(bal & ((1u << lane) - 1u))] = g;
            nG += __popc(bal);
        }
        __syncwarp();
        // degrees and offsets (exclusive scan of min(deg, per_seed))
        int carry = 0;
        for (int base = 0; base < nG; base += 32) {
            const int j = base + lane;
            int c = 0;
            if (j < nG && row_ptr) c = min(row_ptr[G[j] + 1] - row_ptr[G[j]], per_seed);
            int inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int t = __shfl_up_sync(0xffffffffu, inc, o);
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
        for (int j = warp_id(); j < nG; j += blockDim.x / 32) {
            const int cnt = goff[j + 1] - goff[j];
            const int base = row_ptr[G[j]];
            for (int e = lane; e < cnt; e += 32) graph[goff[j] + e] = col[base + e];
        }
    __syncthreads();

    // 3. formation: seeds ++ S_sem ++ S_graph ++ S_ctx, first occurrence, skip
    //    members, stop at N_dyn. Seeds, graph and ctx are walked by warp 0 in
    //    32-wide windows; S_sem (distinct ids by construction) is taken in
    //    parallel with a block-wide order-preserving scan.
    const unsigned lt_mask = (1u << lane) - 1u;
    auto walk = [&](const int32_t* src, int len, int taken) -> int {
        for (int base = 0; base < len && taken < n_dyn; base += 32) {
            const int idx = base + lane;
            int32_t c = idx < len ? src[idx] : -1;
            bool valid = c >= 0 && c < V;
            if (idx < len && !valid) bad_s = 1;
            if (!valid) c = -1 - lane;            // distinct non-matching sentinel
            const unsigned peers = __match_any_sync(0xffffffffu, c);
            const bool first = valid && ((__ffs(peers) - 1) == lane);
            const bool cand = first && !((bits[c < 0 ? 0 : (c >> 5)] >> (c & 31)) & 1u);
            const unsigned bal = __ballot_sync(0xffffffffu, cand);
            const int before = __popc(bal & lt_mask);
            if (cand && taken + before < n_dyn) atomicOr(&bits[c >> 5], 1u << (c & 31));
            taken += min(__popc(bal), n_dyn - taken);
            __syncwarp();
        }
        return taken;
    };
    if (warp_id() == 0) {
        const int t = walk(seeds, n_seed, 0);
        if (lane == 0) taken_s = t;
    }
    __syncthreads();
    {
        const int taken0 = taken_s;
        const int T = blockDim.x;
        const int i0 = (int)((long long)n_sem * tid / T), i1 = (int)((long long)n_sem * (tid + 1) / T);
        // each thread owns <= kSemPerThread consecutive S_sem entries, loaded once
        constexpr int kSemPerThread = 16;
        int32_t cv[kSemPerThread];
        unsigned newm = 0;
#pragma unroll
        for (int u = 0; u < kSemPerThread; ++u) cv[u] = (i0 + u < i1) ? __ldg(&sem[i0 + u]) : -1;
        int cnt = 0;
#pragma unroll
        for (int u = 0; u < kSemPerThread; ++u) {
            const int32_t c = cv[u];
            const bool nw = c >= 0 && c < V && !((bits[c >> 5] >> (c & 31)) & 1u);
            newm |= (unsigned)nw << u;
            cnt += nw;
        }
        int total = 0;
        int off = block_excl_scan(cnt, warp_tot, total);   // contains __syncthreads
        const int budget = n_dyn - taken0;
#pragma unroll
        for (int u = 0; u < kSemPerThread; ++u) {
            if (((newm >> u) & 1u) && off < budget) {
                atomicOr(&bits[cv[u] >> 5], 1u << (cv[u] & 31));
                ++off;
            }
        }
        __syncthreads();
        if (tid == 0) taken_s = taken0 + min(total, budget);
    }
    __syncthreads();
    if (warp_id() == 0 && taken_s < n_dyn) {
        int t = walk(graph, n_graph, taken_s);
        t = walk(ctx_sel, n_ctx_sel, t);
    }
    __syncthreads();

    // 4. compaction: thread t owns words [t*nwords/T, (t+1)*nwords/T)
    const int T = blockDim.x;
    const int w0 = (int)((long long)nwords * tid / T), w1 = (int)((long long)nwords * (tid + 1) / T);
    int cnt = 0, cnt_local = 0;
    for (int w = w0; w < w1; ++w) {
        uint32_t b = bits[w];
        cnt += __popc(b);
        if (R > 1)
            while (b) { int bit = __ffs(b) - 1; b &= b - 1; cnt_local += ((w * 32 + bit) % R) == r; }
    }
    if (R == 1) cnt_local = cnt;
    int total = 0, total_local = 0;
    int off = block_excl_scan(cnt, warp_tot, total);
    int off_local = block_excl_scan(cnt_local, warp_tot, total_local);
    for (int w = w0; w < w1; ++w) {
        uint32_t b = bits[w];
        while (b) {
            int bit = __ffs(b) - 1;
            b &= b - 1;
            int v = w * 32 + bit;
            out_ids[off++] = v;
            if (out_local && (R == 1 || v % R == r)) out_local[off_local++] = v;
        }
    }
    if (tid == 0) {
        *out_n = total;
        if (out_local_n) *out_local_n = total_local;
        if (bad_s) atomicOr(flags, kFlagBadIds);
        if (total > n_static + n_dyn) atomicOr(flags, kFlagBudget);
    }
}

void launch_union(int V, const int32_t* static_ids, int n_static, const int32_t* seeds, int n_seed,
                  const int32_t* sem_sorted, const int* n_sem_dev, int n_sem_max,
                  const int32_t* row_ptr, const int32_t* col,
                  const int32_t* ctx_sel, const int* n_ctx_sel_dev,
                  int n_graph_sem_seeds, int per_seed, int n_dyn, int R, int r,
                  int32_t* out_ids, int32_t* out_n, int32_t* out_local, int32_t* out_local_n,
                  int debug, int* flags, cudaStream_t st) {
    const int nwords = (V + 31) / 32;
    size_t smem = (size_t)nwords * 4 + (size_t)(2 * kMaxG + 1) * 4 + (size_t)kMaxG * per_seed * 4;
    cudaFuncSetAttribute(union_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    union_kernel<<<1, kUnionThreads, smem, st>>>(V, static_ids, n_static, seeds, n_seed, sem_sorted,
                                                  n_sem_dev, n_sem_max, row_ptr, col, ctx_sel, n_ctx_sel_dev,
                                                  n_graph_sem_seeds, per_seed, n_dyn, R, r, out_ids, out_n,
                                                  out_local, out_local_n, debug, flags);
}

}  // namespace es
