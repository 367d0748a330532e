// verify.cu -- N2: lossless verification of a draft chain
// against the target, the rejection criterion alpha of P:42 (Leviathan et
// al.), the verify phase of alg. P:366-367, in the chain form and with the
// rule of SPEC S:380-385; greedy decoding (T = 0) is the paper's setting.
//
// Position j (0 <= j <= g) has the target distribution over the FULL
// vocabulary p_j(v) = exp(z_j[v] it - m_j) / s_j; the draft's restricted
// distribution q_j is draft_probs[j][i] at subset[i] and exactly 0 outside the
// subset (S:407 -- the residual max(0, p - q) re-covers the excluded tokens,
// which is what makes the restricted draft lossless).
//   greedy:   accept x_j while x_j == argmax p_j (ties: lower id); on a
//             mismatch emit argmax p_j; all accepted: the bonus argmax p_g;
//   sampling: accept x_j iff u_j < min(1, p_j(x_j) / q_j(x_j)); on the first
//             rejection emit the draw from normalize(max(0, p_j - q_j)) with
//             w_j; all accepted: the bonus drawn from p_g with w_g. A draw is
//             the smallest v (id order) whose running sum of the weights
//             exceeds w * (their total).
//
// Kernel 1 (verify_pos_kernel): a cluster of 8 CTAs per position (each a
// contiguous slice of V), every position at once (the first rejection is not
// known up front): max / argmax and the fp64 sum over V, combined over the
// cluster through distributed shared memory in rank order (every CTA holds the
// same values, so all take the same decisions); the acceptance test; for a
// rejected position (sampling) or the bonus position the draw -- per-thread
// residual mass over a contiguous id range (the q lookup walks the sorted
// subset from a binary-searched start), the CTA whose mass interval holds
// w * total, a block scan there, and the thread whose range holds it re-walks.
// The fp64 sums run in a different order than the oracle's sequential ones; a
// different token needs w * total within ~1e-15 relative of a CDF step.
// Kernel 2 (verify_decide_kernel, one warp): the accepted prefix and the
// emitted token. HBM-bound: (g + 1) rows of V fp32 logits, read from HBM once
// (the further passes hit L2).
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace es {

constexpr int kVerThreads = 1024;
constexpr int kVerWarps = kVerThreads / 32;
constexpr int kVerCluster = 8;   // CTAs per position (a portable cluster; DSMEM reductions)

struct VerSmem {
    double red_d[kVerWarps];
    double scan_d[kVerWarps + 1];
    float red_v[kVerWarps];
    int red_i[kVerWarps];
    double s_M, s_sum, s_tot;
    int s_arg, s_pick;
    double c_part;   // this CTA's partial, read by the cluster (DSMEM)
    float c_v;
    int c_i;
    int s_lb[2];     // the subset positions bounding this CTA's id slice
    int s_xi;        // the proposal's subset position
    int32_t s_cache[8192];   // the subset entries of this CTA's id slice (when they fit)
};
constexpr int kVerSCap = 8192;

ES_DEV double warp_sum_dd(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block sum of a double (all threads get it)
ES_DEV double block_sum_d(double v, VerSmem& sm) {
    const int lane = lane_id(), wid = warp_id();
    v = warp_sum_dd(v);
    if (lane == 0) sm.red_d[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double t = lane < kVerWarps ? sm.red_d[lane] : 0.0;
        t = warp_sum_dd(t);
        if (lane == 0) sm.s_tot = t;
    }
    __syncthreads();
    const double r = sm.s_tot;
    __syncthreads();
    return r;
}

// exclusive block scan of a double (thread order)
ES_DEV double block_excl_scan_d(double v, VerSmem& sm) {
    const int lane = lane_id(), wid = warp_id();
    double inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) sm.scan_d[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const double w = lane < kVerWarps ? sm.scan_d[lane] : 0.0;
        double wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < kVerWarps) sm.scan_d[lane] = wi - w;
    }
    __syncthreads();
    const double r = sm.scan_d[wid] + inc - v;
    __syncthreads();
    return r;
}

// first index i of the sorted S with S[i] >= v
ES_DEV int lower_bound_i32(const int32_t* S, int n, int v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(&S[mid]) < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// first index i of the sorted S with S[i] >= v, by one warp: a 32-ary search
// (log32 n dependent rounds of 32 parallel probes); every lane returns it
ES_DEV int warp_lower_bound(const int32_t* S, int n, int v) {
    const int lane = lane_id();
    int lo = 0, hi = n;
    while (hi - lo > 32) {
        const int step = (hi - lo + 31) / 32;
        const int p = lo + lane * step;
        const bool below = p < hi && __ldg(&S[p]) < v;
        const int k = __popc(__ballot_sync(0xffffffffu, below));   // probes below v (a prefix)
        if (k == 0) return lo;                                     // S[lo] >= v
        const int nlo = lo + (k - 1) * step + 1;
        hi = min(hi, lo + k * step + 1);
        lo = nlo;
    }
    const int p = lo + lane;
    const bool below = p < hi && __ldg(&S[p]) < v;
    return lo + __popc(__ballot_sync(0xffffffffu, below));
}

// r(v) = max(0, p(v) - q(v)) over [v0, v1), q from qj on S (qj == nullptr: q = 0);
// S entries [c_off, c_off + c_cnt) also in shared memory (cache, may be null)
struct Resid {
    const float* zj; double it, M, s;
    const int32_t* S; int n_S; const float* qj;
    const int32_t* cache = nullptr; int c_off = 0, c_cnt = 0;
    ES_DEV int32_t s_at(int i) const {
        const int o = i - c_off;
        return (cache && o >= 0 && o < c_cnt) ? cache[o] : __ldg(&S[i]);
    }
    ES_DEV double q_at(int v, int& i) const {
        if (!qj) return 0.0;
        while (i < n_S && s_at(i) < v) ++i;
        return (i < n_S && s_at(i) == v) ? (double)__ldg(&qj[i]) : 0.0;
    }
    ES_DEV double r_at(int v, int& i) const {
        const double p = exp((double)__ldg(&zj[v]) * it - M) / s;
        const double r = p - q_at(v, i);
        return r > 0.0 ? r : 0.0;
    }
};

// Cluster-wide reductions (kVerCluster CTAs per position, DSMEM): every CTA
// combines the CTA partials in rank order, so all of them hold identical
// values and take identical decisions.
ES_DEV double cluster_sum_d(double v, VerSmem& sm, cg::cluster_group& cl) {
    const double b = block_sum_d(v, sm);
    if (threadIdx.x == 0) sm.c_part = b;
    cl.sync();
    double t = 0.0;
#pragma unroll
    for (int r = 0; r < kVerCluster; ++r) t += *cl.map_shared_rank(&sm.c_part, r);
    cl.sync();
    return t;
}

// the draw from weights r over [0, V) with w in [0, 1), cluster-wide: each CTA
// holds a contiguous slice [c0, c1); the CTA whose mass interval (prefix in rank
// order) holds w * total finds the id by a block scan and one thread's re-walk.
// Returns -2 on every CTA if the total mass is 0, else the id on the picking
// CTA's thread 0 (-1 elsewhere).
ES_DEV int cluster_draw(const Resid& R0, int c0, int c1, double w, VerSmem& sm, cg::cluster_group& cl) {
    const int tid = threadIdx.x;
    const int n = c1 - c0;
    const int v0 = c0 + (int)((long long)n * tid / kVerThreads), v1 = c0 + (int)((long long)n * (tid + 1) / kVerThreads);
    Resid R = R0;
    int i0 = 0;
    if (R.qj) {
        // the subset entries of this CTA's id slice [c0, c1): bounds by two warps' 32-ary
        // searches, the entries staged in shared memory, each thread's start found there
        if (warp_id() < 2) {
            const int b = warp_lower_bound(R.S, R.n_S, warp_id() == 0 ? c0 : c1);
            if (lane_id() == 0) sm.s_lb[warp_id()] = b;
        }
        __syncthreads();
        const int lb0 = sm.s_lb[0], cnt = sm.s_lb[1] - lb0;
        if (cnt <= kVerSCap) {
            for (int i = tid; i < cnt; i += kVerThreads) sm.s_cache[i] = __ldg(&R.S[lb0 + i]);
            R.cache = sm.s_cache; R.c_off = lb0; R.c_cnt = cnt;
        }
        __syncthreads();
        if (R.cache) {
            int lo = 0, hi = cnt;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (sm.s_cache[mid] < v0) lo = mid + 1; else hi = mid;
            }
            i0 = lb0 + lo;
        } else {
            i0 = lower_bound_i32(R.S, R.n_S, v0);
        }
    }
    double loc = 0.0;
    int last = -1;
    {
        int i = i0;
        for (int v = v0; v < v1; ++v) {
            const double r = R.r_at(v, i);
            if (r > 0.0) { loc += r; last = v; }
        }
    }
    const double mine = block_sum_d(loc, sm);
    if (tid == 0) sm.c_part = mine;
    cl.sync();
    double masses[kVerCluster];
#pragma unroll
    for (int r = 0; r < kVerCluster; ++r) masses[r] = *cl.map_shared_rank(&sm.c_part, r);
    cl.sync();
    const int me = (int)cl.block_rank();
    double tot = 0.0, pre = 0.0;
    int last_rank = -1;
#pragma unroll
    for (int r = 0; r < kVerCluster; ++r) {
        if (r == me) pre = tot;
        tot += masses[r];
        if (masses[r] > 0.0) last_rank = r;
    }
    if (!(tot > 0.0)) return -2;
    const double target = w * tot;
    const bool pick = (mine > 0.0 && pre <= target && target < pre + mine) || (me == last_rank && target >= pre + mine);
    if (!pick) return -1;
    // this CTA: the thread whose mass interval holds the target re-walks its range
    const double tpre = pre + block_excl_scan_d(loc, sm);
    if (tid == 0) sm.s_pick = 0x7fffffff;
    __syncthreads();
    if (loc > 0.0 && tpre <= target && target < tpre + loc) atomicMin(&sm.s_pick, tid);
    __syncthreads();
    const bool none = sm.s_pick == 0x7fffffff;
    if (tid == 0) sm.s_arg = -1;
    __syncthreads();
    if (none) {
        if (last >= 0) atomicMax(&sm.s_arg, last);   // the rounding band above the CTA's mass
    } else if (tid == sm.s_pick) {
        double run = tpre;
        int i = i0, got = last;
        for (int v = v0; v < v1; ++v) {
            const double r = R.r_at(v, i);
            if (r > 0.0) {
                run += r;
                if (run > target) { got = v; break; }
            }
        }
        sm.s_arg = got;
    }
    __syncthreads();
    return sm.s_arg;
}

__global__ void __cluster_dims__(kVerCluster, 1, 1) __launch_bounds__(kVerThreads)
verify_pos_kernel(const float* __restrict__ z, int V, int g, const int32_t* __restrict__ x,
                  const int32_t* __restrict__ S, int n_S, const float* __restrict__ qS, double it, int greedy,
                  const double* __restrict__ u, const double* __restrict__ w, int32_t* __restrict__ pos_acc,
                  int32_t* __restrict__ pos_tok, int* flags) {
    __shared__ VerSmem sm;
    cg::cluster_group cl = cg::this_cluster();
    pdl_trigger();
    pdl_wait();
    const int j = blockIdx.x / kVerCluster, me = (int)cl.block_rank();
    const int tid = threadIdx.x, lane = lane_id(), wid = warp_id();
    const float* zj = z + (size_t)j * V;
    const int c0 = (int)((long long)V * me / kVerCluster), c1 = (int)((long long)V * (me + 1) / kVerCluster);
    const int n = c1 - c0;
    const int v0 = c0 + (int)((long long)n * tid / kVerThreads), v1 = c0 + (int)((long long)n * (tid + 1) / kVerThreads);
    // 1. maximum and argmax (value desc, id asc), in fp32 -- the fp64 product of an
    //    fp32 logit and it orders exactly as the logit itself (it > 0)
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int v = v0; v < v1; ++v) {
        const float zz = __ldg(&zj[v]);
        if (zz > bv) { bv = zz; bi = v; }
    }
    warp_argbest(bv, bi);
    if (lane == 0) { sm.red_v[wid] = bv; sm.red_i[wid] = bi; }
    __syncthreads();
    if (wid == 0) {
        float v = lane < kVerWarps ? sm.red_v[lane] : -INFINITY;
        int i = lane < kVerWarps ? sm.red_i[lane] : 0x7fffffff;
        warp_argbest(v, i);
        if (lane == 0) { sm.c_v = v; sm.c_i = i; }
    }
    cl.sync();
    float Mv = -INFINITY;
    int amax = 0x7fffffff;
#pragma unroll
    for (int r = 0; r < kVerCluster; ++r) {
        const float v = *cl.map_shared_rank(&sm.c_v, r);
        const int i = *cl.map_shared_rank(&sm.c_i, r);
        if (before(v, i, Mv, amax)) { Mv = v; amax = i; }
    }
    cl.sync();
    const double M = (double)Mv * it;
    if (greedy) {
        if (me == 0 && tid == 0) {
            pos_tok[j] = amax;
            pos_acc[j] = j < g ? (int)(__ldg(&x[j]) == amax) : 0;
        }
        return;
    }
    // the proposal's subset position: warp 0's 32-ary search, overlapping the sum below
    if (j < g && wid == 0) {
        const int xj = __ldg(&x[j]);
        const int i = (xj >= 0 && xj < V) ? warp_lower_bound(S, n_S, xj) : n_S;
        if (lane == 0) sm.s_xi = i;
    }
    // 2. s = sum_v exp(z it - M), fp64, cluster-wide
    double loc = 0.0;
    for (int v = v0; v < v1; ++v) loc += exp((double)__ldg(&zj[v]) * it - M);
    const double s = cluster_sum_d(loc, sm, cl);
    // 3. acceptance (j < g) or the bonus draw (j == g) -- identical on every CTA
    const float* qj = nullptr;
    if (j < g) {
        const int xj = __ldg(&x[j]);
        qj = qS + (size_t)j * n_S;
        const int i = sm.s_xi;   // (written before the block reductions of the sum: visible)
        const bool in = i < n_S && __ldg(&S[i]) == xj && __ldg(&qj[i]) > 0.0f;
        if (!in) {
            if (me == 0 && tid == 0) { atomicOr(flags, kFlagBadIds); pos_acc[j] = 0; pos_tok[j] = -1; }
            return;
        }
        double a = exp((double)__ldg(&zj[xj]) * it - M) / s / (double)__ldg(&qj[i]);
        if (a > 1.0) a = 1.0;
        if (__ldg(&u[j]) < a) {
            if (me == 0 && tid == 0) { pos_acc[j] = 1; pos_tok[j] = xj; }
            return;
        }
    }
    const Resid R{zj, it, M, s, S, n_S, j < g ? qj : nullptr};
    int tok = cluster_draw(R, c0, c1, __ldg(&w[j]), sm, cl);
    if (tok == -2) {   // no residual mass (rounding only): draw from p_j
        const Resid P{zj, it, M, s, S, n_S, nullptr};
        tok = cluster_draw(P, c0, c1, __ldg(&w[j]), sm, cl);
    }
    if (tok >= 0 && tid == 0) { pos_acc[j] = 0; pos_tok[j] = tok; }
}

__global__ void verify_decide_kernel(int g, const int32_t* __restrict__ x, const int32_t* __restrict__ pos_acc,
                                     const int32_t* __restrict__ pos_tok, int32_t* __restrict__ tokens,
                                     int32_t* __restrict__ n_acc_out) {
    pdl_wait();
    if (threadIdx.x != 0) return;
    int n = 0;
    while (n < g && pos_acc[n]) { tokens[n] = x[n]; ++n; }
    tokens[n] = pos_tok[n];
    for (int j = n + 1; j <= g; ++j) tokens[j] = -1;
    *n_acc_out = n;
}

void launch_verify(const float* z, int V, int g, const int32_t* x, const int32_t* S, int n_S, const float* qS,
                   double it, int greedy, const double* u, const double* w, int32_t* pos_acc, int32_t* pos_tok,
                   int32_t* tokens, int32_t* n_acc_out, int* flags, cudaStream_t st) {
    launch_pdl(verify_pos_kernel, dim3((g + 1) * kVerCluster), dim3(kVerThreads), 0, st, z, V, g, x, S, n_S, qS, it, greedy, u, w,
               pos_acc, pos_tok, flags);
    launch_pdl(verify_decide_kernel, dim3(1), dim3(32), 0, st, g, x, (const int32_t*)pos_acc,
               (const int32_t*)pos_tok, tokens, n_acc_out);
}

}  // namespace es
