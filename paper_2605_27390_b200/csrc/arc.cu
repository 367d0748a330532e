// arc.cu -- N1: the dynamic buffer's Adaptive Replacement Cache
// (App. A.3 and Table 4: c = N_dyn, p0 = 128, ghost lists
// 256 / 256, min residency 8 decoding steps, warm-up 50 events, P:433-437;
// SPEC S:288-348) -- host code: a sequential, single-writer state machine
// with O(1) list operations (intrusive LRU lists over a hash map) --
// and the incremental subset update it drives on the device:
//   S' = sort((S \ evicted) u admitted)
// by one kernel of per-element binary searches (no full rebuild).
//
// Semantics (the same readings as the oracle, A1/A2): touch moves a
// T1 / T2 member to the MRU end of T2; admit(tokens) is one OOV event (the
// warm-up counts events): a resident token is touched, a B1 ghost raises p by
// max(1, |B2| / |B1|) (integer division; after warm-up) and lands in T2, a B2
// ghost lowers p by max(1, |B1| / |B2|) and lands in T2, anything else lands
// in T1. Before an insertion into a full cache one eviction: from T1 if
// |T1| > p (or T2 is empty), else T2; the LRU-most member resident for
// >= min_res steps since its admission (A1); else the other list's (A2); else
// plain LRU of the chosen list. Evicted tokens enter B1 / B2 at the MRU
// end; ghost lists are trimmed at the LRU end to their capacities.
#include <algorithm>
#include <cstdint>
#include <list>
#include <unordered_map>
#include <vector>

#pragma GCC visibility push(default)   // the C ABI only (as in api.cu)
#include "../../include/evospec.h"
#pragma GCC visibility pop
#include "common.cuh"
#include "kernels.cuh"

namespace es {

struct ArcEntry {
    int list;          // 0 T1, 1 T2, 2 B1, 3 B2
    int64_t admitted;  // admission step (residents)
    std::list<int32_t>::iterator it;
};

struct Arc {
    int c, p, cap[4], min_res, warmup;
    int64_t events = 0;
    std::list<int32_t> L[4];   // LRU at the front
    std::unordered_map<int32_t, ArcEntry> where;

    void push(int l, int32_t t, int64_t admitted) {
        L[l].push_back(t);
        where[t] = ArcEntry{l, admitted, std::prev(L[l].end())};
    }
    void erase(int32_t t) {
        auto f = where.find(t);
        L[f->second.list].erase(f->second.it);
        where.erase(f);
    }
    bool touch(int32_t t) {
        auto f = where.find(t);
        if (f == where.end() || f->second.list > 1) return false;
        const int64_t adm = f->second.admitted;
        erase(t);
        push(1, t, adm);
        return true;
    }
    // the LRU-most member of list l resident for >= min_res steps, or none
    bool eligible(int l, int64_t step, int32_t& out) const {
        for (int32_t t : L[l])
            if (step - where.at(t).admitted >= min_res) { out = t; return true; }
        return false;
    }
    int32_t evict(int64_t step) {
        int l = (!L[0].empty() && ((int)L[0].size() > p || L[1].empty())) ? 0 : 1;
        int32_t t;
        if (!eligible(l, step, t)) {
            if (eligible(1 - l, step, t)) l = 1 - l;
            else t = L[l].front();
        }
        erase(t);
        const int g = l + 2;
        push(g, t, 0);
        while ((int)L[g].size() > cap[g]) erase(L[g].front());
        return t;
    }
    int admit(const int32_t* tok, int n, int64_t step, int32_t* evicted) {
        ++events;
        const bool adapt = events > warmup;
        int ne = 0;
        for (int k = 0; k < n; ++k) {
            const int32_t t = tok[k];
            if (touch(t)) continue;
            bool to2 = false;
            auto f = where.find(t);
            if (f != where.end() && f->second.list == 2) {
                if (adapt) p = std::min(c, p + std::max(1, (int)L[3].size() / (int)L[2].size()));
                erase(t);
                to2 = true;
            } else if (f != where.end() && f->second.list == 3) {
                if (adapt) p = std::max(0, p - std::max(1, (int)L[2].size() / (int)L[3].size()));
                erase(t);
                to2 = true;
            }
            if ((int)(L[0].size() + L[1].size()) >= c) {
                const int32_t e = evict(step);
                if (evicted) evicted[ne] = e;
                ++ne;
            }
            push(to2 ? 1 : 0, t, step);
        }
        return ne;
    }
};

// ---------------------------------------------------------------- device update
// out[i] for a kept S[i]: i - (#removed S entries before i) + (#added ids < S[i]);
// for added a_j: (#kept S entries < a_j) + j. removed and added are sorted.
__device__ __forceinline__ int lb32(const int32_t* a, int n, int32_t v) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (__ldg(&a[m]) < v) lo = m + 1; else hi = m;
    }
    return lo;
}

// Contract (header): removed is a subset of S, added is disjoint from S \ removed.
// A violation cannot corrupt memory: every destination is range-checked, and
// (flags != null) each removed id missing from S / added id already kept raises
// kFlagBadIds (the output is then not the set the caller asked for).
__global__ void subset_update_kernel(const int32_t* __restrict__ S, int n, const int32_t* __restrict__ rem, int nr,
                                     const int32_t* __restrict__ add, int na, int32_t* __restrict__ out,
                                     int32_t* __restrict__ n_out, int32_t* __restrict__ flags) {
    pdl_trigger();
    pdl_wait();
    const int tid = blockIdx.x * blockDim.x + threadIdx.x, T = gridDim.x * blockDim.x;
    const int n_new = n - nr + na;
    bool bad = false;
    for (int i = tid; i < n; i += T) {
        const int32_t v = __ldg(&S[i]);
        const int r = lb32(rem, nr, v);
        if (r < nr && __ldg(&rem[r]) == v) continue;     // evicted
        const int d = i - r + lb32(add, na, v);           // r removed entries precede v
        if (d >= 0 && d < n_new) out[d] = v;
        else bad = true;
    }
    for (int j = tid; j < nr; j += T) {   // every removed id must be in S
        const int32_t v = __ldg(&rem[j]);
        const int p = lb32(S, n, v);
        bad |= !(p < n && __ldg(&S[p]) == v);
    }
    for (int j = tid; j < na; j += T) {
        const int32_t v = __ldg(&add[j]);
        const int p = lb32(S, n, v), rp = lb32(rem, nr, v);
        const bool kept = p < n && __ldg(&S[p]) == v && !(rp < nr && __ldg(&rem[rp]) == v);
        const int d = p - rp + j;   // kept S entries < v, then j added ones
        bad |= kept;
        if (!kept && d >= 0 && d < n_new) out[d] = v;
        else bad = true;
    }
    if (bad && flags) atomicOr(flags, kFlagBadIds);
    if (tid == 0) *n_out = n_new;
}

void launch_subset_update(const int32_t* S, int n, const int32_t* rem, int nr, const int32_t* add, int na,
                          int32_t* out, int32_t* n_out, int32_t* flags, cudaStream_t st) {
    const int threads = 256;
    const int blocks = std::max(1, std::min(kNumSMs, (n + na + threads - 1) / threads));
    launch_pdl(subset_update_kernel, dim3(blocks), dim3(threads), 0, st, S, n, rem, nr, add, na, out, n_out, flags);
}

}  // namespace es

// ---------------------------------------------------------------- C ABI
struct evospec_arc { es::Arc a; };

extern "C" {

evospec_status evospec_arc_create(evospec_arc** out, int32_t capacity,
    int32_t p0, int32_t b1_cap, int32_t b2_cap,
    int32_t min_residency, int32_t warmup_events) {
    if (!out || capacity < 1 || b1_cap < 0 || b2_cap < 0 || min_residency < 0 || warmup_events < 0)
        return EVOSPEC_EINPUT;
    evospec_arc* x = new evospec_arc();
    es::Arc& a = x->a;
    a.c = capacity;
    a.p = std::max(0, std::min(capacity, p0));
    a.cap[0] = a.cap[1] = capacity;
    a.cap[2] = b1_cap;
    a.cap[3] = b2_cap;
    a.min_res = min_residency;
    a.warmup = warmup_events;
    *out = x;
    return EVOSPEC_OK;
}

evospec_status evospec_arc_destroy(evospec_arc* arc) {
    delete arc;
    return EVOSPEC_OK;
}

int32_t evospec_arc_touch(evospec_arc* arc, int32_t token, int64_t step) {
    (void)step;
    return arc && arc->a.touch(token) ? 1 : 0;
}

evospec_status evospec_arc_admit(evospec_arc* arc, const int32_t* tokens,
    int32_t n, int64_t step, int32_t* evicted,
    int32_t* n_evicted) {
    if (!arc || n < 0 || (n > 0 && !tokens) || !n_evicted) return EVOSPEC_EINPUT;
    *n_evicted = arc->a.admit(tokens, n, step, evicted);
    return EVOSPEC_OK;
}

evospec_status evospec_arc_admit_delta(evospec_arc* arc, const int32_t* tokens, int32_t n, int64_t step,
    int32_t* added, int32_t* n_added, int32_t* removed, int32_t* n_removed) {
    if (!arc || n < 0 || (n > 0 && !tokens) || !added || !n_added || !removed || !n_removed) return EVOSPEC_EINPUT;
    es::Arc& a = arc->a;
    std::vector<int32_t> before;
    before.reserve(a.L[0].size() + a.L[1].size());
    for (int l = 0; l < 2; ++l) before.insert(before.end(), a.L[l].begin(), a.L[l].end());
    std::sort(before.begin(), before.end());
    std::vector<int32_t> ev(n > 0 ? n : 1);
    a.admit(tokens, n, step, ev.data());
    std::vector<int32_t> after;
    after.reserve(a.L[0].size() + a.L[1].size());
    for (int l = 0; l < 2; ++l) after.insert(after.end(), a.L[l].begin(), a.L[l].end());
    std::sort(after.begin(), after.end());
    // net membership change: a token admitted and evicted in the same event, or
    // evicted and re-admitted, is in neither list (the update's contract)
    int na = 0, nr = 0;
    size_t i = 0, j = 0;
    while (i < before.size() || j < after.size()) {
        if (j == after.size() || (i < before.size() && before[i] < after[j])) removed[nr++] = before[i++];
        else if (i == before.size() || after[j] < before[i]) added[na++] = after[j++];
        else { ++i; ++j; }
    }
    *n_added = na;
    *n_removed = nr;
    return EVOSPEC_OK;
}

evospec_status evospec_arc_state(const evospec_arc* arc, int32_t* out,
    int32_t cap, int32_t* n_out) {
    if (!arc || !out || !n_out) return EVOSPEC_EINPUT;
    const es::Arc& a = arc->a;
    const int need = 5 + (int)(a.L[0].size() + a.L[1].size() + a.L[2].size() + a.L[3].size());
    if (cap < need) return EVOSPEC_EINPUT;
    int o = 0;
    for (int l = 0; l < 4; ++l) out[o++] = (int32_t)a.L[l].size();
    out[o++] = a.p;
    for (int l = 0; l < 4; ++l)
        for (int32_t t : a.L[l]) out[o++] = t;
    *n_out = o;
    return EVOSPEC_OK;
}

evospec_status evospec_subset_update(const int32_t* subset, int32_t n,
    const int32_t* removed, int32_t n_removed,
    const int32_t* added, int32_t n_added,
    int32_t* out, int32_t* n_out, int32_t* flags,
    void* stream) {
    if (n < 0 || n_removed < 0 || n_added < 0 || n_removed > n || (n > 0 && !subset) ||
        (n_removed > 0 && !removed) || (n_added > 0 && !added) || !out || !n_out)
        return EVOSPEC_EINPUT;
    es::launch_subset_update(subset, n, removed, n_removed, added, n_added, out, n_out, flags, (cudaStream_t)stream);
    const cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? EVOSPEC_OK : EVOSPEC_ECUDA;
}

}  // extern "C"
