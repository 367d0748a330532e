// api.cu -- the C ABI of libevospec.so (include/evospec.h).
//
// Host side only: argument validation, workspace ownership, dispatch, and the
// library-owned NCCL communicator (loaded with dlopen so that the library
// links no NCCL and shares the process's already-loaded libnccl.so.2 when
// torch has one). Every step of the path runs in the kernels of this library.
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nccl.h>

// the C ABI is the only default-visibility surface of the library
#pragma GCC visibility push(default)
#include "../../include/evospec.h"
#pragma GCC visibility pop
#include "kernels.cuh"

using namespace es;

namespace {

thread_local std::string g_last_error;

evospec_status fail(evospec_status st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return st;
}

#define CUDA_TRY(expr)                                                                        \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            return fail(EVOSPEC_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                            \
    } while (0)

#define LAUNCH_CHECK(what)                                                                   \
    do {                                                                                     \
        cudaError_t e_ = cudaGetLastError();                                                 \
        if (e_ != cudaSuccess) return fail(EVOSPEC_ECUDA, "%s: %s", what, cudaGetErrorString(e_)); \
    } while (0)

// ---- NCCL through dlopen ---------------------------------------------------
struct NcclApi {
    bool loaded = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    if (api.loaded) return api;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
    const char* env = getenv("EVOSPEC_NCCL_LIB");
    if (!h && env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return api;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.loaded = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.GroupStart &&
                 api.GroupEnd && api.GetErrorString;
    return api;
}

template <typename T>
cudaError_t dalloc(T** p, size_t n) {
    return cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T));
}

inline int64_t shard_rows(int64_t V, int R, int r) { return (V - r + R - 1) / R; }

}  // namespace

struct evospec_ctx {
    evospec_config cfg;
    int device;
    // semantic scan + selection
    double* s64 = nullptr;
    uint32_t* key32 = nullptr;
    bool no_graph = false;        // draft_step: graph capture failed once (sharded): direct launches
    uint32_t* hist12 = nullptr;   // scan-fused pass-0 histogram; zero between builds (the union kernel
                                  // clears it after the selection has read it)
    bool hist_dirty = false;      // a build stopped between its scan and its union: clear first
    uint32_t* ubits = nullptr;    // [V/32] union bitmap handed to the emit kernel
    uint32_t* sbits = nullptr;    // [V/32] static-core bitmap (static_bits_kernel -> union; zero between builds)
    int* scan_sched = nullptr;    // [2] the TMA scan's stage counter and exit count (zero between launches)
    int32_t* zero_i = nullptr;    // a device 0 (dyn-only union output at offset 0)
    // N1 OOV event (evospec_oov_event_begin / _end): the event's formation runs on a
    // side stream while the caller keeps drafting on the current subset
    cudaStream_t oov_stream = nullptr;
    cudaEvent_t oov_ready = nullptr, oov_done = nullptr;
    int32_t* oov_dyn = nullptr;   // [oov_cap + 1] device: count, then the event's sorted new ids
    int32_t* oov_host = nullptr;  // [oov_cap + 1] pinned
    int32_t* oov_delta = nullptr; // [2 * oov_cap] device: removed, added
    int oov_cap = 0;
    bool oov_pending = false;
    int32_t* ver_acc = nullptr;   // [kMaxChain + 1] verification: per-position accept flags
    int32_t* ver_tok = nullptr;   // [kMaxChain + 1] verification: per-position emitted token
    uint32_t* hist = nullptr;     // [12][4096] further select passes
    int cand_cap = 0;             // candidate superset capacity (union smem)
    int* cand_count = nullptr;
    double* cand_s = nullptr;     // [cand_cap]
    int32_t* cand_id = nullptr;
    int* loc_count = nullptr;     // sharded index: exact local top-N
    double* loc_s = nullptr;      // [max_sem]
    int32_t* loc_id = nullptr;
    double* gat_s = nullptr;      // [R][max_sem] gathered local top-N
    int32_t* gat_id = nullptr;
    int32_t* sem_ids = nullptr;   // S_sem of the last build (unordered)
    int* sem_n = nullptr;
    int32_t* ctx_sel = nullptr;
    int* ctx_n = nullptr;
    // LM head partials
    LmhPartials part{};
    int part_cta_cap = 0;
    int* flags = nullptr;
    float* wmax = nullptr;
    // merge gather
    int32_t* g_ids = nullptr;
    float* g_vals = nullptr;
    float* g_m = nullptr;
    float* g_s = nullptr;
    // draft-step staging
    void* st_q = nullptr;
    void* st_H = nullptr;
    int32_t* st_seeds = nullptr;
    int32_t* st_ctx = nullptr;
    int32_t* st_S = nullptr;
    int32_t* st_nS = nullptr;
    int32_t* st_local = nullptr;
    int32_t* st_nlocal = nullptr;
    int32_t* st_tids = nullptr;
    float* st_tvals = nullptr;
    float* st_m = nullptr;
    float* st_s = nullptr;
    int32_t* st_oids = nullptr;
    float* st_ovals = nullptr;
    float* st_lse = nullptr;
    float* st_probs = nullptr;
    // ragged (batched serving) LM head: stacked [2][max_rows][max_k] static / dynamic triples
    int32_t* rg_ids = nullptr;
    float* rg_vals = nullptr;
    float* rg_m = nullptr;
    float* rg_s = nullptr;
    int32_t* rg_seg = nullptr;   // device {0, n_static}
    int32_t* rg_segcta = nullptr;   // device [kMaxSeg+1] CTA schedule of the dynamic blocks
    // two-list draft step: the union's early copy of the dynamic list + its flag (lmh_tc.cu)
    int32_t* early_ids = nullptr;
    int* early_flag = nullptr;
    // draft_step as a CUDA graph (see evospec_draft_step)
    cudaGraphExec_t g_exec = nullptr;
    evospec_step_io g_key{};
    long long g_launches = 0;
    cudaStream_t cap_stream = nullptr;
    cudaStream_t s_h = nullptr;         // host-staged H copy, overlapping the build
    cudaEvent_t ev_in = nullptr, ev_h = nullptr;
    int last_n_sem = 0;
    ncclComm_t comm = nullptr;
    // measurement hooks
    int64_t launches = 0;
    long long* trace = nullptr;   // EVOSPEC_TRACE=1: per-CTA LM-head stamps [148][8]
    bool timing = false;
    std::vector<cudaEvent_t> ev;   // [stage][slot][2]
    int ev_count[EVOSPEC_NUM_STAGES] = {0};
};

namespace {
constexpr int kTimingSlots = 4096;
constexpr int kTraceLen = kTraceOvf + 2 * kNumSMs;   // LM-head CTAs, finalize rows,
                                                                              // union stamps, scan / candidate stamps

// union stamps live after the LM-head / finalize slots
long long* union_trace(evospec_ctx* ctx, cudaStream_t st) {
    if (!getenv("EVOSPEC_TRACE")) return nullptr;
    if (!ctx->trace && cudaMalloc(&ctx->trace, kTraceLen * sizeof(long long)) != cudaSuccess) return nullptr;
    set_step_trace(ctx->trace + 2 * kNumSMs * 8 + 112);
    return ctx->trace + 2 * kNumSMs * 8;
}

// Records a start/end CUDA event pair around a stage when timing is on.
struct StageTimer {
    evospec_ctx* ctx;
    int stage;
    cudaStream_t st;
    int slot = -1;
    StageTimer(evospec_ctx* c, int s, cudaStream_t stream) : ctx(c), stage(s), st(stream) {
        if (!ctx->timing || ctx->ev_count[stage] >= kTimingSlots) return;
        slot = ctx->ev_count[stage]++;
        cudaEventRecord(ctx->ev[((size_t)stage * kTimingSlots + slot) * 2], st);
    }
    void stop() {
        if (slot >= 0) cudaEventRecord(ctx->ev[((size_t)stage * kTimingSlots + slot) * 2 + 1], st);
        slot = -1;
    }
    ~StageTimer() { stop(); }
};
}  // namespace

extern "C" {

const char* evospec_version(void) { return "evospec-b200 0.1.0 (sm_100a)"; }

const char* evospec_last_error(void) { return g_last_error.c_str(); }

const char* evospec_status_string(evospec_status st) {
    switch (st) {
        case EVOSPEC_OK: return "ok";
        case EVOSPEC_EINPUT: return "input error";
        case EVOSPEC_EINVARIANT: return "invariant violation";
        case EVOSPEC_ECUDA: return "CUDA error";
        case EVOSPEC_ENCCL: return "NCCL error";
        case EVOSPEC_ENOMEM: return "out of device memory";
        default: return "unknown status";
    }
}

evospec_status evospec_destroy(evospec_ctx* ctx) {
    if (!ctx) return EVOSPEC_OK;
    cudaSetDevice(ctx->device);
    void* ptrs[] = {ctx->s64, ctx->key32, ctx->hist12, ctx->hist, ctx->cand_count, ctx->cand_s, ctx->cand_id,
                    ctx->loc_count, ctx->loc_s, ctx->loc_id, ctx->gat_s, ctx->gat_id, ctx->sem_ids, ctx->sem_n,
                    ctx->ctx_sel,
                    ctx->ctx_n, ctx->part.val, ctx->part.id, ctx->part.m, ctx->part.s, ctx->part.cnt, ctx->part.xcnt,
                    ctx->flags, ctx->wmax, ctx->g_ids, ctx->g_vals, ctx->g_m, ctx->g_s, ctx->st_q, ctx->st_H,
                    ctx->st_seeds, ctx->st_ctx, ctx->st_S, ctx->st_nS, ctx->st_local, ctx->st_nlocal,
                    ctx->st_tids, ctx->st_tvals, ctx->st_m, ctx->st_s, ctx->st_oids, ctx->st_ovals,
                    ctx->st_lse, ctx->st_probs, ctx->ubits, ctx->sbits, ctx->scan_sched, ctx->rg_ids, ctx->rg_vals, ctx->rg_m, ctx->rg_s, ctx->rg_seg, ctx->rg_segcta, ctx->ver_acc, ctx->ver_tok, ctx->zero_i};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (ctx->comm && nccl().loaded) nccl().CommDestroy(ctx->comm);
    for (cudaEvent_t e : ctx->ev) cudaEventDestroy(e);
    if (ctx->trace) cudaFree(ctx->trace);
    if (ctx->early_ids) cudaFree(ctx->early_ids);
    if (ctx->early_flag) cudaFree(ctx->early_flag);
    if (ctx->g_exec) cudaGraphExecDestroy(ctx->g_exec);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->s_h) cudaStreamDestroy(ctx->s_h);
    if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
    if (ctx->ev_h) cudaEventDestroy(ctx->ev_h);
    if (ctx->oov_stream) cudaStreamDestroy(ctx->oov_stream);
    if (ctx->oov_ready) cudaEventDestroy(ctx->oov_ready);
    if (ctx->oov_done) cudaEventDestroy(ctx->oov_done);
    if (ctx->oov_dyn) cudaFree(ctx->oov_dyn);
    if (ctx->oov_delta) cudaFree(ctx->oov_delta);
    if (ctx->oov_host) cudaFreeHost(ctx->oov_host);
    delete ctx;
    return EVOSPEC_OK;
}

evospec_status evospec_create(evospec_ctx** out, const evospec_config* cfg, int device) {
    if (!out || !cfg) return fail(EVOSPEC_EINPUT, "create: null argument");
    *out = nullptr;
    const evospec_config& c = *cfg;
    if (c.V < 1 || c.d < 8 || c.d % 8 != 0)
        return fail(EVOSPEC_EINPUT, "create: need V >= 1 and d a positive multiple of 8 (V=%d d=%d)", c.V, c.d);
    if ((c.w_dtype != EVOSPEC_BF16 && c.w_dtype != EVOSPEC_FP32) ||
        (c.h_dtype != EVOSPEC_BF16 && c.h_dtype != EVOSPEC_FP32))
        return fail(EVOSPEC_EINPUT, "create: dtype must be EVOSPEC_BF16 or EVOSPEC_FP32");
    if (c.n_shards < 1 || c.shard_rank < 0 || c.shard_rank >= c.n_shards)
        return fail(EVOSPEC_EINPUT, "create: bad shard %d of %d", c.shard_rank, c.n_shards);
    if (c.max_subset < 0 || c.max_subset > c.V || c.max_rows < 1 || c.max_k < 1 || c.max_k > kMaxK ||
        c.max_sem < 0 || c.max_sem > c.V || c.max_seeds < 0 || c.max_ctx < 0 || c.max_ctx > kMaxCtx)
        return fail(EVOSPEC_EINPUT, "create: capacity out of range (max_k <= %d, max_ctx <= %d)", kMaxK, kMaxCtx);
    if (c.V > (1 << 20)) return fail(EVOSPEC_EINPUT, "create: V > 2^20 unsupported (bitmap in smem)");
    CUDA_TRY(cudaSetDevice(device));
    evospec_ctx* x = new evospec_ctx();
    x->cfg = c;
    x->device = device;
    const int R = c.n_shards;
    const size_t V = (size_t)c.V, d = (size_t)c.d;
    const size_t sem = std::max(1, c.max_sem);
    const int cta_cap = std::max(lmh_gemv_grid(), 2 * kNumSMs);
    x->part_cta_cap = cta_cap;
    const size_t pr = (size_t)cta_cap * c.max_rows;
    const size_t hb = c.h_dtype == EVOSPEC_BF16 ? 2 : 4;
    cudaError_t e = cudaSuccess;
    auto A = [&](cudaError_t r) { if (e == cudaSuccess) e = r; };
    x->cand_cap = union_cand_cap(c.V, 64);
    if (getenv("EVOSPEC_TRACE")) union_trace(x, nullptr);   // (stamps set up before any graph capture)
    if (c.max_sem > x->cand_cap) {
        const int cap_v = x->cand_cap;
        delete x;
        return fail(EVOSPEC_EINPUT, "create: max_sem=%d exceeds the selection capacity %d at V=%d", c.max_sem,
                    cap_v, c.V);
    }
    const size_t cap = (size_t)x->cand_cap;
    A(dalloc(&x->s64, V)); A(dalloc(&x->key32, V)); A(dalloc(&x->hist12, kHistBins)); A(dalloc(&x->ubits, (V + 31) / 32)); A(cudaMemset(x->hist12, 0, kHistBins * sizeof(uint32_t)));
    A(dalloc(&x->scan_sched, 2)); A(cudaMemset(x->scan_sched, 0, 2 * sizeof(int)));
    A(dalloc(&x->sbits, (V + 31) / 32 + 4)); A(cudaMemset(x->sbits, 0, ((V + 31) / 32 + 4) * sizeof(uint32_t)));
    A(dalloc(&x->early_ids, (size_t)c.max_subset + 64)); A(dalloc(&x->early_flag, 1));
    A(cudaMemset(x->early_flag, 0, sizeof(int)));
    A(dalloc(&x->hist, 12 * kHistBins + 32)); A(cudaMemset(x->hist, 0, (12 * kHistBins + 32) * sizeof(uint32_t)));
    A(dalloc(&x->ver_acc, kMaxChain + 1)); A(dalloc(&x->ver_tok, kMaxChain + 1));
    A(dalloc(&x->zero_i, 1)); A(cudaMemset(x->zero_i, 0, sizeof(int32_t)));
    A(dalloc(&x->cand_count, 4)); A(dalloc(&x->cand_s, cap)); A(dalloc(&x->cand_id, cap));
    A(dalloc(&x->loc_count, 4)); A(dalloc(&x->loc_s, sem)); A(dalloc(&x->loc_id, sem));
    A(dalloc(&x->gat_s, sem * R)); A(dalloc(&x->gat_id, sem * R));
    A(dalloc(&x->sem_ids, sem)); A(dalloc(&x->sem_n, 1));
    A(dalloc(&x->ctx_sel, std::max(1, c.max_ctx))); A(dalloc(&x->ctx_n, 1));
    A(dalloc(&x->part.val, pr * std::max(kMaxKP, kTcListLS))); A(dalloc(&x->part.id, pr * std::max(kMaxKP, kTcListLS)));
    A(dalloc(&x->part.m, pr)); A(dalloc(&x->part.s, pr)); A(dalloc(&x->part.cnt, pr)); A(dalloc(&x->part.xcnt, pr));
    x->part.cs = cta_cap;
    A(dalloc(&x->flags, 1)); A(dalloc(&x->wmax, 1));
    const size_t trip = (size_t)R * c.max_rows * c.max_k;
    A(dalloc(&x->g_ids, trip)); A(dalloc(&x->g_vals, trip));
    A(dalloc(&x->g_m, (size_t)R * c.max_rows)); A(dalloc(&x->g_s, (size_t)R * c.max_rows));
    A(cudaMalloc(&x->st_q, d * hb)); A(cudaMalloc(&x->st_H, (size_t)c.max_rows * d * hb));
    A(dalloc(&x->st_seeds, std::max(1, c.max_seeds))); A(dalloc(&x->st_ctx, std::max(1, c.max_ctx)));
    A(dalloc(&x->st_S, std::max(1, c.max_subset))); A(dalloc(&x->st_nS, 1));
    A(dalloc(&x->st_local, std::max(1, c.max_subset))); A(dalloc(&x->st_nlocal, 1));
    const size_t hk = (size_t)c.max_rows * c.max_k;
    A(dalloc(&x->st_tids, hk)); A(dalloc(&x->st_tvals, hk)); A(dalloc(&x->st_m, c.max_rows));
    A(dalloc(&x->st_s, c.max_rows));
    // host-I/O output staging as ONE block [ids | vals | lse | probs] (laid out per call
    // for its n_h, k): a caller whose host outputs are one contiguous block in the same
    // order gets one device-to-host copy per step instead of four
    A(dalloc(&x->st_oids, 3 * hk + c.max_rows));
    x->st_ovals = nullptr; x->st_lse = nullptr; x->st_probs = nullptr;
    A(dalloc(&x->rg_ids, 2 * hk)); A(dalloc(&x->rg_vals, 2 * hk));
    A(dalloc(&x->rg_m, 2 * (size_t)c.max_rows)); A(dalloc(&x->rg_s, 2 * (size_t)c.max_rows)); A(dalloc(&x->rg_seg, 2)); A(dalloc(&x->rg_segcta, kMaxSeg + 1));
    if (e == cudaSuccess) e = cudaMemset(x->flags, 0, sizeof(int));
    if (e == cudaSuccess) {
        const float inf = INFINITY;  // until evospec_prepare_weights: certification never passes
        e = cudaMemcpy(x->wmax, &inf, sizeof(float), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
        evospec_destroy(x);
        return fail(e == cudaErrorMemoryAllocation ? EVOSPEC_ENOMEM : EVOSPEC_ECUDA, "create: %s",
                    cudaGetErrorString(e));
    }
    *out = x;
    return EVOSPEC_OK;
}

evospec_status evospec_prepare_weights(evospec_ctx* ctx, const void* W, int64_t n_rows, void* stream) {
    if (!ctx || !W || n_rows < 0) return fail(EVOSPEC_EINPUT, "prepare_weights: bad argument");
    launch_rownorm_max(W, ctx->cfg.w_dtype, n_rows, ctx->cfg.d, ctx->wmax, (cudaStream_t)stream);
    ctx->launches += 1;
    LAUNCH_CHECK("rownorm_max");
    return EVOSPEC_OK;
}

evospec_status evospec_sync_status(evospec_ctx* ctx, void* stream) {
    if (!ctx) return fail(EVOSPEC_EINPUT, "sync_status: null context");
    int32_t f = 0;
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaMemcpyAsync(&f, ctx->flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (f & (kFlagBadIds | kFlagBudget))
        return fail(EVOSPEC_EINVARIANT, "invariant violated on the device (flags 0x%x: %s%s)", f,
                    (f & kFlagBadIds) ? "unsorted / out-of-range ids " : "", (f & kFlagBudget) ? "budget" : "");
    return EVOSPEC_OK;
}

evospec_status evospec_get_flags(evospec_ctx* ctx, int32_t* flags_out, int clear, void* stream) {
    if (!ctx || !flags_out) return fail(EVOSPEC_EINPUT, "get_flags: null argument");
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaMemcpyAsync(flags_out, ctx->flags, sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (clear) CUDA_TRY(cudaMemsetAsync(ctx->flags, 0, sizeof(int), st));
    return EVOSPEC_OK;
}

evospec_status evospec_comm_unique_id(void* uid_out) {
    if (!uid_out) return fail(EVOSPEC_EINPUT, "comm_unique_id: null");
    NcclApi& n = nccl();
    if (!n.loaded) return fail(EVOSPEC_ENCCL, "comm_unique_id: libnccl.so.2 not loadable");
    ncclUniqueId id;
    ncclResult_t r = n.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(EVOSPEC_ENCCL, "ncclGetUniqueId: %s", n.GetErrorString(r));
    memcpy(uid_out, &id, sizeof(id));
    return EVOSPEC_OK;
}

evospec_status evospec_comm_init(evospec_ctx* ctx, const void* uid) {
    if (!ctx || !uid) return fail(EVOSPEC_EINPUT, "comm_init: null");
    NcclApi& n = nccl();
    if (!n.loaded) return fail(EVOSPEC_ENCCL, "comm_init: libnccl.so.2 not loadable");
    CUDA_TRY(cudaSetDevice(ctx->device));
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    ncclResult_t r = n.CommInitRank(&ctx->comm, ctx->cfg.n_shards, id, ctx->cfg.shard_rank);
    if (r != ncclSuccess) return fail(EVOSPEC_ENCCL, "ncclCommInitRank: %s", n.GetErrorString(r));
    return EVOSPEC_OK;
}

// dyn_base != null: batched mode -- the sorted dynamic list only, written at
// out_ids + *dyn_base, with *out_n = *dyn_base + its length
static evospec_status union_from_candidates(evospec_ctx* ctx, const double* cand_s, const int32_t* cand_id,
                                            int64_t n_cand, const int32_t* static_ids, int32_t n_static,
                                            const int32_t* seeds, int32_t n_seed, const int32_t* row_ptr,
                                            const int32_t* col, const int32_t* ctx_ids, int32_t n_ctx,
                                            const evospec_build_params* p, int32_t* out_ids, int32_t* out_n,
                                            int32_t* out_local_ids, int32_t* out_local_n, cudaStream_t st,
                                            const int32_t* dyn_base, cudaEvent_t wait_before_union,
                                            bool sbits_ready, bool early = false);

// a2 on a vocabulary shard: exact fp64 scores of this shard's E rows (global id
// = row * R + r) and the shard's exact top-N (s desc, id asc), padded with id -1
// when the shard has fewer rows -- what every rank contributes to the candidate
// all-gather.
static evospec_status local_candidates_impl(evospec_ctx* ctx, const void* E, int64_t n_e_rows, const void* q,
                                            int32_t N, double* out_s, int32_t* out_id, cudaStream_t st) {
    const evospec_config& c = ctx->cfg;
    const int R = c.n_shards, r = c.shard_rank;
    StageTimer t(ctx, EVOSPEC_STAGE_SCAN, st);
    if (ctx->hist_dirty) CUDA_TRY(cudaMemsetAsync(ctx->hist12, 0, kHistBins * sizeof(uint32_t), st));
    launch_sem_scan(E, c.w_dtype, n_e_rows, c.d, q, c.h_dtype, ctx->s64, ctx->key32, ctx->hist12, st, ctx->hist,
                    12 * kHistBins, ctx->loc_count, true, ctx->scan_sched);
    ctx->hist_dirty = true;
    ctx->launches += 2;
    LAUNCH_CHECK("sem_scan");
    t.stop();
    StageTimer t_sel(ctx, EVOSPEC_STAGE_SELECT, st);
    CUDA_TRY(cudaMemsetAsync(out_id, 0xFF, (size_t)N * sizeof(int32_t), st));
    CUDA_TRY(launch_topn_cand(ctx->s64, nullptr, n_e_rows, R, r, N, N, ctx->hist12, ctx->hist, ctx->loc_count, out_s,
                              out_id, st, true));
    return EVOSPEC_OK;
}

static evospec_status build_impl(evospec_ctx* ctx, const void* E, int64_t n_e_rows, const void* q,
                                 const int32_t* static_ids, int32_t n_static, const int32_t* seeds, int32_t n_seed,
                                 const int32_t* row_ptr, const int32_t* col, const int32_t* ctx_ids, int32_t n_ctx,
                                 const evospec_build_params* p, int32_t* out_ids, int32_t* out_n,
                                 int32_t* out_local_ids, int32_t* out_local_n, void* stream,
                                 const int32_t* dyn_base, cudaEvent_t wait_before_union = nullptr,
                                 const double* ext_s = nullptr, const int32_t* ext_id = nullptr, int64_t n_ext = 0,
                                 bool early = false) {
    // ext_s / ext_id: the shards' stacked local candidates (evospec_build_subset_from_candidates)
    const bool ext = ext_s != nullptr;
    if (!ctx || (!ext && (!E || !q)) || !p || !out_ids || !out_n) return fail(EVOSPEC_EINPUT, "build_subset: null argument");
    if (ext && (!ext_id || n_ext < 1 || n_ext > (int64_t)ctx->cfg.n_shards * ctx->cfg.max_sem))
        return fail(EVOSPEC_EINPUT, "build_subset_from_candidates: n_cand=%lld not in [1, R * max_sem]", (long long)n_ext);
    const evospec_config& c = ctx->cfg;
    const int R = c.n_shards, r = c.shard_rank;
    cudaStream_t st = (cudaStream_t)stream;
    if (n_static < 0 || (n_static > 0 && !static_ids) || n_seed < 0 || (n_seed > 0 && !seeds))
        return fail(EVOSPEC_EINPUT, "build_subset: bad static / seed arguments");
    if (p->n_sem < 0 || p->n_sem > c.max_sem || p->n_dyn < 0 || p->per_seed < 0 || p->per_seed > 64 ||
        p->n_graph_sem_seeds < 0 || n_seed + std::min(p->n_graph_sem_seeds, p->n_sem) > std::min(c.max_seeds, 128))
        return fail(EVOSPEC_EINPUT, "build_subset: params out of capacity (n_sem <= %d, seeds <= %d, per_seed <= 64)",
                    c.max_sem, std::min(c.max_seeds, 128));
    if ((int64_t)n_static + p->n_dyn > c.max_subset)
        return fail(EVOSPEC_EINPUT, "build_subset: n_static + n_dyn = %lld > max_subset %d",
                    (long long)n_static + p->n_dyn, c.max_subset);
    if (p->ctx_min_count > 0 && (n_ctx < 0 || n_ctx > c.max_ctx || (n_ctx > 0 && !ctx_ids)))
        return fail(EVOSPEC_EINPUT, "build_subset: ctx tokens exceed max_ctx %d", c.max_ctx);
    if ((row_ptr == nullptr) != (col == nullptr)) return fail(EVOSPEC_EINPUT, "build_subset: CSR half given");
    if (R > 1 && (!out_local_ids || !out_local_n))
        return fail(EVOSPEC_EINPUT, "build_subset: sharded context needs out_local_ids / out_local_n");
    const int N = p->n_sem;
    if (ext)
        return union_from_candidates(ctx, ext_s, ext_id, n_ext, static_ids, n_static, seeds, n_seed, row_ptr, col,
                                     ctx_ids, n_ctx, p, out_ids, out_n, out_local_ids, out_local_n, st, dyn_base,
                                     wait_before_union, false);
    const bool full_scan = n_e_rows == c.V;
    const int64_t local_rows = shard_rows(c.V, R, r);
    if (!full_scan && !(R > 1 && n_e_rows == local_rows))
        return fail(EVOSPEC_EINPUT, "build_subset: n_e_rows must be V=%d or this shard's %lld rows", c.V,
                    (long long)local_rows);
    if (!full_scan && !ctx->comm)
        return fail(EVOSPEC_EINPUT, "build_subset: a sharded index needs evospec_comm_init (or the comm-less "
                                    "evospec_build_local_candidates + evospec_build_subset_from_candidates)");

    if (full_scan) {
        // a2: exact fp64 scores (+ fused pass-0 histogram), candidate superset of the top-N
        StageTimer t(ctx, EVOSPEC_STAGE_SCAN, st);
        // the scan zeroes the next selection's histogram scratch and count
        if (ctx->hist_dirty) CUDA_TRY(cudaMemsetAsync(ctx->hist12, 0, kHistBins * sizeof(uint32_t), st));
        // a4's static bitmap: an input-only kernel the scan overlaps (PDL)
        launch_static_bits(static_ids, n_static, c.V, c.debug_checks, ctx->sbits, ctx->flags, st);
        launch_sem_scan(E, c.w_dtype, n_e_rows, c.d, q, c.h_dtype, ctx->s64, ctx->key32, ctx->hist12, st, ctx->hist,
                        12 * kHistBins, ctx->cand_count, true, ctx->scan_sched);
        ctx->hist_dirty = true;
        ctx->launches += 2;
    } else {
        // this shard's exact local top-N, all-gathered (N (s, id) pairs per rank)
        evospec_status ls = local_candidates_impl(ctx, E, n_e_rows, q, N, ctx->loc_s, ctx->loc_id, st);
        if (ls != EVOSPEC_OK) return ls;
        StageTimer t_g(ctx, EVOSPEC_STAGE_MERGE, st);
        NcclApi& n = nccl();
        n.GroupStart();
        ncclResult_t r1 = n.AllGather(ctx->loc_s, ctx->gat_s, (size_t)N, ncclFloat64, ctx->comm, st);
        ncclResult_t r2 = n.AllGather(ctx->loc_id, ctx->gat_id, (size_t)N, ncclInt32, ctx->comm, st);
        ncclResult_t r3 = n.GroupEnd();
        if (r1 != ncclSuccess || r2 != ncclSuccess || r3 != ncclSuccess)
            return fail(EVOSPEC_ENCCL, "build_subset all-gather failed");
        t_g.stop();
    }
    LAUNCH_CHECK("sem_scan");
    return union_from_candidates(ctx, full_scan ? nullptr : ctx->gat_s, full_scan ? nullptr : ctx->gat_id,
                                 (int64_t)N * R, static_ids, n_static, seeds, n_seed, row_ptr, col, ctx_ids, n_ctx, p,
                                 out_ids, out_n, out_local_ids, out_local_n, st, dyn_base, wait_before_union,
                                 full_scan, early);
}

// The global candidate superset of the top-N and the formation / union (a2-a4).
// cand_s / cand_id null: the single-shard scan's scores in the workspace (full
// scan, fused pass-0 histogram); else n_cand gathered (s, id) pairs of all shards
// (each shard's exact local top-N, stacked in rank order).
static evospec_status union_from_candidates(evospec_ctx* ctx, const double* cand_s, const int32_t* cand_id,
                                            int64_t n_cand, const int32_t* static_ids, int32_t n_static,
                                            const int32_t* seeds, int32_t n_seed, const int32_t* row_ptr,
                                            const int32_t* col, const int32_t* ctx_ids, int32_t n_ctx,
                                            const evospec_build_params* p, int32_t* out_ids, int32_t* out_n,
                                            int32_t* out_local_ids, int32_t* out_local_n, cudaStream_t st,
                                            const int32_t* dyn_base, cudaEvent_t wait_before_union,
                                            bool sbits_ready, bool early) {
    const evospec_config& c = ctx->cfg;
    const int R = c.n_shards, r = c.shard_rank;
    const int N = p->n_sem;
    if (!sbits_ready) {   // (the full-scan build launches it ahead of the scan instead)
        launch_static_bits(static_ids, n_static, c.V, c.debug_checks, ctx->sbits, ctx->flags, st);
        ctx->launches += 1;
    }
    StageTimer t_sel(ctx, EVOSPEC_STAGE_SELECT, st);
    if (!cand_s) {
        ctx->launches += 1;
        CUDA_TRY(launch_topn_cand(ctx->s64, nullptr, c.V, 1, 0, N, ctx->cand_cap, ctx->hist12, ctx->hist,
                                  ctx->cand_count, ctx->cand_s, ctx->cand_id, st, true));
    } else {
        ctx->launches += 1;
        CUDA_TRY(launch_topn_cand(cand_s, cand_id, n_cand, 0, 0, N, ctx->cand_cap, nullptr, ctx->hist,
                                  ctx->cand_count, ctx->cand_s, ctx->cand_id, st));
    }
    t_sel.stop();
    ctx->last_n_sem = N;
    // a3 context counts (optional)
    const bool use_ctx = p->ctx_min_count > 0 && p->n_ctx_max > 0 && n_ctx > 0;
    StageTimer t_union(ctx, EVOSPEC_STAGE_UNION, st);
    ctx->launches += 1 + (use_ctx ? 1 : 0);
    if (use_ctx) {
        launch_ctx_select(ctx_ids, n_ctx, c.V, p->ctx_min_count, std::min(p->n_ctx_max, c.max_ctx), ctx->ctx_sel,
                          ctx->ctx_n, ctx->flags, st);
        LAUNCH_CHECK("ctx_select");
    }
    // a2 exact S_sem + a3/a4 formation, cap, union
    if (wait_before_union) {   // (draft_step overlap: the host-staged H, copied under the scan)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(st, &cs);
        CUDA_TRY(cudaStreamWaitEvent(st, wait_before_union, cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0));
    }
    const bool emit = R == 1 && !dyn_base;
    launch_union(c.V, static_ids, n_static, seeds, n_seed, ctx->cand_s, ctx->cand_id, ctx->cand_count, ctx->cand_cap,
                 N, row_ptr, col, use_ctx ? ctx->ctx_sel : nullptr, ctx->ctx_n, p->n_graph_sem_seeds, p->per_seed,
                 p->n_dyn, R, r, out_ids, out_n, out_local_ids, out_local_n, ctx->sem_ids, ctx->sem_n,
                 c.debug_checks, ctx->flags, st, union_trace(ctx, st), dyn_base, ctx->hist12,
                 emit ? ctx->ubits : nullptr, ctx->sbits, early ? ctx->early_ids : nullptr,
                 early ? ctx->early_flag : nullptr);
    LAUNCH_CHECK("union");
    ctx->hist_dirty = false;
    if (emit) {   // single shard: the sorted ids from the bitmap by a multi-CTA kernel
        launch_union_emit(ctx->ubits, c.V, out_ids, out_n, out_local_ids, out_local_n, n_static + p->n_dyn,
                          ctx->flags, st);
        ctx->launches += 1;
        LAUNCH_CHECK("union_emit");
    }
    if (c.debug_checks) return evospec_sync_status(ctx, st);
    return EVOSPEC_OK;
}

evospec_status evospec_oov_event_begin(evospec_ctx* ctx, const void* E, int64_t n_e_rows, const void* q,
                                      const int32_t* static_ids, int32_t n_static, const int32_t* seeds,
                                      int32_t n_seed, const int32_t* row_ptr, const int32_t* col,
                                      const evospec_build_params* p, void* stream) {
    if (!ctx || !p) return fail(EVOSPEC_EINPUT, "oov_event_begin: null argument");
    if (ctx->cfg.n_shards != 1) return fail(EVOSPEC_EINPUT, "oov_event_begin: unsharded contexts only");
    if (ctx->oov_pending) return fail(EVOSPEC_EINPUT, "oov_event_begin: an event is already in flight (call _end)");
    if (p->n_dyn < 1 || p->n_dyn > 1024) return fail(EVOSPEC_EINPUT, "oov_event_begin: n_dyn (max insertions) not in [1, 1024]");
    if (!ctx->oov_stream) {
        CUDA_TRY(cudaStreamCreateWithFlags(&ctx->oov_stream, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->oov_ready, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->oov_done, cudaEventDisableTiming));
    }
    if (p->n_dyn > ctx->oov_cap) {
        if (ctx->oov_dyn) cudaFree(ctx->oov_dyn);
        if (ctx->oov_delta) cudaFree(ctx->oov_delta);
        if (ctx->oov_host) cudaFreeHost(ctx->oov_host);
        ctx->oov_dyn = ctx->oov_delta = ctx->oov_host = nullptr;
        ctx->oov_cap = 0;
        const int cap = std::max(64, p->n_dyn);
        CUDA_TRY(cudaMalloc(&ctx->oov_dyn, (size_t)(cap + 1) * sizeof(int32_t)));
        CUDA_TRY(cudaMalloc(&ctx->oov_delta, (size_t)2 * cap * sizeof(int32_t)));
        CUDA_TRY(cudaMallocHost(&ctx->oov_host, (size_t)(cap + 1) * sizeof(int32_t)));
        ctx->oov_cap = cap;
    }
    // the side stream starts after the work already on the caller's stream (q, seeds)
    CUDA_TRY(cudaEventRecord(ctx->oov_ready, (cudaStream_t)stream));
    CUDA_TRY(cudaStreamWaitEvent(ctx->oov_stream, ctx->oov_ready, 0));
    // the event's candidates: formation with the cap n_dyn (max insertions per event,
    // P:462), static members skipped -- the sorted new ids, as one batched-build sequence
    evospec_status rc = build_impl(ctx, E, n_e_rows, q, static_ids, n_static, seeds, n_seed, row_ptr, col, nullptr, 0,
                                   p, ctx->oov_dyn + 1, ctx->oov_dyn, nullptr, nullptr, ctx->oov_stream, ctx->zero_i);
    if (rc != EVOSPEC_OK) return rc;
    CUDA_TRY(cudaMemcpyAsync(ctx->oov_host, ctx->oov_dyn, (size_t)(p->n_dyn + 1) * sizeof(int32_t),
                             cudaMemcpyDeviceToHost, ctx->oov_stream));
    CUDA_TRY(cudaEventRecord(ctx->oov_done, ctx->oov_stream));
    ctx->oov_pending = true;
    return EVOSPEC_OK;
}

evospec_status evospec_oov_event_end(evospec_ctx* ctx, evospec_arc* arc, int64_t step, const int32_t* subset,
                                    int32_t n, int32_t* out, int32_t* n_out, int32_t* added_host, int32_t* n_added,
                                    int32_t* removed_host, int32_t* n_removed, void* stream) {
    if (!ctx || !arc || !out || !n_out || n < 0 || (n > 0 && !subset))
        return fail(EVOSPEC_EINPUT, "oov_event_end: null / bad argument");
    if (!ctx->oov_pending) return fail(EVOSPEC_EINPUT, "oov_event_end: no event in flight");
    ctx->oov_pending = false;
    CUDA_TRY(cudaEventSynchronize(ctx->oov_done));
    const int cnt = ctx->oov_host[0];
    if (cnt < 0 || cnt > ctx->oov_cap) return fail(EVOSPEC_EINVARIANT, "oov_event_end: candidate count %d", cnt);
    std::vector<int32_t> add(std::max(cnt, 1)), rem(std::max(cnt, 1));
    int32_t na = 0, nr = 0;
    evospec_status rc = evospec_arc_admit_delta(arc, ctx->oov_host + 1, cnt, step, add.data(), &na, rem.data(), &nr);
    if (rc != EVOSPEC_OK) return fail(rc, "oov_event_end: ARC admission failed");
    if (nr > n) return fail(EVOSPEC_EINPUT, "oov_event_end: %d removals from a %d-id subset (not the ARC's subset?)", nr, n);
    cudaStream_t st = (cudaStream_t)stream;
    // (pageable sources: the copies are staged before cudaMemcpyAsync returns)
    if (nr) CUDA_TRY(cudaMemcpyAsync(ctx->oov_delta, rem.data(), (size_t)nr * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    if (na) CUDA_TRY(cudaMemcpyAsync(ctx->oov_delta + ctx->oov_cap, add.data(), (size_t)na * sizeof(int32_t),
                                     cudaMemcpyHostToDevice, st));
    launch_subset_update(subset, n, ctx->oov_delta, nr, ctx->oov_delta + ctx->oov_cap, na, out, n_out,
                         (int32_t*)ctx->flags, st);
    ctx->launches += 1;
    LAUNCH_CHECK("subset_update");
    if (added_host) std::copy(add.begin(), add.begin() + na, added_host);
    if (removed_host) std::copy(rem.begin(), rem.begin() + nr, removed_host);
    if (n_added) *n_added = na;
    if (n_removed) *n_removed = nr;
    return EVOSPEC_OK;
}

evospec_status evospec_build_local_candidates(evospec_ctx* ctx, const void* E_local, int64_t n_e_rows, const void* q,
                                             int32_t n_sem, double* out_s, int32_t* out_id, void* stream) {
    if (!ctx || !E_local || !q || !out_s || !out_id) return fail(EVOSPEC_EINPUT, "build_local_candidates: null argument");
    const evospec_config& c = ctx->cfg;
    const int64_t local_rows = shard_rows(c.V, c.n_shards, c.shard_rank);
    if (n_e_rows != local_rows)
        return fail(EVOSPEC_EINPUT, "build_local_candidates: n_e_rows=%lld, this shard has %lld rows",
                    (long long)n_e_rows, (long long)local_rows);
    if (n_sem < 1 || n_sem > c.max_sem) return fail(EVOSPEC_EINPUT, "build_local_candidates: n_sem not in [1, %d]", c.max_sem);
    return local_candidates_impl(ctx, E_local, n_e_rows, q, n_sem, out_s, out_id, (cudaStream_t)stream);
}

evospec_status evospec_build_subset_from_candidates(evospec_ctx* ctx, const double* cand_s, const int32_t* cand_id,
                                                    int32_t n_cand, const int32_t* static_ids, int32_t n_static,
                                                    const int32_t* seeds, int32_t n_seed, const int32_t* row_ptr,
                                                    const int32_t* col, const int32_t* ctx_ids, int32_t n_ctx,
                                                    const evospec_build_params* p, int32_t* out_ids, int32_t* out_n,
                                                    int32_t* out_local_ids, int32_t* out_local_n, void* stream) {
    if (!cand_s) return fail(EVOSPEC_EINPUT, "build_subset_from_candidates: null candidates");
    return build_impl(ctx, nullptr, 0, nullptr, static_ids, n_static, seeds, n_seed, row_ptr, col, ctx_ids, n_ctx, p,
                      out_ids, out_n, out_local_ids, out_local_n, stream, nullptr, nullptr, cand_s, cand_id, n_cand);
}

evospec_status evospec_build_subset(evospec_ctx* ctx, const void* E, int64_t n_e_rows, const void* q,
                                    const int32_t* static_ids, int32_t n_static, const int32_t* seeds,
                                    int32_t n_seed, const int32_t* row_ptr, const int32_t* col,
                                    const int32_t* ctx_ids, int32_t n_ctx, const evospec_build_params* p,
                                    int32_t* out_ids, int32_t* out_n, int32_t* out_local_ids,
                                    int32_t* out_local_n, void* stream) {
    return build_impl(ctx, E, n_e_rows, q, static_ids, n_static, seeds, n_seed, row_ptr, col, ctx_ids, n_ctx, p,
                      out_ids, out_n, out_local_ids, out_local_n, stream, nullptr);
}

evospec_status evospec_build_subset_batched(evospec_ctx* ctx, const void* E, int64_t n_e_rows, const void* q,
                                            int32_t B, const int32_t* static_ids, int32_t n_static,
                                            const int32_t* seeds, const int32_t* seed_offsets,
                                            const int32_t* row_ptr, const int32_t* col, const int32_t* ctx_ids,
                                            const int32_t* ctx_offsets, const evospec_build_params* p,
                                            int32_t* out_dyn_ids, int32_t* out_dyn_offsets, void* stream) {
    if (!ctx || !q || !p || !out_dyn_ids || !out_dyn_offsets || B < 0 || (B > 0 && !seed_offsets))
        return fail(EVOSPEC_EINPUT, "build_subset_batched: null argument or B < 0");
    if (ctx->cfg.n_shards != 1 || n_e_rows != ctx->cfg.V)
        return fail(EVOSPEC_EINPUT, "build_subset_batched: needs an unsharded context and the full index");
    cudaStream_t st = (cudaStream_t)stream;
    CUDA_TRY(cudaMemsetAsync(out_dyn_offsets, 0, sizeof(int32_t), st));
    const size_t q_bytes = (size_t)ctx->cfg.d * (ctx->cfg.h_dtype == EVOSPEC_BF16 ? 2 : 4);
    for (int b = 0; b < B; ++b) {
        const int s0 = seed_offsets[b], s1 = seed_offsets[b + 1];
        const int c0 = ctx_offsets ? ctx_offsets[b] : 0, c1 = ctx_offsets ? ctx_offsets[b + 1] : 0;
        if (s1 < s0 || c1 < c0) return fail(EVOSPEC_EINPUT, "build_subset_batched: offsets not ascending at %d", b);
        evospec_status rc = build_impl(ctx, E, n_e_rows, (const char*)q + q_bytes * b, static_ids, n_static,
                                       seeds ? seeds + s0 : nullptr, s1 - s0, row_ptr, col,
                                       ctx_ids ? ctx_ids + c0 : nullptr, c1 - c0, p, out_dyn_ids,
                                       out_dyn_offsets + b + 1, nullptr, nullptr, stream, out_dyn_offsets + b);
        if (rc != EVOSPEC_OK) return rc;
    }
    return EVOSPEC_OK;
}

evospec_status evospec_last_scores(evospec_ctx* ctx, double* out_dev, int64_t n, void* stream) {
    if (!ctx || !out_dev || n < 0 || n > ctx->cfg.V) return fail(EVOSPEC_EINPUT, "last_scores: bad argument");
    CUDA_TRY(cudaMemcpyAsync(out_dev, ctx->s64, (size_t)n * sizeof(double), cudaMemcpyDeviceToDevice,
                             (cudaStream_t)stream));
    return EVOSPEC_OK;
}

evospec_status evospec_last_semantic(evospec_ctx* ctx, int32_t* out_dev, int32_t n, void* stream) {
    if (!ctx || !out_dev || n < 0 || n > ctx->cfg.max_sem) return fail(EVOSPEC_EINPUT, "last_semantic: bad argument");
    CUDA_TRY(cudaMemcpyAsync(out_dev, ctx->sem_ids, (size_t)n * 4, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return EVOSPEC_OK;
}

static float gemv_gamma(int d) {
    // recursive-summation bound gamma_n = n u / (1 - n u), u = 2^-24, with the
    // chain length n = d/32 per-lane products + 5 butterfly levels + 1 scale
    const double u = 1.0 / 16777216.0;
    const double n = d / 32.0 + 6.0;
    return (float)(1.01 * n * u / (1.0 - n * u));
}

// Tensor-core path for bf16 trees of >= kTcMinRows rows (FFMA no longer
// keeps pace with HBM there); EVOSPEC_LMH=gemv|tc overrides.
static constexpr int kTcMinRows = 5;
// Accumulation-error envelope of the tcgen05 fp32 accumulator, relative to
// ||h||_2 max||W_v||_2: 2^-16 (~ 256 fp32 roundings); the parity suite checks
// the measured error stays below 1/8 of the resulting delta.
static constexpr float kTcGamma = 1.0f / 65536.0f;

static bool use_tc(const LmhArgs& a) {
    const char* env = getenv("EVOSPEC_LMH");
    if (env && !strcmp(env, "gemv")) return false;
    if (!lmh_tc_supported(a)) return false;
    if (env && !strcmp(env, "tc")) return true;
    return a.n_h >= kTcMinRows;
}

constexpr bool kOverlapDefault = true;    // draft_step static/dynamic LM-head overlap (EVOSPEC_OVERLAP=0: off; step 319 -> 298 us)
constexpr int kRaggedSegRows = 112;   // rows per static segment of the ragged head (measured: 64 887 us, 96 745, 112 710, 128 736 on config Bt)

struct LmhSegs {
    int nseg, seg_ctas, seg_rows;
    const int32_t* seg_pos;   // device [nseg+1] or null (every segment: the whole subset)
    const int32_t* seg_h;     // host [nseg+1]
    const int32_t* seg_cta;   // device [nseg+1] schedule or null (seg_ctas CTAs each)
};

// merged outputs (m_*) non-null: the single-shard merge (LSE, probabilities)
// is fused into the finalisation kernel (used by evospec_draft_step at R = 1)
// Two-list draft step: the union publishes a complete dynamic list before its end
// (EVOSPEC_EARLY_LIST=0: the LM head waits for the union's end)
static bool early_list_enabled() {
    static const bool v = getenv("EVOSPEC_EARLY_LIST") ? atoi(getenv("EVOSPEC_EARLY_LIST")) != 0 : true;
    return v;
}

static evospec_status lmh_impl(evospec_ctx* ctx, const void* W, int64_t n_w_rows, const void* H, int32_t n_h,
                               const int32_t* subset, const int32_t* n_subset_dev, int32_t n_subset_max, int32_t k,
                               float inv_temp, int32_t* topk_ids, float* topk_vals, float* row_max,
                               float* row_sumexp, float* logits_out, void* stream, int32_t* m_ids, float* m_vals,
                               float* m_lse, float* m_probs, const int32_t* seg = nullptr,
                               const LmhSegs* segs = nullptr, const int32_t* list2 = nullptr,
                               const int32_t* n_list2_dev = nullptr, int32_t n_list2_max = 0,
                               int part_cta0 = 0, bool skip_fin = false, const int* fin_a = nullptr) {
    if (!ctx || !W || !H || !subset || (!n_subset_dev && !seg && !list2) || !topk_ids || !topk_vals || !row_max ||
        !row_sumexp)
        return fail(EVOSPEC_EINPUT, "subset_logits_topk: null argument");
    const evospec_config& c = ctx->cfg;
    if (n_h < 1 || n_h > c.max_rows) return fail(EVOSPEC_EINPUT, "subset_logits_topk: n_h=%d not in [1,%d]", n_h, c.max_rows);
    if (k < 1 || k > c.max_k) return fail(EVOSPEC_EINPUT, "subset_logits_topk: k=%d not in [1,%d]", k, c.max_k);
    if (!(inv_temp > 0.0f) || !std::isfinite(inv_temp))
        return fail(EVOSPEC_EINPUT, "subset_logits_topk: inv_temp must be finite and > 0");
    if (n_subset_max < 0 || n_subset_max > c.max_subset)
        return fail(EVOSPEC_EINPUT, "subset_logits_topk: n_subset_max=%d > max_subset %d", n_subset_max, c.max_subset);
    if (n_w_rows < shard_rows(c.V, c.n_shards, c.shard_rank))
        return fail(EVOSPEC_EINPUT, "subset_logits_topk: W_local has %lld rows, shard needs %lld", (long long)n_w_rows,
                    (long long)shard_rows(c.V, c.n_shards, c.shard_rank));
    cudaStream_t st = (cudaStream_t)stream;
    if (c.debug_checks) {
        ctx->launches += 1;
        if (!seg && !list2) launch_check_sorted(subset, n_subset_dev, n_subset_max, c.V, ctx->flags, st);
        LAUNCH_CHECK("check_sorted");
    }
    LmhArgs a{};
    a.W = W; a.n_w_rows = n_w_rows; a.d = c.d; a.w_dtype = c.w_dtype;
    a.H = H; a.n_h = n_h; a.h_dtype = c.h_dtype;
    a.subset = subset; a.n_subset_dev = n_subset_dev; a.n_subset_max = n_subset_max; a.seg = seg;
    a.R = c.n_shards; a.KP = k + kTopkPad; a.LS = a.KP <= 32 ? 64 : a.KP; a.inv_temp = inv_temp;
    // a triple that is merged with other parts (vocabulary shards, or the static /
    // dynamic parts of the ragged head) carries exact top-k values
    a.exact_vals = (c.n_shards > 1 || ((segs || seg) && !fin_a)) ? 1 : 0;
    a.part_cta0 = part_cta0;
    if (fin_a) { a.fin_a_rows = fin_a[0]; a.fin_a_ctas = fin_a[1]; a.fin_a_cta0 = fin_a[2]; }
    a.logits_out = logits_out;
    a.part = ctx->part;
    a.m_ids = m_ids; a.m_vals = m_vals; a.m_lse = m_lse; a.m_probs = m_probs;
    a.par_fold = 1;    // thread-parallel epilogue fold (lmh_epilogue.cuh; the warp fold on single-tile CTAs)
    a.fin_opt = 2;     // finalisation: the candidates' W rows prefetched to L2 for the re-score
    if (list2) {   // two-list mode (draft_step overlap): one SM stays free for the union kernel
        a.list2 = list2; a.n_list2_dev = n_list2_dev; a.n_list2_max = n_list2_max; a.n1 = n_subset_max;
        if (early_list_enabled()) { a.early_ids = ctx->early_ids; a.early_flag = ctx->early_flag; }
        a.grid = lmh_tc_grid() - 1;
        if (!use_tc(a) || a.KP > 32 || segs || seg || logits_out)
            return fail(EVOSPEC_EINPUT, "subset_logits_topk: two-list mode needs the tensor-core path and k + 8 <= 32");
    }
    if (segs) {
        a.nseg = segs->nseg; a.seg_ctas = segs->seg_ctas; a.seg_rows = segs->seg_rows; a.seg_pos = segs->seg_pos;
        a.seg_cta = segs->seg_cta;
        for (int b = 0; b <= segs->nseg; ++b) a.seg_h[b] = segs->seg_h[b];
        if (!use_tc(a)) return fail(EVOSPEC_EINPUT, "segment mode needs the tensor-core path");
    }
    if (getenv("EVOSPEC_TRACE")) {
        if (!ctx->trace) CUDA_TRY(cudaMalloc(&ctx->trace, kTraceLen * sizeof(long long)));
        if (!list2)   // (a memset between the union and a two-list head would break the PDL overlap)
        {
            CUDA_TRY(cudaMemsetAsync(ctx->trace, 0, 2 * kNumSMs * 8 * sizeof(long long), st));
            CUDA_TRY(cudaMemsetAsync(ctx->trace + kTraceOvf, 0, 2 * kNumSMs * sizeof(long long), st));
        }
        a.trace = ctx->trace;
    }
    int n_cta = 0;
    float gamma = gemv_gamma(c.d);
    {
        StageTimer t(ctx, EVOSPEC_STAGE_LMH, st);
        if (use_tc(a)) {
            if (a.KP <= 32) { a.gid_keys = 1; a.LS = kTcListLS; }   // buffered lists: ids, stride 128
            CUDA_TRY(launch_lmh_tc(a, st));
            ctx->launches += 1;
            n_cta = segs ? segs->seg_ctas : (a.grid > 0 ? a.grid : lmh_tc_grid());
            gamma = kTcGamma;
        } else {
            for (int h0 = 0; h0 < n_h;) {
                const int g = lmh_gemv_group_width(a, n_h - h0);
                n_cta = launch_lmh_gemv(a, h0, g, st);
                ctx->launches += 1;
                LAUNCH_CHECK("lmh_gemv");
                h0 += g;
            }
        }
    }
    if (skip_fin) return EVOSPEC_OK;   // (the ragged head's static block: finalised with its dynamic lists)
    {
        StageTimer t(ctx, EVOSPEC_STAGE_FINALIZE, st);
        if (!launch_lmh_finalize(a, n_cta, k, ctx->wmax, topk_ids, topk_vals, row_max, row_sumexp, ctx->flags, st,
                                 gamma))
            return fail(EVOSPEC_EINPUT, "subset_logits_topk: %d partial lists exceed the finalisation's capacity", n_cta);
        ctx->launches += 1;
    }
    LAUNCH_CHECK("lmh_finalize");
    if (c.debug_checks) return evospec_sync_status(ctx, stream);   // (header: EINVARIANT on the product path)
    return EVOSPEC_OK;
}

evospec_status evospec_subset_logits_topk(evospec_ctx* ctx, const void* W, int64_t n_w_rows, const void* H,
                                          int32_t n_h, const int32_t* subset, const int32_t* n_subset_dev,
                                          int32_t n_subset_max, int32_t k, float inv_temp, int32_t* topk_ids,
                                          float* topk_vals, float* row_max, float* row_sumexp, float* logits_out,
                                          void* stream) {
    return lmh_impl(ctx, W, n_w_rows, H, n_h, subset, n_subset_dev, n_subset_max, k, inv_temp, topk_ids, topk_vals,
                    row_max, row_sumexp, logits_out, stream, nullptr, nullptr, nullptr, nullptr);
}

evospec_status evospec_subset_logits_topk_merged(evospec_ctx* ctx, const void* W, int64_t n_w_rows, const void* H,
                                                 int32_t n_h, const int32_t* subset, const int32_t* n_subset_dev,
                                                 int32_t n_subset_max, int32_t k, float inv_temp, int32_t* out_ids,
                                                 float* out_vals, float* out_lse, float* out_probs, float* row_max,
                                                 float* row_sumexp, void* stream) {
    if (!ctx) return fail(EVOSPEC_EINPUT, "subset_logits_topk_merged: null context");
    if (ctx->cfg.n_shards != 1)
        return fail(EVOSPEC_EINPUT, "subset_logits_topk_merged: single-shard contexts only (R = %d)", ctx->cfg.n_shards);
    if (!out_ids || !out_vals || !out_lse) return fail(EVOSPEC_EINPUT, "subset_logits_topk_merged: null output");
    int32_t* tids = ctx->g_ids;   // the shard triple lands in the workspace; the outputs are the merged ones
    float* tvals = ctx->g_vals;
    return lmh_impl(ctx, W, n_w_rows, H, n_h, subset, n_subset_dev, n_subset_max, k, inv_temp, tids, tvals,
                    row_max ? row_max : ctx->g_m, row_sumexp ? row_sumexp : ctx->g_s, nullptr, stream, out_ids,
                    out_vals, out_lse, out_probs);
}

__global__ void set2_kernel(int32_t* p, int32_t a, int32_t b) { p[0] = a; p[1] = b; }

evospec_status evospec_subset_logits_topk_ragged(evospec_ctx* ctx, const void* W, int64_t n_w_rows, const void* H,
                                                 const int32_t* h_offsets, int32_t B, const int32_t* static_ids,
                                                 int32_t n_static, const int32_t* dyn_ids,
                                                 const int32_t* dyn_offsets, int32_t max_dyn, int32_t k,
                                                 float inv_temp, int32_t* topk_ids, float* topk_vals,
                                                 float* row_max, float* row_sumexp, void* stream) {
    if (!ctx || !W || !H || !h_offsets || B < 1 || !topk_ids || !topk_vals || !row_max || !row_sumexp ||
        (n_static > 0 && !static_ids) || !dyn_ids || !dyn_offsets)
        return fail(EVOSPEC_EINPUT, "subset_logits_topk_ragged: null argument or B < 1");
    const evospec_config& c = ctx->cfg;
    if (h_offsets[0] != 0) return fail(EVOSPEC_EINPUT, "subset_logits_topk_ragged: h_offsets[0] must be 0");
    for (int b = 0; b < B; ++b)
        if (h_offsets[b + 1] < h_offsets[b])
            return fail(EVOSPEC_EINPUT, "subset_logits_topk_ragged: h_offsets not ascending at %d", b);
    const int n_rows = h_offsets[B];
    if (n_rows < 1 || n_rows > c.max_rows)
        return fail(EVOSPEC_EINPUT, "subset_logits_topk_ragged: %d rows not in [1, max_rows=%d]", n_rows, c.max_rows);
    if (n_static < 0 || n_static > c.max_subset || max_dyn < 0 || max_dyn > c.max_subset)
        return fail(EVOSPEC_EINPUT, "subset_logits_topk_ragged: n_static / max_dyn exceed max_subset %d", c.max_subset);
    if (k < 1 || k > c.max_k) return fail(EVOSPEC_EINPUT, "subset_logits_topk_ragged: k=%d not in [1,%d]", k, c.max_k);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t row_bytes = (size_t)c.d * (c.h_dtype == EVOSPEC_BF16 ? 2 : 4);
    const size_t hk = (size_t)n_rows * k;
    int32_t* ids1 = ctx->rg_ids + hk;
    float* vals1 = ctx->rg_vals + hk;
    // static block: every row against the shared static set (row groups the
    // tensor-core kernel holds in TMEM)
    set2_kernel<<<1, 1, 0, st>>>(ctx->rg_seg, 0, n_static);
    ctx->launches += 1;
    LAUNCH_CHECK("set2");
    LmhArgs probe{};
    probe.w_dtype = c.w_dtype; probe.h_dtype = c.h_dtype; probe.d = c.d; probe.n_w_rows = n_w_rows;
    probe.KP = k + kTopkPad; probe.n_h = 1;
    const bool seg_ok = lmh_tc_supported(probe) && probe.KP <= 32;
    int max_rows_seq = 0;
    for (int b = 0; b < B; ++b) max_rows_seq = std::max(max_rows_seq, h_offsets[b + 1] - h_offsets[b]);
    // both blocks in segment mode: one finalisation per row reads the row's static-group
    // lists and its sequence's dynamic lists together (no exact re-score of every top-k
    // entry for a merge, no merge launch); the dynamic launch's lists sit behind the static's
    const bool dyn_seg = seg_ok && B <= std::min(kMaxSeg, lmh_tc_grid()) && max_rows_seq <= kTcMaxRows;
    int fin_a[3] = {0, 0, 0};
    if (seg_ok) {
        // static block: one launch, row groups of <= 128 as segments over the same
        // static range (their CTAs read the same W rows at about the same time)
        // rows per static segment: smaller segments leave shared memory for more
        // pipeline stages but stream the static rows more often (swept, kRaggedSegRows)
        const int seg_cap = kRaggedSegRows;
        const int ns = (n_rows + seg_cap - 1) / seg_cap;
        const int per = (n_rows + ns - 1) / ns;
        int sh[kMaxSeg + 1];
        for (int b = 0; b <= ns; ++b) sh[b] = std::min(n_rows, b * per);
        const LmhSegs ss{ns, lmh_tc_grid() / ns, per, nullptr, sh, nullptr};
        evospec_status rc = lmh_impl(ctx, W, n_w_rows, H, n_rows, static_ids ? static_ids : dyn_ids, ctx->rg_seg + 1,
                                     n_static, k, inv_temp, ctx->rg_ids, ctx->rg_vals, ctx->rg_m, ctx->rg_s, nullptr,
                                     stream, nullptr, nullptr, nullptr, nullptr, nullptr, &ss, nullptr, nullptr, 0,
                                     0, dyn_seg);
        if (rc != EVOSPEC_OK) return rc;
        fin_a[0] = per; fin_a[1] = ss.seg_ctas; fin_a[2] = 0;
    } else {
        for (int r0 = 0; r0 < n_rows; r0 += kTcMaxRows) {
            const int g = std::min(kTcMaxRows, n_rows - r0);
            evospec_status rc = lmh_impl(ctx, W, n_w_rows, (const char*)H + row_bytes * r0, g,
                                         static_ids ? static_ids : dyn_ids, nullptr, n_static, k, inv_temp,
                                         ctx->rg_ids + (size_t)r0 * k, ctx->rg_vals + (size_t)r0 * k, ctx->rg_m + r0,
                                         ctx->rg_s + r0, nullptr, stream, nullptr, nullptr, nullptr, nullptr,
                                         ctx->rg_seg);
            if (rc != EVOSPEC_OK) return rc;
        }
    }
    if (dyn_seg) {
        // dynamic blocks: one launch, sequence b = segment b (its rows, its dyn_b)
        // CTAs in proportion to each sequence's dyn_b length (device sizes -> device schedule)
        launch_seg_schedule(dyn_offsets, h_offsets, B, lmh_tc_grid(), ctx->rg_segcta, st);
        ctx->launches += 1;
        LAUNCH_CHECK("seg_schedule");
        const LmhSegs ds{B, lmh_tc_grid() / B, std::max(1, max_rows_seq), dyn_offsets, h_offsets, ctx->rg_segcta};
        return lmh_impl(ctx, W, n_w_rows, H, n_rows, dyn_ids, nullptr, max_dyn, k, inv_temp, topk_ids, topk_vals,
                        row_max, row_sumexp, nullptr, stream, nullptr, nullptr, nullptr, nullptr, ctx->rg_seg, &ds,
                        nullptr, nullptr, 0, lmh_tc_grid(), false, fin_a);
    } else {
        for (int b = 0; b < B; ++b) {
            const int r0 = h_offsets[b], g = h_offsets[b + 1] - r0;
            if (g == 0) continue;
            evospec_status rc = lmh_impl(ctx, W, n_w_rows, (const char*)H + row_bytes * r0, g, dyn_ids, nullptr,
                                         max_dyn, k, inv_temp, ids1 + (size_t)r0 * k, vals1 + (size_t)r0 * k,
                                         ctx->rg_m + n_rows + r0, ctx->rg_s + n_rows + r0, nullptr, stream, nullptr,
                                         nullptr, nullptr, nullptr, dyn_offsets + b);
            if (rc != EVOSPEC_OK) return rc;
        }
    }
    // static u dynamic are disjoint: the two triples merge like two vocabulary shards
    launch_merge(2, n_rows, k, ctx->rg_ids, ctx->rg_vals, ctx->rg_m, ctx->rg_s, topk_ids, topk_vals, nullptr, nullptr,
                 st, row_max, row_sumexp);
    ctx->launches += 1;
    LAUNCH_CHECK("merge");
    return EVOSPEC_OK;
}

evospec_status evospec_merge_shards(evospec_ctx* ctx, int32_t n_h, int32_t k, const int32_t* ids, const float* vals,
                                    const float* m, const float* s, int32_t* out_ids, float* out_vals, float* out_lse,
                                    float* out_probs, void* stream) {
    if (!ctx || !ids || !vals || !m || !s || !out_ids || !out_vals || !out_lse)
        return fail(EVOSPEC_EINPUT, "merge_shards: null argument");
    const evospec_config& c = ctx->cfg;
    if (n_h < 1 || n_h > c.max_rows || k < 1 || k > c.max_k)
        return fail(EVOSPEC_EINPUT, "merge_shards: n_h=%d / k=%d out of capacity", n_h, k);
    const int R = c.n_shards;
    if (R * k > 64 * 32) return fail(EVOSPEC_EINPUT, "merge_shards: R*k > 2048");
    cudaStream_t st = (cudaStream_t)stream;
    StageTimer t_merge(ctx, EVOSPEC_STAGE_MERGE, st);
    const int32_t* gi = ids;
    const float *gv = vals, *gm = m, *gs = s;
    if (ctx->comm && R > 1) {
        NcclApi& n = nccl();
        const size_t nk = (size_t)n_h * k;
        n.GroupStart();
        ncclResult_t r1 = n.AllGather(ids, ctx->g_ids, nk, ncclInt32, ctx->comm, st);
        ncclResult_t r2 = n.AllGather(vals, ctx->g_vals, nk, ncclFloat32, ctx->comm, st);
        ncclResult_t r3 = n.AllGather(m, ctx->g_m, (size_t)n_h, ncclFloat32, ctx->comm, st);
        ncclResult_t r4 = n.AllGather(s, ctx->g_s, (size_t)n_h, ncclFloat32, ctx->comm, st);
        ncclResult_t r5 = n.GroupEnd();
        if (r1 || r2 || r3 || r4 || r5) return fail(EVOSPEC_ENCCL, "merge_shards: all-gather failed");
        gi = ctx->g_ids; gv = ctx->g_vals; gm = ctx->g_m; gs = ctx->g_s;
    }
    launch_merge(R, n_h, k, gi, gv, gm, gs, out_ids, out_vals, out_lse, out_probs, st);
    ctx->launches += 1;
    LAUNCH_CHECK("merge");
    return EVOSPEC_OK;
}

evospec_status evospec_verify_chain(evospec_ctx* ctx, const float* target_logits, int32_t V, int32_t g,
                                    const int32_t* proposals, const int32_t* subset_ids, int32_t n_subset,
                                    const float* draft_probs, float inv_temp, int32_t greedy, const double* u,
                                    const double* w, int32_t* tokens, int32_t* n_accepted, void* stream) {
    if (!ctx || !target_logits || !tokens || !n_accepted || (g > 0 && !proposals))
        return fail(EVOSPEC_EINPUT, "verify_chain: null argument");
    if (V < 1 || g < 0 || g > kMaxChain) return fail(EVOSPEC_EINPUT, "verify_chain: V=%d / g=%d out of range", V, g);
    if (!(inv_temp > 0.0f) || !std::isfinite(inv_temp)) return fail(EVOSPEC_EINPUT, "verify_chain: inv_temp must be > 0");
    if (!greedy && (!w || (g > 0 && (!u || !subset_ids || !draft_probs || n_subset < 1))))
        return fail(EVOSPEC_EINPUT, "verify_chain: sampling mode needs the subset, draft_probs, u and w");
    cudaStream_t st = (cudaStream_t)stream;
    launch_verify(target_logits, V, g, proposals, subset_ids, n_subset, draft_probs, (double)inv_temp, greedy ? 1 : 0,
                  u, w, ctx->ver_acc, ctx->ver_tok, tokens, n_accepted, ctx->flags, st);
    ctx->launches += 2;
    LAUNCH_CHECK("verify_chain");
    return EVOSPEC_OK;
}

evospec_status evospec_coverage(evospec_ctx* ctx, const float* target_logits, int32_t n_rows, int32_t V,
                                const int32_t* subset_ids, int32_t n_subset, float inv_temp, const int32_t* ks,
                                int32_t n_ks, double* covered_mass, double* recall, void* stream) {
    if (!ctx || !target_logits || !covered_mass || (n_subset > 0 && !subset_ids) || (n_ks > 0 && (!ks || !recall)))
        return fail(EVOSPEC_EINPUT, "coverage: null argument");
    if (n_rows < 0 || V < 1 || n_subset < 0 || n_subset > V || n_ks < 0 || n_ks > 64)
        return fail(EVOSPEC_EINPUT, "coverage: n_rows=%d / V=%d / n_subset=%d / n_ks=%d out of range", n_rows, V,
                    n_subset, n_ks);
    if (!(inv_temp > 0.0f) || !std::isfinite(inv_temp)) return fail(EVOSPEC_EINPUT, "coverage: inv_temp must be > 0");
    if (n_rows == 0) return EVOSPEC_OK;
    launch_coverage(target_logits, n_rows, V, subset_ids, n_subset, (double)inv_temp, ks, n_ks, covered_mass, recall,
                    ctx->flags,
                    (cudaStream_t)stream);
    ctx->launches += 1;
    LAUNCH_CHECK("coverage");
    return EVOSPEC_OK;
}

evospec_status evospec_kd_loss(evospec_ctx* ctx, int32_t B, int32_t g, int32_t K, const float* target_logits,
                               const float* draft_logits, const int32_t* verified, float T_kd, float beta,
                               float* loss, float* grad, float* weights, void* stream) {
    if (!ctx || !target_logits || !draft_logits || !verified || !loss) return fail(EVOSPEC_EINPUT, "kd_loss: null argument");
    if (B < 0 || g < 1 || g > 32 || K < 1 || K > 1024)
        return fail(EVOSPEC_EINPUT, "kd_loss: B=%d / g=%d / K=%d out of range (g <= 32, K <= 1024)", B, g, K);
    if (!(T_kd > 0.0f) || !std::isfinite(T_kd) || !(beta >= 0.0f) || !std::isfinite(beta))
        return fail(EVOSPEC_EINPUT, "kd_loss: T_kd must be > 0 and beta >= 0");
    if (B == 0) return EVOSPEC_OK;
    launch_kd_loss(B, g, K, target_logits, draft_logits, verified, T_kd, beta, loss, grad, weights, ctx->flags,
                   (cudaStream_t)stream);
    ctx->launches += 1;
    LAUNCH_CHECK("kd_loss");
    return EVOSPEC_OK;
}

// The draft step's two-list mode (single shard, tensor-core head): the LM head streams
// the static rows while the union forms the dynamic list
static bool step_overlap(const evospec_ctx* ctx, const evospec_step_io* io) {
    const evospec_config& c = ctx->cfg;
    static const bool ov_env = getenv("EVOSPEC_OVERLAP") ? atoi(getenv("EVOSPEC_OVERLAP")) != 0 : kOverlapDefault;
    return ov_env && c.n_shards == 1 && c.w_dtype == EVOSPEC_BF16 && c.h_dtype == EVOSPEC_BF16 && c.d % 64 == 0 &&
           io->n_h >= kTcMinRows && io->n_h <= kTcMaxRows && io->k + kTopkPad <= 32 && io->n_static > 0 &&
           !c.debug_checks && !getenv("EVOSPEC_LMH");
}

// phases: 1 host->device staging, 2 the compute (build + LM head + merge), 4 device->host
static evospec_status draft_step_impl(evospec_ctx* ctx, const evospec_step_io* io, cudaStream_t st,
                                      int phases = 7) {
    const evospec_config& c = ctx->cfg;
    if (io->n_h < 1 || io->n_h > c.max_rows || io->n_seed < 0 || io->n_seed > c.max_seeds || io->n_ctx < 0 ||
        io->n_ctx > c.max_ctx || !io->q || !io->H || !io->out_ids || !io->out_vals || !io->out_lse)
        return fail(EVOSPEC_EINPUT, "draft_step: bad I/O arguments");
    if (c.n_shards > 1 && !ctx->comm) return fail(EVOSPEC_EINPUT, "draft_step: sharded context needs evospec_comm_init");
    const size_t hb = c.h_dtype == EVOSPEC_BF16 ? 2 : 4;
    const void *q = io->q, *H = io->H;
    const int32_t *seeds = io->seeds, *cx = io->ctx_ids;
    if (io->host_io && !ctx->s_h) {
        CUDA_TRY(cudaStreamCreateWithFlags(&ctx->s_h, cudaStreamNonBlocking));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&ctx->ev_h, cudaEventDisableTiming));
    }
    if (io->host_io && (phases & 1)) {
        StageTimer t(ctx, EVOSPEC_STAGE_COPY, st);
        // H is needed only by the LM head: its copy runs on a side stream under the build;
        // in two-list mode the seeds too (only the union reads them, after waiting for it)
        const bool seeds_side = step_overlap(ctx, io);
        CUDA_TRY(cudaEventRecord(ctx->ev_in, st));
        CUDA_TRY(cudaStreamWaitEvent(ctx->s_h, ctx->ev_in, 0));
        CUDA_TRY(cudaMemcpyAsync(ctx->st_q, io->q, (size_t)c.d * hb, cudaMemcpyHostToDevice, st));
        if (io->n_seed > 0 && seeds_side)
            CUDA_TRY(cudaMemcpyAsync(ctx->st_seeds, io->seeds, (size_t)io->n_seed * 4, cudaMemcpyHostToDevice, ctx->s_h));
        CUDA_TRY(cudaMemcpyAsync(ctx->st_H, io->H, (size_t)io->n_h * c.d * hb, cudaMemcpyHostToDevice, ctx->s_h));
        CUDA_TRY(cudaEventRecord(ctx->ev_h, ctx->s_h));
        if (io->n_seed > 0 && !seeds_side)
            CUDA_TRY(cudaMemcpyAsync(ctx->st_seeds, io->seeds, (size_t)io->n_seed * 4, cudaMemcpyHostToDevice, st));
        if (io->n_ctx > 0 && io->ctx_ids)
            CUDA_TRY(cudaMemcpyAsync(ctx->st_ctx, io->ctx_ids, (size_t)io->n_ctx * 4, cudaMemcpyHostToDevice, st));
    }
    if (io->host_io) { q = ctx->st_q; H = ctx->st_H; seeds = ctx->st_seeds; cx = io->ctx_ids ? ctx->st_ctx : nullptr; }
    const size_t hk_io = (size_t)io->n_h * io->k;
    float* const st_v = (float*)(ctx->st_oids + hk_io);   // the staging block's layout for this call
    float* const st_l = st_v + hk_io;
    float* const st_p = st_l + io->n_h;
    int32_t* oi = io->host_io ? ctx->st_oids : io->out_ids;
    float* ov = io->host_io ? st_v : io->out_vals;
    float* ol = io->host_io ? st_l : io->out_lse;
    float* op = io->host_io ? (io->out_probs ? st_p : nullptr) : io->out_probs;
    if (phases & 2) {
    // overlap (single shard, tensor-core head): the union writes only the dynamic list and
    // the LM head streams the static rows (an input) while the union still runs, then the
    // dynamic rows (two-list mode, lmh_tc.cu)
    const bool overlap = step_overlap(ctx, io);
    if (overlap) {
        // the host-staged H (side stream, under the scan) is waited for before the union,
        // so the union -> LM head PDL edge stays intact
        evospec_status s = build_impl(ctx, io->E, io->n_e_rows, q, io->static_ids, io->n_static, seeds, io->n_seed,
                                      io->csr_row_ptr, io->csr_col, cx, io->n_ctx, &io->build, ctx->st_S, ctx->st_nS,
                                      nullptr, nullptr, st, ctx->zero_i, io->host_io ? ctx->ev_h : nullptr,
                                      nullptr, nullptr, 0, early_list_enabled());
        if (s != EVOSPEC_OK) return s;
        s = lmh_impl(ctx, io->W_local, io->n_w_rows, H, io->n_h, io->static_ids, nullptr, io->n_static, io->k,
                     io->inv_temp, ctx->st_tids, ctx->st_tvals, ctx->st_m, ctx->st_s, nullptr, st, oi, ov, ol, op,
                     nullptr, nullptr, ctx->st_S, ctx->st_nS, io->build.n_dyn);
        if (s != EVOSPEC_OK) return s;
    } else {
    const int n_sub_max = io->n_static + io->build.n_dyn;
    evospec_status s = evospec_build_subset(ctx, io->E, io->n_e_rows, q, io->static_ids, io->n_static, seeds,
                                            io->n_seed, io->csr_row_ptr, io->csr_col, cx, io->n_ctx, &io->build,
                                            ctx->st_S, ctx->st_nS, c.n_shards > 1 ? ctx->st_local : nullptr,
                                            c.n_shards > 1 ? ctx->st_nlocal : nullptr, st);
    if (s != EVOSPEC_OK) return s;
    const int32_t* sub = c.n_shards > 1 ? ctx->st_local : ctx->st_S;
    const int32_t* nsub = c.n_shards > 1 ? ctx->st_nlocal : ctx->st_nS;
    if (io->host_io) {   // the staged H (side stream) before the LM head
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(st, &cs);
        CUDA_TRY(cudaStreamWaitEvent(st, ctx->ev_h, cs == cudaStreamCaptureStatusActive ? cudaEventWaitExternal : 0));
    }
    const bool fuse = c.n_shards == 1;    // single shard: the merge is the finalisation itself
    s = lmh_impl(ctx, io->W_local, io->n_w_rows, H, io->n_h, sub, nsub, n_sub_max, io->k, io->inv_temp, ctx->st_tids,
                 ctx->st_tvals, ctx->st_m, ctx->st_s, nullptr, st, fuse ? oi : nullptr, fuse ? ov : nullptr,
                 fuse ? ol : nullptr, fuse ? op : nullptr);
    if (s != EVOSPEC_OK) return s;
    if (!fuse) {
        s = evospec_merge_shards(ctx, io->n_h, io->k, ctx->st_tids, ctx->st_tvals, ctx->st_m, ctx->st_s, oi, ov, ol,
                                 op, st);
        if (s != EVOSPEC_OK) return s;
    }
    }   // !overlap
    }   // phases & 2
    if (io->host_io && (phases & 4)) {
        StageTimer t(ctx, EVOSPEC_STAGE_COPY, st);
        const size_t hk = (size_t)io->n_h * io->k;
        const char* hb0 = (const char*)io->out_ids;
        const bool one_block = (const char*)io->out_vals == hb0 + hk * 4 &&
                               (const char*)io->out_lse == hb0 + hk * 8 &&
                               (!io->out_probs || (const char*)io->out_probs == hb0 + hk * 8 + (size_t)io->n_h * 4);
        if (one_block) {
            CUDA_TRY(cudaMemcpyAsync(io->out_ids, oi, hk * 8 + (size_t)io->n_h * 4 + (io->out_probs ? hk * 4 : 0),
                                     cudaMemcpyDeviceToHost, st));
        } else {
            CUDA_TRY(cudaMemcpyAsync(io->out_ids, oi, hk * 4, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(io->out_vals, ov, hk * 4, cudaMemcpyDeviceToHost, st));
            CUDA_TRY(cudaMemcpyAsync(io->out_lse, ol, (size_t)io->n_h * 4, cudaMemcpyDeviceToHost, st));
            if (io->out_probs) CUDA_TRY(cudaMemcpyAsync(io->out_probs, op, hk * 4, cudaMemcpyDeviceToHost, st));
        }
    }
    return EVOSPEC_OK;
}

// The whole step as one CUDA graph (single shard): captured on the context's
// own stream the first time an I/O descriptor is seen, replayed while the
// descriptor (pointers, sizes, parameters) stays the same -- one launch instead
// of ~10 kernel launches, copies and memsets per step. Timing / tracing /
// debug checks and sharded contexts take the direct path.
evospec_status evospec_draft_step(evospec_ctx* ctx, const evospec_step_io* io, void* stream) {
    if (!ctx || !io) return fail(EVOSPEC_EINPUT, "draft_step: null argument");
    cudaStream_t st = (cudaStream_t)stream;
    // sharded steps are captured too (NCCL all-gathers are capturable); if a capture
    // fails the context falls back to direct launches for good
    const bool use_graph = !ctx->no_graph && !ctx->timing && !ctx->cfg.debug_checks &&
                           (ctx->cfg.n_shards == 1 || ctx->comm) && !getenv("EVOSPEC_NO_GRAPH") &&
                           !getenv("EVOSPEC_TRACE");
    if (!use_graph) return draft_step_impl(ctx, io, st);
    // host staging copies stay ordinary stream copies (measured faster than graph
    // memcpy nodes from pinned memory); the graph holds the compute
    if (ctx->g_exec && memcmp(&ctx->g_key, io, sizeof(*io)) == 0) {
        evospec_status s0 = draft_step_impl(ctx, io, st, 1);
        if (s0 != EVOSPEC_OK) return s0;
        CUDA_TRY(cudaGraphLaunch(ctx->g_exec, st));
        ctx->launches += ctx->g_launches;
        return draft_step_impl(ctx, io, st, 4);
    }
    if (!ctx->cap_stream) CUDA_TRY(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    const long long l0 = ctx->launches;
    CUDA_TRY(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    evospec_status s = draft_step_impl(ctx, io, ctx->cap_stream, 2);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(ctx->cap_stream, &g);
    if (s != EVOSPEC_OK || e != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        if (ctx->cfg.n_shards > 1) {   // (a communicator that cannot be captured: run direct from now on)
            cudaGetLastError();
            ctx->no_graph = true;
            return draft_step_impl(ctx, io, st);
        }
        if (s != EVOSPEC_OK) return s;
        return fail(EVOSPEC_ECUDA, "draft_step: graph capture failed: %s", cudaGetErrorString(e));
    }
    if (ctx->g_exec) { cudaGraphExecDestroy(ctx->g_exec); ctx->g_exec = nullptr; }
    const cudaError_t ei = cudaGraphInstantiate(&ctx->g_exec, g, 0);
    cudaGraphDestroy(g);
    if (ei != cudaSuccess) { ctx->g_exec = nullptr; return fail(EVOSPEC_ECUDA, "draft_step: %s", cudaGetErrorString(ei)); }
    memcpy(&ctx->g_key, io, sizeof(*io));
    ctx->g_launches = ctx->launches - l0;
    s = draft_step_impl(ctx, io, st, 1);
    if (s != EVOSPEC_OK) return s;
    CUDA_TRY(cudaGraphLaunch(ctx->g_exec, st));
    return draft_step_impl(ctx, io, st, 4);
}

evospec_status evospec_set_timing(evospec_ctx* ctx, int enable) {
    if (!ctx) return fail(EVOSPEC_EINPUT, "set_timing: null");
    if (enable && ctx->ev.empty()) {
        CUDA_TRY(cudaSetDevice(ctx->device));
        ctx->ev.resize((size_t)EVOSPEC_NUM_STAGES * kTimingSlots * 2);
        for (auto& e : ctx->ev) CUDA_TRY(cudaEventCreate(&e));
    }
    if (enable)
        for (int i = 0; i < EVOSPEC_NUM_STAGES; ++i) ctx->ev_count[i] = 0;
    ctx->timing = enable != 0;
    return EVOSPEC_OK;
}

evospec_status evospec_read_stats(evospec_ctx* ctx, evospec_stats* out) {
    if (!ctx || !out) return fail(EVOSPEC_EINPUT, "read_stats: null");
    memset(out, 0, sizeof(*out));
    out->launches = ctx->launches;
    for (int s = 0; s < EVOSPEC_NUM_STAGES; ++s) {
        out->calls[s] = ctx->ev_count[s];
        double sum = 0.0;
        for (int i = 0; i < ctx->ev_count[s]; ++i) {
            cudaEvent_t a = ctx->ev[((size_t)s * kTimingSlots + i) * 2], b = ctx->ev[((size_t)s * kTimingSlots + i) * 2 + 1];
            CUDA_TRY(cudaEventSynchronize(b));
            float ms = 0.0f;
            CUDA_TRY(cudaEventElapsedTime(&ms, a, b));
            sum += ms;
        }
        out->stage_ms[s] = (float)sum;
    }
    return EVOSPEC_OK;
}

evospec_status evospec_read_trace(evospec_ctx* ctx, int64_t* host_out, int32_t n) {
    if (!ctx || !host_out || n < 0 || n > kTraceLen) return fail(EVOSPEC_EINPUT, "read_trace: bad argument");
    if (!ctx->trace) return fail(EVOSPEC_EINPUT, "read_trace: run with EVOSPEC_TRACE=1");
    CUDA_TRY(cudaMemcpy(host_out, ctx->trace, (size_t)n * sizeof(long long), cudaMemcpyDeviceToHost));
    return EVOSPEC_OK;
}

}  // extern "C"
