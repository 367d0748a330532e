// kernels.cuh -- launch interface between api.cu and the kernel files.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace es {

constexpr int kScanWarps = 16;      // sem scan: warps per CTA (1 CTA / SM)
constexpr int kSelThreads = 512;    // topn candidates (PDL, soft grid barrier), 4096 bins = 8 / thread
constexpr int kHistBins = 4096;     // top 12 bits of the fp32 score key
constexpr int kUnionThreads = 1024;
constexpr int kTopkPad = 8;         // extra fp32 candidates kept per row for the exact re-score
constexpr int kMaxK = 64;
constexpr int kMaxKP = kMaxK + kTopkPad;
constexpr int kTcListLS = 128;      // list stride of the tensor-core head's candidate lists (k + 8 <= 32)
constexpr int kMaxCtx = 8192;

// device flag bits (mirror EVOSPEC_FLAG_* in include/evospec.h)
constexpr int kFlagBadIds = 0x1;
constexpr int kFlagUncertified = 0x2;
constexpr int kFlagSelectOverflow = 0x4;
constexpr int kFlagBudget = 0x8;

// ---- semantic (sem.cu)
void set_step_trace(long long* p);   // EVOSPEC_TRACE stamps of the scan / candidate kernels
void launch_sem_scan(const void* E, int e_dtype, int64_t n_rows, int d, const void* q, int q_dtype,
                     double* s64, uint32_t* key32, uint32_t* hist12, cudaStream_t st, uint32_t* zero_w = nullptr,
                     int n_zero_w = 0, int* zero_c = nullptr, bool hist_zero = false,
                     int* sched = nullptr);   // sched: 2 ints, zero (the TMA scan's stage counter)
cudaError_t launch_topn_cand(const double* s64, const int32_t* ids, int64_t n, int id_mul, int id_add,
                             int N, int cap, const uint32_t* hist_pre, uint32_t* hist_g, int* out_count,
                             double* out_s, int32_t* out_id, cudaStream_t st, bool prezeroed = false);

// ---- union / formation (union.cu)
void launch_ctx_select(const int32_t* ctx, int n_ctx, int V, int min_count, int n_max,
                       int32_t* out, int* out_n, int* flags, cudaStream_t st);
int union_cand_cap(int V, int per_seed);
void launch_static_bits(const int32_t* static_ids, int n_static, int V, int debug, uint32_t* sbits, int* flags,
                        cudaStream_t st);
void launch_union(int V, const int32_t* static_ids, int n_static, const int32_t* seeds, int n_seed,
                  const double* cand_s, const int32_t* cand_id, const int* n_cand_dev, int cap, int n_sem,
                  const int32_t* row_ptr, const int32_t* col,
                  const int32_t* ctx_sel, const int* n_ctx_sel_dev,
                  int n_graph_sem_seeds, int per_seed, int n_dyn, int R, int r,
                  int32_t* out_ids, int32_t* out_n, int32_t* out_local, int32_t* out_local_n,
                  int32_t* sem_out, int* sem_out_n, int debug, int* flags, cudaStream_t st,
                  long long* trace = nullptr, const int32_t* dyn_base = nullptr,
                  uint32_t* clear_hist = nullptr, uint32_t* emit_bits = nullptr, uint32_t* sbits = nullptr,
                  int32_t* early_ids = nullptr, int* early_flag = nullptr);
void launch_union_emit(const uint32_t* bits, int V, int32_t* out_ids, int32_t* out_n, int32_t* out_local,
                       int32_t* out_local_n, int budget_max, int* flags, cudaStream_t st);

// ---- LM head (lmh_gemv.cu, lmh_tc.cu)
// Per-CTA partial state of the LM head, per H row: entries [0, cnt) are the
// CTA's best candidates sorted by (z desc, id asc); entries [cnt, cnt + xcnt)
// are unsorted extras from the CTA's last tile that beat entry KP-1 of the
// sorted list (the last tile is not folded, its survivors are appended).
constexpr int kMaxSeg = 128;
// EVOSPEC_TRACE: per-CTA counters of rows whose candidate buffer overflowed in the
// LM head's last tile / a middle tile (profiling aid), after the timestamp slots
constexpr int kTraceOvf = 2 * 148 * 8 + 16 + 32 + 64 + 2 * 148 + 8;     // segments of one segment-mode LM-head launch

struct LmhPartials {
    float* val;    // [n_cta][n_h][LS]
    int32_t* id;   // [n_cta][n_h][LS] keys: subset positions (sorted subset: position order = id order) or ids
    float* m;      // [n_h][cs]  (row-major by H row: a row's states are contiguous for the finalisation)
    float* s;      // [n_h][cs]
    int* cnt;      // [n_h][cs] sorted entries
    int* xcnt;     // [n_h][cs] unsorted extras
    int cs;        // CTA stride of the state arrays (the context's CTA capacity)
};
// index of CTA cta's softmax / count state for H row `row`
__host__ __device__ inline size_t part_st(const LmhPartials& P, int cta, int row) { return (size_t)row * P.cs + cta; }
struct LmhArgs {
    const void* W; int64_t n_w_rows; int d; int w_dtype;
    const void* H; int n_h; int h_dtype;
    const int32_t* subset; const int* n_subset_dev; int n_subset_max;
    const int32_t* seg;   // optional device [2]: positions [seg[0], seg[1]) of subset (ragged segments)
    // segment mode (tensor-core path, nseg > 0): segment b = H rows [seg_h[b], seg_h[b+1])
    // against subset positions [seg_pos[b], seg_pos[b+1]) (seg_pos == null: every
    // segment takes the whole subset); seg_ctas CTAs per segment, CTA c serves
    // segment c / seg_ctas (the rest idle); n_h = total rows, seg_rows = max rows
    int exact_vals;   // re-score every top-k entry (the triple feeds a cross-part merge)
    int nseg, seg_ctas, seg_rows;
    const int32_t* seg_pos;
    const int32_t* seg_cta;   // optional device [nseg+1]: CTAs [seg_cta[b], seg_cta[b+1]) serve segment b
    int seg_h[kMaxSeg + 1];
    int R; int KP; int LS; float inv_temp;   // LS: list stride (KP <= 32: 64, else KP)
    float* logits_out;  // optional [n_h][n_subset_max]
    long long* trace;   // optional per-CTA globaltimer stamps [n_cta][8] (profiling)
    // optional fused single-shard merge outputs (R = 1): ids/vals [n_h][k], lse [n_h], probs [n_h][k]
    int32_t* m_ids; float* m_vals; float* m_lse; float* m_probs;
    LmhPartials part;
    int fin_opt;    // finalisation options (bits): 2 = W rows of the candidates prefetched to L2
    int par_fold;   // thread-parallel tile fold (lmh_epilogue.cuh epi_par_*), buffered path
    // two-list mode (draft_step overlap): `subset` holds n1 ids known at launch (the static
    // core, an input) and `list2` the ids produced by the previous kernel (the dynamic
    // list, n_list2_dev on the device); partials carry virtual positions vp (vp < n1: subset
    // [vp], else list2[vp - n1]); the tensor-core kernel streams its slice of the first list
    // before griddepcontrol.wait. grid: CTAs of the launch (0 = all SMs)
    const int32_t* list2; const int32_t* n_list2_dev; int n_list2_max; int n1;
    // two-list mode, early second list: the union publishes the complete dynamic list
    // (unsorted) at early_ids with *early_flag = length + 1 before its end, or -1 (wait
    // for the end: list2 / n_list2_dev); the finalisation resets the flag to 0
    const int32_t* early_ids; int* early_flag;
    int grid;
    int part_cta0;   // list / state index of this launch's CTA 0 (a second launch writes behind the first)
    // the finalisation of the ragged head reads two list ranges per row: its launch's segment
    // (the dynamic lists) and, when fin_a_rows > 0, static row group r / fin_a_rows, whose
    // fin_a_ctas lists start at fin_a_cta0 + group * fin_a_ctas
    int fin_a_rows, fin_a_ctas, fin_a_cta0;
    int gid_keys;   // partial lists carry vocabulary ids, not subset positions (tensor-core
                    // kernel, buffered lists; ties then order by id in two-list mode too)
};

// This CTA's contiguous share [p0, p1) of the subset positions: all of
// [0, min(*n_subset_dev, n_subset_max)), or the segment [seg[0], seg[1]).
// Positions stay absolute, so partial lists and the finalisation index
// a.subset directly.
// vocabulary id of a (virtual) subset position
__device__ __forceinline__ int32_t lmh_id_at(const LmhArgs& a, int vp) {
    return (a.list2 && vp >= a.n1) ? __ldg(&a.list2[vp - a.n1]) : __ldg(&a.subset[vp]);
}

__device__ __forceinline__ void lmh_cta_range(const LmhArgs& a, int& p0, int& p1) {
    int s0 = 0, s1;
    if (a.seg) {
        s0 = a.seg[0];
        s1 = s0 + min(a.seg[1] - s0, a.n_subset_max);
    } else {
        s1 = min(*a.n_subset_dev, a.n_subset_max);
    }
    const int n = max(0, s1 - s0);
    p0 = s0 + (int)((long long)n * blockIdx.x / gridDim.x);
    p1 = s0 + (int)((long long)n * (blockIdx.x + 1) / gridDim.x);
}

// returns the number of CTAs whose partials were written
int launch_lmh_gemv(const LmhArgs& a, int h_row0, int n_h_grp, cudaStream_t st);
int lmh_gemv_grid();
int lmh_gemv_group_width(const LmhArgs& a, int n_left);
constexpr int kTcMaxRows = 128;
constexpr int kMaxChain = 63;   // verification: longest draft chain (the paper's horizon is 6)
void launch_kd_loss(int B, int g, int K, const float* zp, const float* zq, const int32_t* verified, float T,
                    float beta, float* J, float* grad, float* w_out, int* flags, cudaStream_t st);
void launch_coverage(const float* z, int n_rows, int V, const int32_t* S, int n_S, double it, const int32_t* ks,
                     int n_ks, double* mass, double* recall, int* flags, cudaStream_t st);
void launch_verify(const float* z, int V, int g, const int32_t* x, const int32_t* S, int n_S, const float* qS,
                   double it, int greedy, const double* u, const double* w, int32_t* pos_acc, int32_t* pos_tok,
                   int32_t* tokens, int32_t* n_acc_out, int* flags, cudaStream_t st);
void launch_subset_update(const int32_t* S, int n, const int32_t* rem, int nr, const int32_t* add, int na,
                          int32_t* out, int32_t* n_out, int32_t* flags, cudaStream_t st);
bool lmh_tc_supported(const LmhArgs& a);
int lmh_tc_grid();
cudaError_t launch_lmh_tc(const LmhArgs& a, cudaStream_t st);

// ---- finalize / merge / prepare (finalize.cu)
bool launch_lmh_finalize(const LmhArgs& a, int n_cta, int k, const float* wmax_dev,
                         int32_t* topk_ids, float* topk_vals, float* row_max, float* row_sumexp,
                         int* flags, cudaStream_t st, float gamma);
struct SegRows { int h[kMaxSeg + 1]; };
void launch_seg_schedule(const int32_t* seg_pos, const int32_t* seg_h_host, int nseg, int grid, int32_t* seg_cta,
                         cudaStream_t st);
void launch_merge(int R, int n_h, int k, const int32_t* ids, const float* vals, const float* m,
                  const float* s, int32_t* out_ids, float* out_vals, float* out_lse, float* out_probs,
                  cudaStream_t st, float* out_m = nullptr, float* out_s = nullptr);
void launch_rownorm_max(const void* W, int w_dtype, int64_t n_rows, int d, float* out, cudaStream_t st);
void launch_check_sorted(const int32_t* ids, const int* n_dev, int n_host, int V, int* flags,
                         cudaStream_t st);

}  // namespace es
