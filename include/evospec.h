/*
 * evospec.h -- C ABI of libevospec.so, the B200 (sm_100a) hot path of
 * EvoSpec's dynamic-vocabulary draft LM head (arXiv 2605.27390).
 *
 * The path (PAPER.md = P:n, SPEC.md = S:n):
 *   evospec_build_subset        a1-a4  V_t = V_static u S_sem(h) u S_graph(.)
 *                                       (Eq. vocab_union; runtime
 *                                       formation P:458; budget P:60)
 *   evospec_subset_logits_topk  a5-a7  z = (H . W[V_t]^T) * inv_temp, fused
 *                                       online softmax (m, s) and top-k
 *                                       (Eq. projection; alg:evospec
 *                                       "restricted to V_t" P:364)
 *   evospec_merge_shards        a8     vocab-shard merge of (top-k, m, s)
 *                                       triples (north star; NCCL all-gather
 *                                       when the context owns a communicator)
 *
 * Conventions (all entry points):
 *   - Plain pointers and sizes only. "dev" pointers are CUDA device memory
 *     owned by the CALLER (the library never frees them); "host" pointers are
 *     host memory. Every call is asynchronous on the given stream (a
 *     cudaStream_t passed as void*; NULL = legacy default stream) and performs
 *     no host synchronisation unless stated.
 *   - Layouts are row-major, contiguous, little-endian. bf16 is stored as its
 *     16-bit pattern. Token ids are int32 GLOBAL vocabulary ids.
 *   - Shards: with n_shards = R, shard r owns the ids v = r (mod R); its
 *     W_local / E_local hold id v at local row v / R.
 *   - Ties: every ordering is (value desc, id asc).
 *   - Errors: host-checkable problems return EVOSPEC_EINPUT before any launch
 *     (null pointers, sizes out of the context's capacity, k < 1, inv_temp <= 0
 *     or non-finite, d mismatch). CUDA / NCCL failures return EVOSPEC_ECUDA /
 *     EVOSPEC_ENCCL. Device-side conditions (unsorted or out-of-range ids when
 *     debug_checks = 1, a top-k row whose exact order could not be certified,
 *     a selection tie band larger than the workspace) are accumulated in a
 *     device flag word read by evospec_get_flags(). With debug_checks = 1 the
 *     build / LM-head calls synchronize their stream before returning and
 *     return EVOSPEC_EINVARIANT when an invariant flag (EVOSPEC_FLAG_BAD_IDS,
 *     EVOSPEC_FLAG_BUDGET) is set -- the SPEC's invariant exit on the
 *     product path; without debug_checks, evospec_sync_status() gives the same
 *     verdict at a point the caller chooses. Detail for the last error on the
 *     calling thread: evospec_last_error().
 */
#ifndef EVOSPEC_H
#define EVOSPEC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct evospec_ctx evospec_ctx;

typedef int32_t evospec_status;
#define EVOSPEC_OK          0
#define EVOSPEC_EINPUT      2   /* mirrors SPEC's input-error exit code */
#define EVOSPEC_EINVARIANT  3   /* mirrors SPEC's invariant exit code   */
#define EVOSPEC_ECUDA      10
#define EVOSPEC_ENCCL      11
#define EVOSPEC_ENOMEM     12

#define EVOSPEC_BF16 0
#define EVOSPEC_FP32 1

/* Device flag bits (evospec_get_flags). */
#define EVOSPEC_FLAG_BAD_IDS        0x1  /* debug: unsorted / out-of-range ids   */
#define EVOSPEC_FLAG_UNCERTIFIED    0x2  /* a top-k row whose exact order could
                                            not be certified from the kept band  */
#define EVOSPEC_FLAG_SELECT_OVERFLOW 0x4 /* semantic selection overflowed        */
#define EVOSPEC_FLAG_BUDGET         0x8  /* |V_t \ V_static| > N_dyn (never)      */

/* Context configuration, fixed at create time. Sizes are capacities. */
typedef struct {
    int32_t V;            /* global vocabulary size |V|                 */
    int32_t d;            /* hidden size d; multiple of 8                      */
    int32_t w_dtype;      /* EVOSPEC_BF16 / EVOSPEC_FP32: W_local and E_local  */
    int32_t h_dtype;      /* dtype of H and q                                  */
    int32_t n_shards;     /* R >= 1 vocabulary shards                          */
    int32_t shard_rank;   /* r in [0, R)                                       */
    int32_t max_subset;   /* capacity for n_S (global), >= n_static + n_dyn    */
    int32_t max_rows;     /* max n_h per call (draft-tree nodes: 60)    */
    int32_t max_k;        /* max k, 1..64                                      */
    int32_t max_sem;      /* max N_sem (semantic top-N)                        */
    int32_t max_seeds;    /* max n_seed + n_graph_sem_seeds                    */
    int32_t max_ctx;      /* max context tokens for the count source (<= 8192) */
    int32_t debug_checks; /* 1: validate id lists on the device                */
} evospec_config;

/* Builder parameters; paper defaults in brackets (tab:hyperparams P:417-424). */
typedef struct {
    int32_t n_sem;             /* N_sem, semantic top-N            [10]         */
    int32_t n_graph_sem_seeds; /* S_sem prefix that seeds the graph [10]        */
    int32_t per_seed;          /* graph successors per seed         [8]         */
    int32_t ctx_min_count;     /* context-count source; 0 = off     [0]         */
    int32_t n_ctx_max;         /* max tokens from the count source  [0]         */
    int32_t n_dyn;             /* N_dyn dynamic budget              [256]       */
} evospec_build_params;

/* ---- lifecycle ---------------------------------------------------------- */

/* Allocates the context and its device workspace on `device`. */
evospec_status evospec_create(evospec_ctx **out, const evospec_config *cfg, int device);
/* Frees the workspace (and the NCCL communicator, if any). NULL is a no-op. */
evospec_status evospec_destroy(evospec_ctx *ctx);
const char *evospec_status_string(evospec_status st);
/* Thread-local detail of the last non-OK status returned on this thread. */
const char *evospec_last_error(void);
/* Library version string. */
const char *evospec_version(void);

/* Per-weight-tensor preparation (once per W, off the hot path): computes the
 * max row 2-norm of W_local [n_rows, d] into the context; the top-k
 * certification band uses it. Async on stream. */
evospec_status evospec_prepare_weights(evospec_ctx *ctx, const void *W_local_dev,
                                       int64_t n_rows, void *stream);

/* Reads (and with clear=1 resets) the device flag word. Synchronises the
 * stream. flags_out: host int32. */
evospec_status evospec_get_flags(evospec_ctx *ctx, int32_t *flags_out, int clear, void *stream);
/* Synchronizes `stream` and returns EVOSPEC_EINVARIANT if an invariant flag
 * (EVOSPEC_FLAG_BAD_IDS or EVOSPEC_FLAG_BUDGET) is set in the context's flag
 * word (flags are left as they are; evospec_get_flags clears), else EVOSPEC_OK;
 * CUDA errors as EVOSPEC_ECUDA. */
evospec_status evospec_sync_status(evospec_ctx *ctx, void *stream);

/* ---- multi-GPU communicator (vocab sharding) ---------------- */

/* Writes a 128-byte NCCL unique id into uid_out (host). Rank 0 calls it; the
 * caller broadcasts the bytes (e.g. over a torch.distributed group). */
evospec_status evospec_comm_unique_id(void *uid_out);
/* Creates the context's own communicator of n_shards ranks, rank shard_rank.
 * Blocking (collective over all ranks). */
evospec_status evospec_comm_init(evospec_ctx *ctx, const void *uid);

/* ---- a1-a4: subset builder --------------------------------------------- */

/* Builds V_t = sort(V_static u dyn), dyn = the first N_dyn ids, in formation
 * order, of  seeds ++ S_sem ++ S_graph ++ S_ctx  that are not static and not
 * already taken (readings C1-C9 in DESIGN.md):
 *   S_sem  = top-N_sem ids by (q . E_v desc, id asc), exact (fp64) scores;
 *   G      = dedupe(seeds ++ S_sem[:n_graph_sem_seeds]);
 *   S_graph= concat over g in G of the first per_seed entries of CSR row g;
 *   S_ctx  = ids of ctx_ids with count >= ctx_min_count by (count desc, id
 *            asc), the first n_ctx_max (off when ctx_min_count = 0).
 * E_dev: [n_e_rows, d] w_dtype. n_e_rows == V: the full index (every rank
 *   scans all of it). n_e_rows == rows of this shard (R > 1): each rank scans
 *   its interleaved shard and the candidates are exchanged over the context's
 *   communicator (requires evospec_comm_init).
 * q_dev: [d] h_dtype (the target-side hidden state of the verify pass).
 * static_dev: [n_static] sorted ascending unique; seed_dev: [n_seed].
 * csr_row_ptr_dev [V+1] / csr_col_dev [nnz]: rows sorted (p desc, id asc);
 *   both may be NULL (no graph). ctx_dev: [n_ctx] or NULL.
 * Outputs (device, caller-owned): out_ids [n_static + n_dyn] sorted ascending,
 *   out_n [1] = n_S; out_local_ids [capacity n_static + n_dyn] = the ids of
 *   out_ids owned by this shard (v mod R == r), out_local_n [1]; the local
 *   pair may be NULL when R == 1. Nothing is synchronised: n_S stays on the
 *   device and the LM-head call reads it there. */
evospec_status evospec_build_subset(evospec_ctx *ctx,
    const void *E_dev, int64_t n_e_rows, const void *q_dev,
    const int32_t *static_dev, int32_t n_static,
    const int32_t *seed_dev, int32_t n_seed,
    const int32_t *csr_row_ptr_dev, const int32_t *csr_col_dev,
    const int32_t *ctx_dev, int32_t n_ctx,
    const evospec_build_params *params,
    int32_t *out_ids, int32_t *out_n,
    int32_t *out_local_ids, int32_t *out_local_n,
    void *stream);

/* The sharded build in two steps, without a communicator (the
 * NCCL path of evospec_build_subset is step 1, an all-gather, step 2):
 * 1. evospec_build_local_candidates: this shard's exact semantic top-n_sem
 *    (a2, P:95-96 over the shard's rows: E_local [n_e_rows = this shard's row
 *    count, d], global id = local row * R + r) -> out_s [n_sem] fp64 scores,
 *    out_id [n_sem] int32 global ids (device; ordered by (s desc, id asc);
 *    padded with id -1 when the shard has fewer rows).
 * 2. evospec_build_subset_from_candidates: the R shards' candidates stacked in
 *    rank order (cand_s / cand_id [n_cand = R * n_sem], device) -> the global
 *    exact top-n_sem and the formation / union of evospec_build_subset (a2-a4):
 *    every rank gets the same S and its owned slice. The caller moves the
 *    candidates between GPUs (or stacks them on one GPU, as the parity tests do).
 * EVOSPEC_EINPUT on null / out-of-range arguments (n_e_rows not this shard's,
 * n_sem outside [1, max_sem], n_cand outside [1, R * max_sem]). Async. */
evospec_status evospec_build_local_candidates(evospec_ctx *ctx, const void *E_local, int64_t n_e_rows,
    const void *q_dev, int32_t n_sem, double *out_s, int32_t *out_id, void *stream);
evospec_status evospec_build_subset_from_candidates(evospec_ctx *ctx, const double *cand_s, const int32_t *cand_id,
    int32_t n_cand, const int32_t *static_dev, int32_t n_static, const int32_t *seed_dev, int32_t n_seed,
    const int32_t *csr_row_ptr_dev, const int32_t *csr_col_dev, const int32_t *ctx_dev, int32_t n_ctx,
    const evospec_build_params *params, int32_t *out_ids, int32_t *out_n, int32_t *out_local_ids,
    int32_t *out_local_n, void *stream);

/* Batched serving (config Bt, SURVEY §8(a) a4 "a shared static set + 64 ragged
 * dynamic lists"): one query per sequence, the static set shared. For each
 * sequence b < B the builder above runs with q_b = q_dev + b*d, seeds
 * seed_dev[seed_offsets[b] : seed_offsets[b+1]] and context tokens
 * ctx_dev[ctx_offsets[b] : ctx_offsets[b+1]] (ctx_offsets may be NULL), and
 * only the sorted DYNAMIC list dyn_b (static excluded; same formation and cap,
 * P:458) is output -- the direct input of the ragged LM head below.
 * seed_offsets / ctx_offsets: HOST arrays [B+1] (the caller's batch layout).
 * Outputs (device): out_dyn_ids [B * n_dyn] compacted, sequence b at
 *   [out_dyn_offsets[b], out_dyn_offsets[b+1]); out_dyn_offsets [B+1] device,
 *   out_dyn_offsets[0] = 0. Nothing is synchronised.
 * Unsharded contexts and the full index (n_e_rows == V) only; EVOSPEC_EINPUT
 * otherwise. Work: one E scan per sequence (B scans). */
evospec_status evospec_build_subset_batched(evospec_ctx *ctx,
    const void *E_dev, int64_t n_e_rows, const void *q_dev, int32_t B,
    const int32_t *static_dev, int32_t n_static,
    const int32_t *seed_dev, const int32_t *seed_offsets,
    const int32_t *csr_row_ptr_dev, const int32_t *csr_col_dev,
    const int32_t *ctx_dev, const int32_t *ctx_offsets,
    const evospec_build_params *params,
    int32_t *out_dyn_ids, int32_t *out_dyn_offsets,
    void *stream);

/* The last full-index scan's fp64 scores s_v = q . E_v (a2), rows [0, n) (n <= V)
 * into out_dev (device): the scan's own output, for testing its ring (the TMA
 * pipeline's release / refill ordering) against the oracle and itself. */
evospec_status evospec_last_scores(evospec_ctx *ctx, double *out_dev, int64_t n, void *stream);
/* Debug/parity accessor: copies the S_sem SET of the last build on this
 * context (N_sem device ids, in no particular order) into out_dev. Async. */
evospec_status evospec_last_semantic(evospec_ctx *ctx, int32_t *out_dev, int32_t n, void *stream);

/* ---- a5-a7: gathered LM head + fused softmax / top-k --------------------- */

/* For each row r < n_h of H and each position j < n_S (n_S read from
 * n_subset_dev on the device, n_S <= n_subset_max):
 *   z[r][j] = inv_temp * sum_c H[r][c] * W_local[subset[j] / R][c]
 * and returns this shard's triple:
 *   topk_ids  [n_h, k] int32  global ids of the k largest z, (z desc, id asc)
 *   topk_vals [n_h, k] fp32   their z (ordered by the exact fp64 re-score)
 *   row_max   [n_h]    fp32   m = max_j z[r][j]
 *   row_sumexp[n_h]    fp32   s = sum_j exp(z[r][j] - m)
 * Empty subset: m = -inf, s = 0; k > n_S pads id -1 / value -inf.
 * W_local_dev: [n_w_rows, d] w_dtype; H_dev: [n_h, d] h_dtype.
 * subset_dev: sorted ascending unique, every id owned by this shard.
 * logits_out: optional [n_h, n_subset_max] fp32 z (debug / parity only;
 * NULL on the hot path -- the logits are otherwise never written). */
evospec_status evospec_subset_logits_topk(evospec_ctx *ctx,
    const void *W_local_dev, int64_t n_w_rows,
    const void *H_dev, int32_t n_h,
    const int32_t *subset_dev, const int32_t *n_subset_dev, int32_t n_subset_max,
    int32_t k, float inv_temp,
    int32_t *topk_ids, float *topk_vals, float *row_max, float *row_sumexp,
    float *logits_out, void *stream);

/* Single-shard LM head with the merge fused (R = 1): the same projection,
 * softmax and exact top-k as evospec_subset_logits_topk, and the outputs of
 * evospec_merge_shards at R = 1 written by the finalisation kernel itself:
 *   out_ids [n_h, k] int32 global ids, out_vals [n_h, k] fp32 z,
 *   out_lse [n_h] fp32 = m + ln s, out_probs [n_h, k] fp32 (may be NULL),
 *   row_max / row_sumexp [n_h] (may be NULL) the m, s of Eq. 1.
 * EVOSPEC_EINPUT for contexts with n_shards > 1 (use the triple + merge). */
evospec_status evospec_subset_logits_topk_merged(evospec_ctx *ctx,
    const void *W_local_dev, int64_t n_w_rows,
    const void *H_dev, int32_t n_h,
    const int32_t *subset_dev, const int32_t *n_subset_dev, int32_t n_subset_max,
    int32_t k, float inv_temp,
    int32_t *out_ids, float *out_vals, float *out_lse, float *out_probs,
    float *row_max, float *row_sumexp, void *stream);

/* Ragged batched LM head (config Bt): sequence b owns H rows
 * [h_offsets[b], h_offsets[b+1]) and the vocabulary V_b = static u dyn_b,
 * dyn_b = dyn_dev[dyn_offsets[b] : dyn_offsets[b+1]] (sorted ascending,
 * disjoint from static -- what evospec_build_subset_batched outputs). Each row
 * gets the triple of Eq. 1 restricted to its own V_b:
 *   topk over V_b (z desc, id asc), m = max z, s = sum exp(z - m).
 * h_offsets: HOST [B+1], h_offsets[0] = 0, total rows <= max_rows.
 * dyn_offsets: DEVICE [B+1]; max_dyn bounds every dyn_b length (<= max_subset).
 * static_dev may be NULL when n_static = 0. The static block is shared by all
 * rows (its rows are streamed once per group of 128 H rows); the two disjoint
 * parts are merged per row like two vocabulary shards. */
evospec_status evospec_subset_logits_topk_ragged(evospec_ctx *ctx,
    const void *W_local_dev, int64_t n_w_rows, const void *H_dev,
    const int32_t *h_offsets, int32_t B,
    const int32_t *static_dev, int32_t n_static,
    const int32_t *dyn_dev, const int32_t *dyn_offsets, int32_t max_dyn,
    int32_t k, float inv_temp,
    int32_t *topk_ids, float *topk_vals, float *row_max, float *row_sumexp,
    void *stream);

/* ---- a8: vocab-shard merge ------------------------------------------------ */

/* With a communicator (R > 1): all-gathers this rank's triple over NCCL into
 * the workspace, then merges. Without one: the inputs are the R triples
 * already stacked as [R, n_h, k] / [R, n_h] (R = n_shards; R = 1 is the
 * single-GPU finalisation). Over the shards with s_r > 0:
 *   M = max_r m_r, Sigma = sum_r s_r exp(m_r - M), LSE = M + ln Sigma,
 *   out top-k of the R*k candidates by (value desc, id asc),
 *   out_probs = exp(value - LSE).
 * Outputs: out_ids [n_h, k] int32, out_vals [n_h, k] fp32, out_lse [n_h] fp32,
 * out_probs [n_h, k] fp32 (may be NULL). */
evospec_status evospec_merge_shards(evospec_ctx *ctx, int32_t n_h, int32_t k,
    const int32_t *topk_ids, const float *topk_vals,
    const float *row_max, const float *row_sumexp,
    int32_t *out_ids, float *out_vals, float *out_lse, float *out_probs,
    void *stream);

/* ---- N2: lossless verification of a draft chain ----------- */

/* Verifies g draft proposals against the target, the rejection criterion
 * alpha of P:42 (Leviathan et al.) in the chain form of SPEC S:380-385 (verify
 * phase of alg. P:366-367; greedy T = 0 is the paper's setting).
 * Position j (0 <= j <= g): p_j(v) = exp(z_j[v] inv_temp - m_j) / s_j over the
 * FULL vocabulary [0, V), fp64; q_j = draft_probs[j][i] at subset_ids[i] and
 * exactly 0 outside the subset.
 *   greedy != 0: accept x_j while x_j == argmax p_j (ties: lower id); on a
 *     mismatch emit argmax p_j and stop; all accepted: the bonus argmax p_g.
 *     subset_ids, draft_probs, u, w may be NULL.
 *   greedy == 0: accept x_j iff u[j] < min(1, p_j(x_j) / q_j(x_j)); on the
 *     first rejection emit the draw from normalize(max(0, p_j - q_j)) with w[j]
 *     and stop; all accepted: the bonus drawn from p_g with w[g]. A draw with
 *     w in [0, 1) is the smallest v (id order) whose running sum of the
 *     weights exceeds w * (their total); if the residual mass is 0 (rounding
 *     only) the draw is from p_j.
 * Arguments (device memory, caller-owned): target_logits [g+1, V] fp32 row-
 * major; proposals [g] int32 (each must have q_j > 0: otherwise the position
 * is rejected with token -1 and EVOSPEC_FLAG_BAD_IDS is raised); subset_ids
 * [n_subset] sorted ascending unique; draft_probs [g, n_subset] fp32; u [g]
 * and w [g+1] fp64 uniforms in [0, 1) drawn by the caller (g = 0: only w).
 * Outputs: tokens [g+1] int32 = the accepted proposals, then the corrected or
 * bonus token, then -1 pads; n_accepted [1] int32 (the round emits
 * n_accepted + 1 tokens). 0 <= g <= 63. Async on `stream`; two
 * kernel launches. EVOSPEC_EINPUT on null / out-of-range host arguments. */
evospec_status evospec_verify_chain(evospec_ctx *ctx, const float *target_logits, int32_t V, int32_t g,
    const int32_t *proposals, const int32_t *subset_ids, int32_t n_subset, const float *draft_probs,
    float inv_temp, int32_t greedy, const double *u, const double *w,
    int32_t *tokens, int32_t *n_accepted, void *stream);

/* ---- N4: coverage of the active vocabulary ---------------- */

/* For each target row r < n_rows: p_r(v) = exp(z_r[v] inv_temp - m_r) / s_r
 * over [0, V) (fp64) and
 *   covered_mass[r]   = sum_{v in V_t} p_r(v)     (Eq. 2's constraint P:58-62,
 *                                                  App. E)
 *   recall[r][t]      = |V_t n top-ks[t](p_r)| / ks[t], the target top-k
 *                       ordered (p desc, id asc)
 * target_logits [n_rows, V] fp32; subset_ids [n_subset] sorted ascending
 * unique (V_t); ks [n_ks] int32 in [1, min(V, 1024)] (device; an entry outside
 * yields NaN for that k and raises EVOSPEC_FLAG_BAD_IDS), n_ks <= 64; outputs covered_mass
 * [n_rows] and recall [n_rows, n_ks] fp64 (device). Async, one launch.
 * EVOSPEC_EINPUT on null / out-of-range host arguments. */
evospec_status evospec_coverage(evospec_ctx *ctx, const float *target_logits, int32_t n_rows, int32_t V,
    const int32_t *subset_ids, int32_t n_subset, float inv_temp, const int32_t *ks, int32_t n_ks,
    double *covered_mass, double *recall, void *stream);

/* ---- N3: curriculum-weighted distillation objective -------- */

/* Forward and gradient (w.r.t. the draft logits) of Eq. lora_objective
 * with the horizon weights of Eq. curriculum_weight,
 * per trajectory b < B and step j < g on the retained support of K target
 * logits (the LoRA update itself is out of scope):
 *   p_hat = softmax(target / T_kd), p_til = softmax(draft / T_kd),
 *   L_base[b] = logsumexp(draft[b][0]) - draft[b][0][verified[b]]  (the
 *     first-step cross entropy against the verified token, temperature 1),
 *   weights[b][j] = exp(-beta L_base[b] j),
 *   loss[b] = sum_j weights[b][j] T_kd^2 KL(p_hat || p_til),
 *   grad[b][j][i] = weights[b][j] T_kd (p_til[i] - p_hat[i])  (weights held
 *     fixed: a confidence proxy).
 * target_logits / draft_logits [B, g, K] fp32, verified [B] int32 (support
 * index in [0, K); outside: that trajectory's loss / grad / weights are NaN and
 * EVOSPEC_FLAG_BAD_IDS is raised); outputs loss [B], grad [B, g, K] (may be
 * NULL), weights [B, g] (may be NULL), fp32, device. g <= 32, K <= 1024 (the
 * paper: gamma = 6, T_kd = 1, beta = 0.3). fp32 arithmetic.
 * Terms with p_hat = 0 (a -inf target logit) contribute 0 to the KL. Async.
 * Reading K1: L_base is taken on the retained first-step support
 * (the verified token is the target's top-1, so it is on it); SPEC's program
 * takes the draft's restricted distribution over the V_t snapshot instead --
 * callers holding that value can pass those logits as draft_logits[b][0]. */
evospec_status evospec_kd_loss(evospec_ctx *ctx, int32_t B, int32_t g, int32_t K, const float *target_logits,
    const float *draft_logits, const int32_t *verified, float T_kd, float beta,
    float *loss, float *grad, float *weights, void *stream);

/* ---- N1: ARC dynamic buffer + incremental subset update ---- */

/* The dynamic buffer's Adaptive Replacement Cache (App. A.3;
 * SPEC S:288-348): resident lists T1 / T2 (|T1| + |T2| <= capacity = N_dyn),
 * ghost lists B1 / B2, adaptive target p. Host-side, single writer;
 * no GPU needed. Paper defaults: capacity 256, p0 128, ghost caps
 * 256 / 256, min residency 8 decoding steps, warm-up 50 events.
 *   touch:  a T1 / T2 member moves to the MRU end of T2; returns 1 on a hit.
 *   admit:  one OOV event (the warm-up counts events): each token (a
 *           deduplicated list) is touched if resident; a B1 ghost raises p by
 *           max(1, |B2| / |B1|), a B2 ghost lowers it by max(1, |B1| / |B2|)
 *           (after warm-up; integer division) and lands in T2; otherwise it
 *           lands in T1. An insertion into a full cache first evicts one
 *           member: from T1 if |T1| > p (or T2 empty), else T2; the LRU-most
 *           member resident >= min_residency steps since its admission, else
 *           the other list's, else plain LRU of the chosen list. Evicted ids
 *           (in order) go to evicted[] (capacity n) and to B1 / B2.
 *   state:  [|T1|, |T2|, |B1|, |B2|, p, T1..., T2..., B1..., B2...], each list
 *           LRU -> MRU (trace-equivalence testing).
 * EVOSPEC_EINPUT on null / out-of-range arguments. */
typedef struct evospec_arc evospec_arc;
evospec_status evospec_arc_create(evospec_arc **out, int32_t capacity, int32_t p0, int32_t b1_cap, int32_t b2_cap,
    int32_t min_residency, int32_t warmup_events);
evospec_status evospec_arc_destroy(evospec_arc *arc);
int32_t        evospec_arc_touch(evospec_arc *arc, int32_t token, int64_t step);
evospec_status evospec_arc_admit(evospec_arc *arc, const int32_t *tokens, int32_t n, int64_t step,
    int32_t *evicted, int32_t *n_evicted);
evospec_status evospec_arc_state(const evospec_arc *arc, int32_t *out, int32_t cap, int32_t *n_out);
/* evospec_arc_admit as a membership delta: admits tokens[n] (one OOV event) and
 * returns the NET change of the member set T1 u T2 -- added[] (members now, not
 * before) and removed[] (members before, not now), each ascending, capacity n
 * each -- exactly the removed / added arguments evospec_subset_update expects (a
 * token admitted and evicted within the event appears in neither). */
evospec_status evospec_arc_admit_delta(evospec_arc *arc, const int32_t *tokens, int32_t n, int64_t step,
    int32_t *added, int32_t *n_added, int32_t *removed, int32_t *n_removed);

/* Incremental update of the sorted active vocabulary on the device (no full
 * rebuild): out = sort((subset \ removed) u added). subset [n] sorted unique;
 * removed [n_removed] sorted, a subset of `subset`; added [n_added] sorted,
 * disjoint from subset \ removed; out [n - n_removed + n_added] and n_out [1]
 * device. One kernel (per-element binary searches). Async on `stream`.
 * flags (device int32 [1] or NULL): OR-ed with EVOSPEC_FLAG_BAD_IDS when the
 * contract is violated (a removed id not in subset, an added id already kept);
 * writes stay inside out[] whatever the input, but the content is then not the
 * requested set. (evospec_oov_event computes a conforming delta from ARC.) */
evospec_status evospec_subset_update(const int32_t *subset, int32_t n, const int32_t *removed, int32_t n_removed,
    const int32_t *added, int32_t n_added, int32_t *out, int32_t *n_out, int32_t *flags, void *stream);

/* N1 OOV event, in two phases so that it overlaps the draft steps (Path A runs
 * asynchronously; App. B): when the verified token falls
 * outside V_t, _begin enqueues the event's candidate formation on
 * the context's side stream -- the exact semantic top-n_sem of the target-side
 * hidden state q (the HNSW top-10 of P:458, C2), the graph top-per_seed of
 * seeds u S_sem[:n_graph_sem_seeds] (target top-10 u semantic top-10,
 * 8 successors each), the first n_dyn (max insertions per event, 32 at P:462)
 * new non-static ids -- after the work already on `stream` (q, seeds), and
 * returns at once; the caller keeps running LM-head calls on the current
 * subset (any stream; no build / draft_step on this context meanwhile).
 * _end waits for the candidates, admits them into the ARC in ascending id order
 * (reading A3) as one event at `step` (evospec_arc_admit_delta), and enqueues the
 * incremental update out = sort((subset \ removed) u added) on `stream`; the
 * net delta is also returned to the host (added_host / removed_host [n_dyn] or
 * NULL). subset [n]: the current V_t = static u ARC members (sorted); out
 * [n + n_dyn] and n_out [1] device. Unsharded contexts; one event in flight.
 * EVOSPEC_EINPUT on null / out-of-range arguments or a second _begin / an _end
 * without one. */
evospec_status evospec_oov_event_begin(evospec_ctx *ctx, const void *E_dev, int64_t n_e_rows, const void *q_dev,
    const int32_t *static_dev, int32_t n_static, const int32_t *seed_dev, int32_t n_seed,
    const int32_t *csr_row_ptr_dev, const int32_t *csr_col_dev, const evospec_build_params *params, void *stream);
evospec_status evospec_oov_event_end(evospec_ctx *ctx, evospec_arc *arc, int64_t step, const int32_t *subset_dev,
    int32_t n, int32_t *out_dev, int32_t *n_out_dev, int32_t *added_host, int32_t *n_added, int32_t *removed_host,
    int32_t *n_removed, void *stream);

/* ---- one draft step through the whole path -------------------------------- */

/* Per-step I/O for evospec_draft_step. `host_io` = 1: q, H, seeds, ctx and
 * the four outputs are HOST buffers (pinned for async copies) and the call
 * stages them through the context's device buffers (H2D before, D2H after,
 * on the same stream); 0: they are device buffers. Model-resident tensors
 * (E, W_local, static set, CSR) are always device pointers. */
typedef struct {
    const void *E;        int64_t n_e_rows;
    const void *W_local;  int64_t n_w_rows;
    const int32_t *static_ids; int32_t n_static;
    const int32_t *csr_row_ptr; const int32_t *csr_col;
    evospec_build_params build;
    int32_t n_h; int32_t k; float inv_temp;
    const void *q;                 /* [d]        */
    const void *H;                 /* [n_h, d]   */
    const int32_t *seeds; int32_t n_seed;
    const int32_t *ctx_ids; int32_t n_ctx;
    int32_t *out_ids;              /* [n_h, k]   */
    float *out_vals;               /* [n_h, k]   */
    float *out_lse;                /* [n_h]      */
    float *out_probs;              /* [n_h, k]   */
    int32_t host_io;
} evospec_step_io;

/* build_subset -> subset_logits_topk -> merge_shards on one stream. With
 * host_io = 1 the call returns after the D2H copies are enqueued; the caller
 * synchronises the stream before reading the outputs. */
evospec_status evospec_draft_step(evospec_ctx *ctx, const evospec_step_io *io, void *stream);

/* ---- measurement hooks (bench / profiling; off by default) ---------------- */

#define EVOSPEC_STAGE_SCAN      0  /* a2 semantic scan q . E^T                 */
#define EVOSPEC_STAGE_SELECT    1  /* a2 top-N select + exact order (+ NCCL)   */
#define EVOSPEC_STAGE_UNION     2  /* a3/a4 context counts, formation, union   */
#define EVOSPEC_STAGE_LMH       3  /* a5-a7 gathered LM head main kernel(s)    */
#define EVOSPEC_STAGE_FINALIZE  4  /* a6/a7 per-shard finalisation + re-score  */
#define EVOSPEC_STAGE_MERGE     5  /* a8 all-gather + merge                    */
#define EVOSPEC_STAGE_COPY      6  /* draft_step host<->device staging         */
#define EVOSPEC_NUM_STAGES      7

typedef struct {
    int64_t launches;                    /* kernels this library launched     */
    int32_t calls[EVOSPEC_NUM_STAGES];   /* timed calls per stage             */
    float stage_ms[EVOSPEC_NUM_STAGES];  /* summed device time per stage (ms) */
} evospec_stats;

/* enable = 1: reset the counters and record CUDA events around every stage
 * on the caller's stream (up to 4096 calls per stage); enable = 0: stop. */
evospec_status evospec_set_timing(evospec_ctx *ctx, int enable);
/* Synchronises the recorded events and returns the sums since the last
 * evospec_set_timing(ctx, 1). The launch counter runs always. */
evospec_status evospec_read_stats(evospec_ctx *ctx, evospec_stats *out);
/* Profiling: with EVOSPEC_TRACE set in the environment, the tcgen05 LM-head
 * kernel stamps %globaltimer (ns) per CTA into 8 slots [start, producers
 * done, MMA done, tile-0 accumulator ready, tile-0 folded, tile-1 ready,
 * tile-1 folded, end] (slots [0, 148*8)), the finalize kernel per H row
 * (slots [148*8, 2*148*8)) and the union kernel 7 phase stamps (slots
 * [2*148*8, +7)); this copies the first n int64 (synchronous). */
evospec_status evospec_read_trace(evospec_ctx *ctx, int64_t *host_out, int32_t n);

#ifdef __cplusplus
}
#endif
#endif /* EVOSPEC_H */
