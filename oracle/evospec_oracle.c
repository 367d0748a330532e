/*
 * evospec_oracle.c -- plain, slow, obviously-correct CPU oracle for the
 * EvoSpec dynamic-vocabulary draft LM-head path.
 *
 * TEST INFRASTRUCTURE ONLY. Nothing in the product path links, loads or
 * calls this file: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it. It shares no code, header,
 * table or constant with paper_2605_27390_b200/ (the CUDA path).
 *
 * All arithmetic is IEEE double, sequential in the hidden index c, on bf16 /
 * fp32 inputs decoded exactly (bf16 bits << 16 is an fp32 with the same
 * value; fp32 -> double is exact). No -ffast-math. Single-threaded.
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n,
 * "§8(c) step i" = SURVEY.md §8(c) oracle step i (the reading of the paper
 * adopted in DESIGN.md "Readings").
 *
 * Return codes: 0 ok, 2 input error (mirrors SPEC exit code 2).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EO_OK 0
#define EO_EINPUT 2

enum { EO_BF16 = 0, EO_FP32 = 1 };

/* §8(c) step 1: exact decode of one element. */
static double eo_decode(const void *base, int dtype, int64_t idx) {
    if (dtype == EO_BF16) {
        uint32_t bits = ((uint32_t)((const uint16_t *)base)[idx]) << 16;
        float f;
        memcpy(&f, &bits, sizeof f);
        return (double)f;
    }
    return (double)((const float *)base)[idx];
}

/* Ordering key "(-value, id)": larger value first, lower id on ties
 * ("ties broken by smallest token id"). */
typedef struct {
    double v;
    int32_t id;
} eo_key;

static int eo_cmp_desc(const void *a, const void *b) {
    const eo_key *x = (const eo_key *)a, *y = (const eo_key *)b;
    if (x->v > y->v) return -1;
    if (x->v < y->v) return 1;
    return (x->id < y->id) ? -1 : (x->id > y->id);
}

static int eo_cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* ------------------------------------------------------------------ */
/* a2: semantic scores, MIPS over the index rows.     */
/* s_v = sum_{c=0}^{d-1} q[c] * E[v][c]        (§8(c) step 2)           */
/* ------------------------------------------------------------------ */
int eo_sem_scores(const void *E, int e_dtype, int64_t n_rows, int d,
                  const void *q, int q_dtype, double *out) {
    if (!E || !q || !out || n_rows < 0 || d < 1) return EO_EINPUT;
    for (int64_t v = 0; v < n_rows; ++v) {
        double acc = 0.0;
        for (int c = 0; c < d; ++c)
            acc += eo_decode(q, q_dtype, c) * eo_decode(E, e_dtype, v * (int64_t)d + c);
        out[v] = acc;
    }
    return EO_OK;
}

/* §8(c) step 3: the first N of [0,n) ordered by (-s_v, v). */
int eo_topn(const double *s, int64_t n, int N, int32_t *out_ids) {
    if (!s || !out_ids || N < 0 || N > n) return EO_EINPUT;
    eo_key *keys = (eo_key *)malloc(sizeof(eo_key) * (size_t)(n > 0 ? n : 1));
    if (!keys) return EO_EINPUT;
    for (int64_t v = 0; v < n; ++v) { keys[v].v = s[v]; keys[v].id = (int32_t)v; }
    qsort(keys, (size_t)n, sizeof(eo_key), eo_cmp_desc);
    for (int i = 0; i < N; ++i) out_ids[i] = keys[i].id;
    free(keys);
    return EO_OK;
}

/* ------------------------------------------------------------------ */
/* a3: statistical expansion over the co-occurrence CSR (P:98,  */
/* P:458; per_seed = 8 "top-8 outgoing neighbors").             */
/* S_graph = concat_{g in G} col[row_ptr[g] : row_ptr[g]+min(per_seed, */
/* deg g)]  (§8(c) step 5; rows are pre-sorted by (p desc, id asc)).   */
/* ------------------------------------------------------------------ */
int eo_graph_expand(const int32_t *G, int nG, const int32_t *row_ptr,
                    const int32_t *col, int per_seed, int32_t *out, int *out_n) {
    if ((nG > 0 && !G) || !out_n || per_seed < 0) return EO_EINPUT;
    int n = 0;
    for (int i = 0; i < nG; ++i) {
        int32_t g = G[i];
        if (!row_ptr) continue;              /* no graph: contributes nothing */
        int32_t deg = row_ptr[g + 1] - row_ptr[g];
        int32_t take = deg < per_seed ? deg : per_seed;
        for (int32_t j = 0; j < take; ++j) out[n++] = col[row_ptr[g] + j];
    }
    *out_n = n;
    return EO_OK;
}

/* §8(c) step 6 (reading C5): tokens of ctx with count >= min_count,
 * ordered by (-count, id), the first n_max. Off when min_count == 0. */
int eo_ctx_tokens(const int32_t *ctx, int n_ctx, int V, int min_count, int n_max,
                  int32_t *out, int *out_n) {
    if (!out_n || (n_ctx > 0 && !ctx)) return EO_EINPUT;
    *out_n = 0;
    if (min_count <= 0 || n_max <= 0 || n_ctx <= 0) return EO_OK;
    int32_t *count = (int32_t *)calloc((size_t)V, sizeof(int32_t));
    if (!count) return EO_EINPUT;
    for (int i = 0; i < n_ctx; ++i) {
        if (ctx[i] < 0 || ctx[i] >= V) { free(count); return EO_EINPUT; }
        count[ctx[i]]++;
    }
    eo_key *keys = (eo_key *)malloc(sizeof(eo_key) * (size_t)V);
    int nk = 0;
    for (int v = 0; v < V; ++v)
        if (count[v] >= min_count) { keys[nk].v = (double)count[v]; keys[nk].id = v; nk++; }
    qsort(keys, (size_t)nk, sizeof(eo_key), eo_cmp_desc);
    int take = nk < n_max ? nk : n_max;
    for (int i = 0; i < take; ++i) out[i] = keys[i].id;
    *out_n = take;
    free(keys);
    free(count);
    return EO_OK;
}

/* ------------------------------------------------------------------ */
/* a1-a4: V_t = V_static u S_sem(h) u S_graph(.) (Eq. vocab_union,     */
/* P:88-93), runtime formation, budget |V_t \ V_static| <=     */
/* N_dyn (Eq. optimization), cap order.           */
/* ------------------------------------------------------------------ */
int eo_build_subset(const void *E, int e_dtype, int V, int d,
                    const void *q, int q_dtype,
                    const int32_t *static_ids, int n_static,
                    const int32_t *seed_ids, int n_seed,
                    const int32_t *row_ptr, const int32_t *col,
                    const int32_t *ctx_ids, int n_ctx,
                    int n_sem, int n_graph_sem_seeds, int per_seed,
                    int ctx_min_count, int n_ctx_max, int n_dyn,
                    int32_t *out_S, int32_t *out_nS,
                    int32_t *out_sem, int32_t *out_dyn, int32_t *out_ndyn) {
    if (!E || !q || !out_S || !out_nS || V < 1 || d < 1 || n_sem < 0 || n_sem > V ||
        n_dyn < 0 || n_static < 0 || n_static > V || n_seed < 0 ||
        n_graph_sem_seeds < 0 || per_seed < 0)
        return EO_EINPUT;
    /* inputs: static sorted strictly ascending, all ids in range */
    for (int i = 0; i < n_static; ++i) {
        if (static_ids[i] < 0 || static_ids[i] >= V) return EO_EINPUT;
        if (i > 0 && static_ids[i] <= static_ids[i - 1]) return EO_EINPUT;
    }
    for (int i = 0; i < n_seed; ++i)
        if (seed_ids[i] < 0 || seed_ids[i] >= V) return EO_EINPUT;

    int rc = EO_OK;
    double *s = (double *)malloc(sizeof(double) * (size_t)V);
    int32_t *sem = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_sem > 0 ? n_sem : 1));
    int nG_max = n_seed + n_graph_sem_seeds;
    int32_t *G = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nG_max > 0 ? nG_max : 1));
    int32_t *graph = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nG_max * per_seed + 1));
    int32_t *ctxs = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_ctx_max > 0 ? n_ctx_max : 1));
    uint8_t *in_static = (uint8_t *)calloc((size_t)V, 1);
    uint8_t *in_dyn = (uint8_t *)calloc((size_t)V, 1);
    uint8_t *in_G = (uint8_t *)calloc((size_t)V, 1);
    int32_t *dyn = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_dyn > 0 ? n_dyn : 1));
    if (!s || !sem || !G || !graph || !ctxs || !in_static || !in_dyn || !in_G || !dyn) {
        rc = EO_EINPUT;
        goto done;
    }

    /* step 2-3: S_sem */
    eo_sem_scores(E, e_dtype, V, d, q, q_dtype, s);
    eo_topn(s, V, n_sem, sem);

    /* step 4: G = dedupe_first(seed_ids ++ S_sem[0:n_graph_sem_seeds]) (C4) */
    int nG = 0;
    for (int i = 0; i < n_seed; ++i)
        if (!in_G[seed_ids[i]]) { in_G[seed_ids[i]] = 1; G[nG++] = seed_ids[i]; }
    for (int i = 0; i < n_graph_sem_seeds && i < n_sem; ++i)
        if (!in_G[sem[i]]) { in_G[sem[i]] = 1; G[nG++] = sem[i]; }

    /* step 5: S_graph */
    int n_graph = 0;
    eo_graph_expand(G, nG, row_ptr, col, per_seed, graph, &n_graph);
    for (int i = 0; i < n_graph; ++i)
        if (graph[i] < 0 || graph[i] >= V) { rc = EO_EINPUT; goto done; }

    /* step 6: S_ctx */
    int n_ctxs = 0;
    rc = eo_ctx_tokens(ctx_ids, n_ctx, V, ctx_min_count, n_ctx_max, ctxs, &n_ctxs);
    if (rc) goto done;

    /* step 7: C = seeds ++ S_sem ++ S_graph ++ S_ctx; first-occurrence,
     * skip static members, stop at N_dyn (C6, C7). */
    for (int i = 0; i < n_static; ++i) in_static[static_ids[i]] = 1;
    int nd = 0;
    const int32_t *parts[4] = {seed_ids, sem, graph, ctxs};
    int lens[4] = {n_seed, n_sem, n_graph, n_ctxs};
    for (int p = 0; p < 4 && nd < n_dyn; ++p)
        for (int i = 0; i < lens[p] && nd < n_dyn; ++i) {
            int32_t c = parts[p][i];
            if (in_static[c] || in_dyn[c]) continue;
            in_dyn[c] = 1;
            dyn[nd++] = c;
        }

    /* step 8: S = sort_ascending(static u dyn) */
    int nS = 0;
    for (int i = 0; i < n_static; ++i) out_S[nS++] = static_ids[i];
    for (int i = 0; i < nd; ++i) out_S[nS++] = dyn[i];
    qsort(out_S, (size_t)nS, sizeof(int32_t), eo_cmp_i32);
    *out_nS = nS;
    if (out_sem) memcpy(out_sem, sem, sizeof(int32_t) * (size_t)n_sem);
    if (out_dyn) memcpy(out_dyn, dyn, sizeof(int32_t) * (size_t)nd);
    if (out_ndyn) *out_ndyn = nd;

done:
    free(s); free(sem); free(G); free(graph); free(ctxs);
    free(in_static); free(in_dyn); free(in_G); free(dyn);
    return rc;
}

/* ------------------------------------------------------------------ */
/* a5: gathered LM-head contraction, Eq. projection over     */
/* V_t (alg:evospec P:364): l[r][j] = sum_c H[r][c] * W[S_j][c];       */
/* z = l * inv_temp (reading C11).  A shard r of R owns the ids        */
/* v = r (mod R) and stores id v at local row v / R (§8(e)).            */
/* ------------------------------------------------------------------ */
int eo_subset_logits(const void *W, int w_dtype, int64_t n_rows_local, int d,
                     const void *H, int h_dtype, int n_h,
                     const int32_t *S, int n_S, int R, double inv_temp,
                     double *out_z) {
    if (!W || !H || (n_S > 0 && (!S || !out_z)) || d < 1 || n_h < 0 || R < 1 ||
        !(inv_temp > 0.0) || !isfinite(inv_temp))
        return EO_EINPUT;
    for (int j = 0; j < n_S; ++j) {
        int64_t row = S[j] / R;
        if (S[j] < 0 || row >= n_rows_local) return EO_EINPUT;
    }
    for (int r = 0; r < n_h; ++r)
        for (int j = 0; j < n_S; ++j) {
            int64_t row = S[j] / R;
            double acc = 0.0;
            for (int c = 0; c < d; ++c)
                acc += eo_decode(H, h_dtype, (int64_t)r * d + c) *
                       eo_decode(W, w_dtype, row * (int64_t)d + c);
            out_z[(int64_t)r * n_S + j] = acc * inv_temp;
        }
    return EO_OK;
}

/* ------------------------------------------------------------------ */
/* a6-a7: softmax restricted to S (Eq. 1; zero mass off S)  */
/* m = max z, s = sum e^{z-m}, LSE = m + ln s, p = e^{z-LSE};           */
/* top-k = first k under (-z, S_j).                           */
/* Empty support: m = -inf, s = 0 (reading C16); k > n_S pads id -1,   */
/* value -inf, prob 0.                                                 */
/* ------------------------------------------------------------------ */
int eo_softmax_topk(const double *z, int n_h, int n_S, const int32_t *S, int k,
                    int32_t *ids, double *vals, double *m, double *s,
                    double *lse, double *probs) {
    if (k < 1 || n_h < 0 || n_S < 0 || !ids || !vals || !m || !s) return EO_EINPUT;
    eo_key *keys = (eo_key *)malloc(sizeof(eo_key) * (size_t)(n_S > 0 ? n_S : 1));
    if (!keys) return EO_EINPUT;
    for (int r = 0; r < n_h; ++r) {
        const double *zr = z + (int64_t)r * n_S;
        double mr = -INFINITY, sr = 0.0;
        for (int j = 0; j < n_S; ++j) if (zr[j] > mr) mr = zr[j];
        for (int j = 0; j < n_S; ++j) sr += exp(zr[j] - mr);
        double lr = n_S > 0 ? mr + log(sr) : -INFINITY;
        m[r] = mr;
        s[r] = sr;
        if (lse) lse[r] = lr;
        for (int j = 0; j < n_S; ++j) { keys[j].v = zr[j]; keys[j].id = S[j]; }
        qsort(keys, (size_t)n_S, sizeof(eo_key), eo_cmp_desc);
        for (int i = 0; i < k; ++i) {
            int64_t o = (int64_t)r * k + i;
            if (i < n_S) {
                ids[o] = keys[i].id;
                vals[o] = keys[i].v;
                if (probs) probs[o] = exp(keys[i].v - lr);
            } else {
                ids[o] = -1;
                vals[o] = -INFINITY;
                if (probs) probs[o] = 0.0;
            }
        }
    }
    free(keys);
    return EO_OK;
}

/* ------------------------------------------------------------------ */
/* a8: vocab-shard merge (north star; §8(c) step 12).                   */
/* M = max_r m_r, Sigma = sum_r s_r e^{m_r - M}, LSE = M + ln Sigma,    */
/* over shards with s_r > 0; top-k of concat(topk_r) by (-val, id);     */
/* p = e^{val - LSE}.  Inputs are stacked [R][n_h][k] and [R][n_h].     */
/* ------------------------------------------------------------------ */
int eo_merge(int R, int n_h, int k, const int32_t *ids, const double *vals,
             const double *m, const double *s, int32_t *out_ids, double *out_vals,
             double *out_lse, double *out_probs) {
    if (R < 1 || n_h < 0 || k < 1 || !ids || !vals || !m || !s || !out_ids || !out_vals)
        return EO_EINPUT;
    eo_key *keys = (eo_key *)malloc(sizeof(eo_key) * (size_t)R * (size_t)k);
    if (!keys) return EO_EINPUT;
    for (int r = 0; r < n_h; ++r) {
        double M = -INFINITY;
        for (int t = 0; t < R; ++t) {
            int64_t o = (int64_t)t * n_h + r;
            if (s[o] > 0.0 && m[o] > M) M = m[o];
        }
        double sig = 0.0;
        for (int t = 0; t < R; ++t) {
            int64_t o = (int64_t)t * n_h + r;
            if (s[o] > 0.0) sig += s[o] * exp(m[o] - M);
        }
        double L = sig > 0.0 ? M + log(sig) : -INFINITY;
        if (out_lse) out_lse[r] = L;
        int nk = 0;
        for (int t = 0; t < R; ++t)
            for (int i = 0; i < k; ++i) {
                int64_t o = ((int64_t)t * n_h + r) * k + i;
                if (ids[o] < 0) continue;     /* padding */
                keys[nk].v = vals[o];
                keys[nk].id = ids[o];
                nk++;
            }
        qsort(keys, (size_t)nk, sizeof(eo_key), eo_cmp_desc);
        for (int i = 0; i < k; ++i) {
            int64_t o = (int64_t)r * k + i;
            if (i < nk) {
                out_ids[o] = keys[i].id;
                out_vals[o] = keys[i].v;
                if (out_probs) out_probs[o] = exp(keys[i].v - L);
            } else {
                out_ids[o] = -1;
                out_vals[o] = -INFINITY;
                if (out_probs) out_probs[o] = 0.0;
            }
        }
    }
    free(keys);
    return EO_OK;
}

/* ------------------------------------------------------------------ */
/* N2: lossless verification of a draft chain against  */
/* the target, the rejection criterion alpha of P:42 (Leviathan et    */
/* al.), verify phase of alg. P:366-367, chain form and rule of SPEC  */
/* S:380-385; greedy decoding (T = 0) is the paper's setting.   */
/*                                                                    */
/* Position j (0 <= j <= g): p_j(v) = exp(z_j[v] it - m_j) / s_j over  */
/* the FULL vocabulary [0, V) (it = inv_temp, m_j = max, s_j = sum),   */
/* fp64. The draft's restricted distribution q_j is qS[j][i] at S[i]   */
/* (S sorted, unique) and exactly 0 outside S.                 */
/* Greedy: accept x_j while x_j == argmax p_j (ties: lower id); on a   */
/*   mismatch emit argmax p_j and stop; all g accepted: emit argmax   */
/*   p_g (the bonus token).                                            */
/* Sampling: accept x_j iff u_j < min(1, p_j(x_j) / q_j(x_j)); on the  */
/*   first rejection emit the token drawn from normalize(max(0, p_j -  */
/*   q_j)) with w_j, stop; all accepted: the bonus drawn from p_g with */
/*   w_g. Draw from weights r with w in [0, 1): the smallest v (id     */
/*   order) whose running sum r(0) + ... + r(v) exceeds w * sum_v r(v). */
/*   (Reading V1: if the residual mass is 0 -- possible only through   */
/*   rounding, since p_j(x) < q_j(x) forces mass elsewhere -- the draw */
/*   is from p_j instead.)                                             */
/* The uniforms u, w are inputs (drawn by the caller).                 */
/* Out: tokens[0 .. n_acc] = the accepted proposals then the emitted   */
/* token; *n_acc_out = n_acc. Returns 3 if a proposal has q = 0        */
/* (proposals must come from q's support), 2 on bad input.      */
/* ------------------------------------------------------------------ */
static int eo_find_sorted(const int32_t *S, int n, int32_t v) {
    int lo = 0, hi = n - 1;
    while (lo <= hi) {
        int mid = lo + (hi - lo) / 2;
        if (S[mid] == v) return mid;
        if (S[mid] < v) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* the target distribution of row zj: m, s in fp64 (sequential over v) */
static void eo_target_stats(const float *zj, int V, double it, double *m, double *s, int32_t *amax) {
    double M = -INFINITY;
    int32_t a = -1;
    for (int v = 0; v < V; ++v) {
        double x = (double)zj[v] * it;
        if (x > M) { M = x; a = v; }          /* strict: ties keep the lower id */
    }
    double sum = 0.0;
    for (int v = 0; v < V; ++v) sum += exp((double)zj[v] * it - M);
    *m = M; *s = sum; *amax = a;
}

/* draw from r(v) = max(0, p(v) - q(v)) (q from qj on S, 0 elsewhere; qj == NULL: q = 0) */
static int32_t eo_draw(const float *zj, int V, double it, double m, double s, const int32_t *S, int n_S,
                       const float *qj, double w) {
    double tot = 0.0;
    int i = 0;
    for (int v = 0; v < V; ++v) {
        double q = 0.0;
        while (qj && i < n_S && S[i] < v) ++i;
        if (qj && i < n_S && S[i] == v) q = (double)qj[i];
        double r = exp((double)zj[v] * it - m) / s - q;
        if (r > 0.0) tot += r;
    }
    if (!(tot > 0.0)) return eo_draw(zj, V, it, m, s, S, n_S, NULL, w);   /* reading V1 */
    double target = w * tot, run = 0.0;
    int32_t last = -1;
    i = 0;
    for (int v = 0; v < V; ++v) {
        double q = 0.0;
        while (qj && i < n_S && S[i] < v) ++i;
        if (qj && i < n_S && S[i] == v) q = (double)qj[i];
        double r = exp((double)zj[v] * it - m) / s - q;
        if (r > 0.0) {
            run += r;
            last = v;
            if (run > target) return v;
        }
    }
    return last;   /* w * tot at the very top of the rounding band */
}

int eo_verify_chain(const float *z, int V, int g, const int32_t *x, const int32_t *S, int n_S,
                    const float *qS, double inv_temp, int greedy, const double *u, const double *w,
                    int32_t *tokens, int32_t *n_acc_out) {
    if (!z || V < 1 || g < 0 || (g > 0 && !x) || !tokens || !n_acc_out || !(inv_temp > 0.0)) return EO_EINPUT;
    if (!greedy && (!u || !w || (g > 0 && (!S || !qS || n_S < 1)))) return EO_EINPUT;
    int n_acc = 0;
    for (int j = 0; j <= g; ++j) {
        const float *zj = z + (int64_t)j * V;
        double m, s;
        int32_t amax;
        eo_target_stats(zj, V, inv_temp, &m, &s, &amax);
        if (j == g) {   /* every proposal accepted: the bonus token */
            tokens[j] = greedy ? amax : eo_draw(zj, V, inv_temp, m, s, S, n_S, NULL, w[j]);
            break;
        }
        if (x[j] < 0 || x[j] >= V) return EO_EINPUT;
        if (greedy) {
            if (x[j] == amax) { tokens[j] = x[j]; ++n_acc; continue; }
            tokens[j] = amax;
            break;
        }
        int i = eo_find_sorted(S, n_S, x[j]);
        const float *qj = qS + (int64_t)j * n_S;
        if (i < 0 || !(qj[i] > 0.0f)) return 3;
        double p = exp((double)zj[x[j]] * inv_temp - m) / s;
        double a = p / (double)qj[i];
        if (a > 1.0) a = 1.0;
        if (u[j] < a) { tokens[j] = x[j]; ++n_acc; continue; }
        tokens[j] = eo_draw(zj, V, inv_temp, m, s, S, n_S, qj, w[j]);
        break;
    }
    *n_acc_out = n_acc;
    return EO_OK;
}

/* ------------------------------------------------------------------ */
/* N4: coverage of the active vocabulary against a     */
/* target distribution -- the covered mass of Eq. 2's constraint      */
/* "sum_{x in V_t} p >= 1 - eps_cov" and App. E's "covered  */
/* probability mass" and Recall@k.         */
/* Row r: p_r(v) = exp(z_r[v] it - m_r) / s_r over [0, V), fp64;       */
/*   mass_r = sum_{v in S} p_r(v);                                     */
/*   recall_r[k] = |S n top-k(p_r)| / k, top-k by (p desc, id asc).   */
/* Out: mass [n_rows], recall [n_rows][n_ks] (fp64).                  */
/* ------------------------------------------------------------------ */
typedef struct { float z; int32_t id; } eo_zid;
static int eo_cmp_zid_desc(const void *a, const void *b) {
    const eo_zid *x = (const eo_zid *)a, *y = (const eo_zid *)b;
    if (x->z > y->z) return -1;
    if (x->z < y->z) return 1;
    return (x->id > y->id) - (x->id < y->id);
}

int eo_coverage(const float *z, int n_rows, int V, const int32_t *S, int n_S, double inv_temp,
                const int32_t *ks, int n_ks, double *mass, double *recall) {
    if (!z || n_rows < 0 || V < 1 || n_S < 0 || (n_S > 0 && !S) || !(inv_temp > 0.0) || n_ks < 0 ||
        (n_ks > 0 && (!ks || !recall)) || !mass)
        return EO_EINPUT;
    for (int i = 0; i < n_S; ++i)
        if (S[i] < 0 || S[i] >= V || (i > 0 && S[i - 1] >= S[i])) return EO_EINPUT;
    for (int t = 0; t < n_ks; ++t)
        if (ks[t] < 1 || ks[t] > V) return EO_EINPUT;
    eo_zid *order = (eo_zid *)malloc(sizeof(eo_zid) * (size_t)V);
    if (!order) return EO_EINPUT;
    for (int r = 0; r < n_rows; ++r) {
        const float *zr = z + (int64_t)r * V;
        double M = -INFINITY;
        for (int v = 0; v < V; ++v) if ((double)zr[v] * inv_temp > M) M = (double)zr[v] * inv_temp;
        double s = 0.0;
        for (int v = 0; v < V; ++v) s += exp((double)zr[v] * inv_temp - M);
        double cm = 0.0;
        for (int i = 0; i < n_S; ++i) cm += exp((double)zr[S[i]] * inv_temp - M) / s;
        mass[r] = cm;
        if (n_ks == 0) continue;
        /* p order = logit order (inv_temp > 0); ties by the smaller id */
        for (int v = 0; v < V; ++v) { order[v].z = zr[v]; order[v].id = v; }
        qsort(order, (size_t)V, sizeof(eo_zid), eo_cmp_zid_desc);
        for (int t = 0; t < n_ks; ++t) {
            int hit = 0;
            for (int i = 0; i < ks[t]; ++i) hit += eo_find_sorted(S, n_S, order[i].id) >= 0;
            recall[(int64_t)r * n_ks + t] = (double)hit / (double)ks[t];
        }
    }
    free(order);
    return EO_OK;
}

/* ------------------------------------------------------------------ */
/* N3: the curriculum-weighted distillation objective  */
/* of Eq. lora_objective with the adaptive horizon weights */
/* of Eq. curriculum_weight, forward and gradient with    */
/* respect to the draft logits only (the LoRA loop is out of scope).   */
/* Trajectory b, step j (0-based; the paper's j-1): on the retained   */
/* support of K target logits,                                         */
/*   p_hat = softmax(zp[b][j] / T),  p_til = softmax(zq[b][j] / T),    */
/*   L_base[b] = logsumexp(zq[b][0]) - zq[b][0][v_b]  (the first-step */
/*     cross entropy against the verified token at support index v_b, */
/*     temperature 1 -- reading K1),                                   */
/*   w[b][j] = exp(-beta * L_base[b] * j),                             */
/*   J[b] = sum_j w[b][j] T^2 KL(p_hat || p_til),                      */
/*   dJ/dzq[b][j][i] = w[b][j] T (p_til[i] - p_hat[i])  (w held fixed: */
/*     the weight is a confidence proxy, reading K1).                  */
/* fp64 throughout. Out: J [B], grad [B][g][K], w [B][g].             */
/* ------------------------------------------------------------------ */
static void eo_softmax_row(const float *z, int K, double scale, double *p, double *lse) {
    double M = -INFINITY;
    for (int i = 0; i < K; ++i) if ((double)z[i] * scale > M) M = (double)z[i] * scale;
    double s = 0.0;
    for (int i = 0; i < K; ++i) s += exp((double)z[i] * scale - M);
    for (int i = 0; i < K; ++i) p[i] = exp((double)z[i] * scale - M) / s;
    if (lse) *lse = M + log(s);
}

int eo_kd_loss(int B, int g, int K, const float *zp, const float *zq, const int32_t *verified, double T,
               double beta, double *J, double *grad, double *w_out) {
    if (B < 0 || g < 1 || K < 1 || !zp || !zq || !verified || !J || !(T > 0.0) || !(beta >= 0.0)) return EO_EINPUT;
    double *ph = (double *)malloc(sizeof(double) * (size_t)K * 2);
    if (!ph) return EO_EINPUT;
    double *pt = ph + K;
    for (int b = 0; b < B; ++b) {
        if (verified[b] < 0 || verified[b] >= K) { free(ph); return EO_EINPUT; }
        const float *q0 = zq + (int64_t)b * g * K;
        double lse0;
        eo_softmax_row(q0, K, 1.0, pt, &lse0);
        const double Lb = lse0 - (double)q0[verified[b]];
        double tot = 0.0;
        for (int j = 0; j < g; ++j) {
            const float *zpj = zp + ((int64_t)b * g + j) * K, *zqj = zq + ((int64_t)b * g + j) * K;
            const double w = exp(-beta * Lb * (double)j);
            eo_softmax_row(zpj, K, 1.0 / T, ph, NULL);
            eo_softmax_row(zqj, K, 1.0 / T, pt, NULL);
            double kl = 0.0;
            for (int i = 0; i < K; ++i)
                if (ph[i] > 0.0) kl += ph[i] * (log(ph[i]) - log(pt[i]));
            tot += w * T * T * kl;
            if (grad)
                for (int i = 0; i < K; ++i) grad[((int64_t)b * g + j) * K + i] = w * T * (pt[i] - ph[i]);
            if (w_out) w_out[(int64_t)b * g + j] = w;
        }
        J[b] = tot;
    }
    free(ph);
    return EO_OK;
}

/* ------------------------------------------------------------------ */
/* N1: the dynamic buffer's Adaptive Replacement Cache */
/* (App. A.3) and the incremental   */
/* subset update it drives.                                           */
/* Lists are arrays in LRU -> MRU order. Residents carry the step of  */
/* their admission (reading A1: residency counts from admission;      */
/* promotions keep it).                                                */
/*   touch(t): t in T1 -> T2 MRU; t in T2 -> T2 MRU; else miss.        */
/*   admit(tokens, step) = one OOV event (warm-up counts events):      */
/*     resident -> touch; in B1 -> (after warm-up) p = min(c, p +      */
/*     max(1, |B2| / |B1|)), to T2; in B2 -> (after warm-up) p = max(0, */
/*     p - max(1, |B1| / |B2|)), to T2; else to T1 (MRU). Before an    */
/*     insertion into a full cache one eviction: from T1 if |T1| > p   */
/*     (or T2 is empty), else from T2; within the list the LRU-most    */
/*     member resident >= min_res steps; if that list has none, the    */
/*     other list's (reading A2); if nobody has, plain LRU of the      */
/*     chosen list. Evicted tokens go to B1 / B2 (MRU), ghost  */
/*     lists trimmed at their LRU end to their caps. Integer division  */
/*     in the adaptation deltas (p is an integer).              */
/* ------------------------------------------------------------------ */
#define EO_ARC_MAX 4096
typedef struct {
    int c, p, b1cap, b2cap, min_res, warmup, events;
    int n1, n2, nb1, nb2;
    int32_t t1[EO_ARC_MAX], t2[EO_ARC_MAX], b1[EO_ARC_MAX], b2[EO_ARC_MAX];
    int64_t s1[EO_ARC_MAX], s2[EO_ARC_MAX];   /* admission steps of T1 / T2 members */
} eo_arc;

static int eo_arc_find(const int32_t *a, int n, int32_t t) {
    for (int i = 0; i < n; ++i) if (a[i] == t) return i;
    return -1;
}
static void eo_arc_del(int32_t *a, int64_t *s, int *n, int i) {
    for (int k = i; k + 1 < *n; ++k) { a[k] = a[k + 1]; if (s) s[k] = s[k + 1]; }
    (*n)--;
}
static void eo_arc_push(int32_t *a, int64_t *s, int *n, int32_t t, int64_t st) {
    a[*n] = t;
    if (s) s[*n] = st;
    (*n)++;
}
static void eo_arc_ghost(int32_t *g, int *n, int cap, int32_t t) {
    eo_arc_push(g, NULL, n, t, 0);
    while (*n > cap) eo_arc_del(g, NULL, n, 0);
}

size_t eo_arc_size(void) { return sizeof(eo_arc); }

int eo_arc_init(eo_arc *a, int c, int p0, int b1cap, int b2cap, int min_res, int warmup) {
    if (!a || c < 1 || c > EO_ARC_MAX || b1cap < 0 || b1cap > EO_ARC_MAX || b2cap < 0 || b2cap > EO_ARC_MAX ||
        min_res < 0 || warmup < 0)
        return EO_EINPUT;
    memset(a, 0, sizeof(*a));
    a->c = c; a->p = p0 < 0 ? 0 : (p0 > c ? c : p0);
    a->b1cap = b1cap; a->b2cap = b2cap; a->min_res = min_res; a->warmup = warmup;
    return EO_OK;
}

int eo_arc_touch(eo_arc *a, int32_t t, int64_t step) {
    (void)step;
    int i = eo_arc_find(a->t1, a->n1, t);
    if (i >= 0) {
        int64_t s = a->s1[i];
        eo_arc_del(a->t1, a->s1, &a->n1, i);
        eo_arc_push(a->t2, a->s2, &a->n2, t, s);
        return 1;
    }
    i = eo_arc_find(a->t2, a->n2, t);
    if (i >= 0) {
        int64_t s = a->s2[i];
        eo_arc_del(a->t2, a->s2, &a->n2, i);
        eo_arc_push(a->t2, a->s2, &a->n2, t, s);
        return 1;
    }
    return 0;
}

/* the LRU-most member of list (a, s, n) resident >= min_res at step; -1 if none */
static int eo_arc_eligible(const eo_arc *A, const int64_t *s, int n, int64_t step) {
    for (int i = 0; i < n; ++i) if (step - s[i] >= A->min_res) return i;
    return -1;
}

static int32_t eo_arc_evict(eo_arc *A, int64_t step) {
    int from1 = (A->n1 > 0 && (A->n1 > A->p || A->n2 == 0));
    int i = from1 ? eo_arc_eligible(A, A->s1, A->n1, step) : eo_arc_eligible(A, A->s2, A->n2, step);
    if (i < 0) {   /* reading A2: the other list's eligible member, else plain LRU of the chosen list */
        int j = from1 ? eo_arc_eligible(A, A->s2, A->n2, step) : eo_arc_eligible(A, A->s1, A->n1, step);
        if (j >= 0) { from1 = !from1; i = j; } else i = 0;
    }
    int32_t t;
    if (from1) {
        t = A->t1[i];
        eo_arc_del(A->t1, A->s1, &A->n1, i);
        eo_arc_ghost(A->b1, &A->nb1, A->b1cap, t);
    } else {
        t = A->t2[i];
        eo_arc_del(A->t2, A->s2, &A->n2, i);
        eo_arc_ghost(A->b2, &A->nb2, A->b2cap, t);
    }
    return t;
}

int eo_arc_admit(eo_arc *A, const int32_t *tokens, int n, int64_t step, int32_t *evicted, int *n_evicted) {
    if (!A || n < 0 || (n > 0 && !tokens) || !n_evicted) return EO_EINPUT;
    A->events++;
    const int adapt = A->events > A->warmup;
    int ne = 0;
    for (int k = 0; k < n; ++k) {
        int32_t t = tokens[k];
        if (eo_arc_touch(A, t, step)) continue;
        int to2 = 0, i;
        if ((i = eo_arc_find(A->b1, A->nb1, t)) >= 0) {
            if (adapt) {
                int d = A->nb2 / A->nb1; if (d < 1) d = 1;
                A->p = A->p + d > A->c ? A->c : A->p + d;
            }
            eo_arc_del(A->b1, NULL, &A->nb1, i);
            to2 = 1;
        } else if ((i = eo_arc_find(A->b2, A->nb2, t)) >= 0) {
            if (adapt) {
                int d = A->nb1 / A->nb2; if (d < 1) d = 1;
                A->p = A->p - d < 0 ? 0 : A->p - d;
            }
            eo_arc_del(A->b2, NULL, &A->nb2, i);
            to2 = 1;
        }
        if (A->n1 + A->n2 >= A->c) {
            int32_t e = eo_arc_evict(A, step);
            if (evicted) evicted[ne] = e;
            ne++;
        }
        if (to2) eo_arc_push(A->t2, A->s2, &A->n2, t, step);
        else eo_arc_push(A->t1, A->s1, &A->n1, t, step);
    }
    *n_evicted = ne;
    return EO_OK;
}

/* state dump: n1, n2, nb1, nb2, p followed by the four lists (LRU -> MRU) */
int eo_arc_state(const eo_arc *A, int32_t *out, int cap) {
    int need = 5 + A->n1 + A->n2 + A->nb1 + A->nb2;
    if (!out || cap < need) return EO_EINPUT;
    int o = 0;
    out[o++] = A->n1; out[o++] = A->n2; out[o++] = A->nb1; out[o++] = A->nb2; out[o++] = A->p;
    for (int i = 0; i < A->n1; ++i) out[o++] = A->t1[i];
    for (int i = 0; i < A->n2; ++i) out[o++] = A->t2[i];
    for (int i = 0; i < A->nb1; ++i) out[o++] = A->b1[i];
    for (int i = 0; i < A->nb2; ++i) out[o++] = A->b2[i];
    return EO_OK;
}

/* incremental subset update: S' = sort((S \ remove) u add), S sorted unique,
 * remove a subset of S, add disjoint from S \ remove (the definition, sorted). */
static int eo_cmp_i32b(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}
int eo_subset_update(const int32_t *S, int n, const int32_t *rem, int nr, const int32_t *add, int na,
                     int32_t *out, int *n_out) {
    if ((n > 0 && !S) || (nr > 0 && !rem) || (na > 0 && !add) || !out || !n_out) return EO_EINPUT;
    int o = 0;
    for (int i = 0; i < n; ++i) {
        int gone = 0;
        for (int j = 0; j < nr; ++j) if (rem[j] == S[i]) { gone = 1; break; }
        if (!gone) out[o++] = S[i];
    }
    for (int j = 0; j < na; ++j) out[o++] = add[j];
    qsort(out, (size_t)o, sizeof(int32_t), eo_cmp_i32b);
    for (int i = 1; i < o; ++i) if (out[i - 1] == out[i]) return EO_EINPUT;   /* add not disjoint */
    *n_out = o;
    return EO_OK;
}
