"""Pins the C oracle (oracle/) to things other than itself (CPU only).

Each test names the passage or property it checks. Chosen so that a plausible
mistake anywhere in the oracle (a dropped term, a wrong sign or index, a
transposed operand, a wrong bf16 decode, a wrong tie rule, a wrong cap or
formation order, a wrong LSE combine) fails at least one of them:
  * worked examples copied into tests/golden/spec_examples.json (cited);
  * an independent implementation of a definition (numpy/ml_dtypes matmul,
    scipy logsumexp, np.lexsort, the pure-Python brute force in brute.py);
  * closed forms and invariants (sum p = 1, equal logits, shift, linearity,
    merge(split) = unsplit, shard-order invariance).
"""
import json
import math
import os

import ml_dtypes
import numpy as np
import pytest
from scipy.special import logsumexp

import synth
from tests import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def f32(a):
    return np.asarray(a, dtype=np.float32)


def csr_from_rows(V, rows):
    row_ptr = [0]
    col = []
    for u in range(V):
        col.extend(rows.get(str(u), rows.get(u, [])))
        row_ptr.append(len(col))
    return np.array(row_ptr, np.int32), np.array(col if col else [0], np.int32)


def bf16_decode_independent(bits):
    # ml_dtypes' bfloat16 is an independent implementation of the format
    return np.asarray(bits, np.uint16).view(ml_dtypes.bfloat16).astype(np.float64)


# ---------------------------------------------------------------- a5 logits
def test_projection_example(oracle_mod):
    g = GOLD["projection"]
    z = oracle_mod.subset_logits(f32(g["W"]), f32([g["h"]]), [0, 1, 2])
    assert z.tolist() == [g["logits"]]


def test_projection_zero(oracle_mod):
    g = GOLD["projection_zero"]
    z = oracle_mod.subset_logits(f32(g["W"]), f32([g["h"]]), [0, 1, 2])
    assert z.tolist() == [g["logits"]]


def test_projection_subset_selects_rows(oracle_mod):
    g = GOLD["projection"]
    z = oracle_mod.subset_logits(f32(g["W"]), f32([g["h"]]), [2, 0])
    assert z.tolist() == [[5, 2]]


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_full_vocab_subset_equals_unpruned_matmul(oracle_mod, dtype):
    """North star: the full-vocab subset reproduces the unpruned projection."""
    V, d, n_h = 300, 96, 5
    W = synth.matrix(1, V, d, 0.02, dtype)
    H = synth.matrix(2, n_h, d, 1.0, dtype)
    dec = bf16_decode_independent if dtype == "bf16" else (lambda a: np.asarray(a, np.float64))
    ref = dec(H) @ dec(W).T
    z = oracle_mod.subset_logits(W, H, np.arange(V))
    np.testing.assert_allclose(z, ref, rtol=1e-12, atol=1e-12)
    # inv_temp scales
    z2 = oracle_mod.subset_logits(W, H, np.arange(V), inv_temp=1 / 0.7)
    np.testing.assert_allclose(z2, ref / 0.7, rtol=1e-12, atol=1e-12)


def test_linearity(oracle_mod):
    """l(a h1 + b h2) = a l(h1) + b l(h2)."""
    V, d = 50, 16
    W = synth.matrix(3, V, d, 1.0, "fp32")
    h1 = synth.int_matrix(4, 1, d, "fp32")     # integer h: a*h1 + b*h2 exact in fp32
    h2 = synth.int_matrix(5, 1, d, "fp32")
    a, b = 0.5, -2.0
    hc = (a * h1.astype(np.float64) + b * h2.astype(np.float64)).astype(np.float32)
    S = np.arange(V)
    lhs = oracle_mod.subset_logits(W, hc, S)
    rhs = a * oracle_mod.subset_logits(W, h1, S) + b * oracle_mod.subset_logits(W, h2, S)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-9, atol=1e-9)


def test_sharded_rows_map(oracle_mod):
    """§8(e) interleaved ownership: shard r holds id v at local row v // R."""
    V, d, R = 97, 8, 3
    W = synth.int_matrix(6, V, d, "fp32")
    H = synth.int_matrix(7, 2, d, "fp32")
    S = np.sort(np.random.default_rng(0).choice(V, 40, replace=False)).astype(np.int32)
    full = oracle_mod.subset_logits(W, H, S)
    for r in range(R):
        Sr = S[S % R == r]
        zr = oracle_mod.subset_logits(np.ascontiguousarray(W[r::R]), H, Sr, R=R)
        np.testing.assert_array_equal(zr, full[:, S % R == r])


# ------------------------------------------------------- a6/a7 softmax, topk
@pytest.mark.parametrize("name", ["restricted_singleton", "restricted_equal", "restricted_2_0"])
def test_restricted_examples(oracle_mod, name):
    g = GOLD[name]
    z = np.array([g["logits"]], np.float64)
    r = oracle_mod.softmax_topk(z, g["support"], len(g["support"]))
    got = dict(zip(r["ids"][0].tolist(), r["probs"][0].tolist()))
    tol = g.get("tol", 1e-12)
    for sid, p in zip(g["support"], g["probs"]):
        assert abs(got[sid] - p) <= tol


def test_topk_examples(oracle_mod):
    g = GOLD["topk"]
    r = oracle_mod.softmax_topk(np.array([g["logits"]], float), [0, 1, 2], g["k"])
    assert r["ids"][0].tolist() == g["ids"] and r["vals"][0].tolist() == g["vals"]
    g = GOLD["topk_tie"]
    r = oracle_mod.softmax_topk(np.array([g["logits"]], float), [0, 1, 2], g["k"])
    assert r["ids"][0].tolist() == g["ids"]


def test_topk_ties_follow_subset_ids_not_positions(oracle_mod):
    # tie between ids 9 and 4 (support order [4, 9]): lower id wins
    r = oracle_mod.softmax_topk(np.array([[1.0, 1.0, 0.0]]), [4, 9, 11], 2)
    assert r["ids"][0].tolist() == [4, 9]


def test_topk_k_equals_support_is_permutation_and_lexsort(oracle_mod):
    rng = np.random.default_rng(0)
    S = np.sort(rng.choice(500, 64, replace=False)).astype(np.int32)
    z = rng.integers(-3, 4, size=(3, 64)).astype(np.float64)  # many exact ties
    r = oracle_mod.softmax_topk(z, S, 64)
    for i in range(3):
        assert sorted(r["ids"][i].tolist()) == S.tolist()
        order = np.lexsort((S, -z[i]))  # independent (-z, id) sort
        assert r["ids"][i].tolist() == S[order].tolist()


def test_softmax_closed_forms(oracle_mod):
    rng = np.random.default_rng(1)
    z = rng.standard_normal((4, 200)) * 3
    S = np.arange(200, dtype=np.int32)
    r = oracle_mod.softmax_topk(z, S, 200)
    for i in range(4):
        assert abs(math.fsum(r["probs"][i]) - 1.0) < 1e-12
        assert abs(r["lse"][i] - logsumexp(z[i])) < 1e-12
        assert r["m"][i] == z[i].max()
        assert abs(r["lse"][i] - (r["m"][i] + math.log(r["s"][i]))) < 1e-12
    # equal logits c -> LSE = c + ln n
    r = oracle_mod.softmax_topk(np.full((1, 37), 2.5), np.arange(37), 3)
    assert abs(r["lse"][0] - (2.5 + math.log(37))) < 1e-12
    assert r["ids"][0].tolist() == [0, 1, 2]


def test_shift_invariance_via_augmented_column(oracle_mod):
    """adding c to every logit (h'=[h,c], W'=[W,1]) keeps ids and p; LSE + c."""
    V, d, c = 64, 12, 3.0
    W = synth.matrix(8, V, d, 1.0, "fp32")
    H = synth.matrix(9, 2, d, 1.0, "fp32")
    W2 = np.concatenate([W, np.ones((V, 1), np.float32)], 1)
    H2 = np.concatenate([H, np.full((2, 1), c, np.float32)], 1)
    S = np.arange(0, V, 2, dtype=np.int32)
    a = oracle_mod.subset_logits_topk(W, H, S, 5)
    b = oracle_mod.subset_logits_topk(W2, H2, S, 5)
    np.testing.assert_array_equal(a["ids"], b["ids"])
    np.testing.assert_allclose(a["probs"], b["probs"], atol=1e-12)
    np.testing.assert_allclose(a["lse"] + c, b["lse"], atol=1e-9)


@pytest.mark.parametrize("inv_temp", [1.0, 1 / 0.7])
def test_restricted_equals_conditioned_full_softmax_bruteforce(oracle_mod, inv_temp):
    """S:97, brute force for V <= 64 (brute.py, fsum)."""
    V, d = 64, 8
    W = synth.int_matrix(10, V, d, "fp32")
    H = synth.int_matrix(11, 1, d, "fp32")
    full = [float(brute.dot(H[0], W[v])) for v in range(V)]
    S = [1, 5, 6, 17, 30, 31, 44, 63]
    r = oracle_mod.subset_logits_topk(W, H, np.array(S, np.int32), len(S), inv_temp=inv_temp)
    cond = brute.full_softmax_conditioned(full, S, inv_temp)
    got = dict(zip(r["ids"][0].tolist(), r["probs"][0].tolist()))
    for v in S:
        assert abs(got[v] - cond[v]) < 1e-12
    assert r["ids"][0].tolist() == brute.order_desc([full[v] for v in S], S)


# ----------------------------------------------------------- a2 semantic
def test_mips_example(oracle_mod):
    g = GOLD["mips"]
    s = oracle_mod.sem_scores(f32(g["E"]), f32(g["q"]))
    assert s.tolist() == g["scores"]
    assert oracle_mod.topn(s, g["N"]).tolist() == g["ids"]


def test_sem_scores_bf16_against_independent_decode(oracle_mod):
    V, d = 257, 128
    E = synth.matrix(12, V, d, 0.02, "bf16")
    q = synth.matrix(13, 1, d, 1.0, "fp32")
    s = oracle_mod.sem_scores(E, q)
    ref = bf16_decode_independent(E) @ q[0].astype(np.float64)
    np.testing.assert_allclose(s, ref, rtol=1e-12, atol=1e-13)


def test_topn_full_permutation_and_ties(oracle_mod):
    rng = np.random.default_rng(2)
    s = rng.integers(-5, 6, size=300).astype(np.float64)   # heavy exact ties
    ids = oracle_mod.topn(s, 300)
    assert sorted(ids.tolist()) == list(range(300))
    assert ids.tolist() == np.lexsort((np.arange(300), -s)).tolist()
    assert oracle_mod.topn(s, 17).tolist() == ids[:17].tolist()


# ------------------------------------------------------------ a3 graph
def test_graph_expand_examples(oracle_mod):
    row_ptr, col = csr_from_rows(GOLD["graph"]["V"], GOLD["graph"]["rows"])
    for name in ["graph_expand_1", "graph_expand_2", "graph_expand_none"]:
        g = GOLD[name]
        assert oracle_mod.graph_expand(g["seeds"], row_ptr, col, g["per_seed"]).tolist() == g["out"]


@pytest.mark.parametrize("name", ["ctx", "ctx_tie"])
def test_ctx_tokens_examples(oracle_mod, name):
    g = GOLD[name]
    assert oracle_mod.ctx_tokens(g["ctx"], g["V"], g["min_count"], g["n_max"]).tolist() == g["out"]


# ------------------------------------------------------------ a4 union
def _onehot_sem(V, order):
    """E (d=1) and q=[1] whose semantic order starts with `order`."""
    E = np.zeros((V, 1), np.float32)
    for rank, v in enumerate(order):
        E[v, 0] = len(order) - rank
    return E, f32([1.0])


@pytest.mark.parametrize("n_dyn", [4, 6])
def test_formation_worked_example(oracle_mod, n_dyn):
    g = GOLD["formation"]
    E, q = _onehot_sem(g["V"], g["sem_order"])
    row_ptr, col = csr_from_rows(g["V"], g["rows"])
    r = oracle_mod.build_subset(E, q, g["static"], g["seeds"], row_ptr, col,
                                n_sem=len(g["sem_order"]), n_graph_sem_seeds=g["n_graph_sem_seeds"],
                                per_seed=g["per_seed"], n_dyn=n_dyn)
    assert r["sem"].tolist() == g["sem_order"]
    assert r["S"].tolist() == g[f"S_ndyn{n_dyn}"]
    assert r["dyn"].tolist() == g[f"dyn_ndyn{n_dyn}"]


def test_union_examples(oracle_mod):
    for name in ["union", "union_overlap"]:
        g = GOLD[name]
        V = 20
        # dyn enters as seeds; n_sem = 0 so nothing else contributes
        E = np.zeros((V, 1), np.float32)
        r = oracle_mod.build_subset(E, f32([1.0]), g["static"], g["dyn"], None, None,
                                    n_sem=0, n_graph_sem_seeds=0, per_seed=0, n_dyn=8)
        S = set(r["S"].tolist())
        if "contains" in g:
            assert all(v in S for v in g["contains"]) and all(v not in S for v in g["absent"])
        if "size" in g:
            assert len(S) == g["size"]


def test_cap_example(oracle_mod):
    g = GOLD["cap"]
    V = 100
    seeds = list(range(20, 40))               # 20 unique seeds
    rows = {str(20): list(range(60, 80))}      # 20 new graph ids from the first seed
    row_ptr, col = csr_from_rows(V, rows)
    E = np.zeros((V, 1), np.float32)
    r = oracle_mod.build_subset(E, f32([1.0]), [0], seeds, row_ptr, col, n_sem=0,
                                n_graph_sem_seeds=0, per_seed=20, n_dyn=g["cap"])
    assert len(r["dyn"]) == g["n_dyn_out"]
    assert r["dyn"].tolist() == seeds + list(range(60, 72))  # formation order, 20 + first 12


@pytest.mark.parametrize("seed", range(6))
def test_build_subset_bruteforce(oracle_mod, seed):
    rng = np.random.default_rng(100 + seed)
    V, d = 64, 6
    E = synth.int_matrix(seed, V, d, "fp32")
    q = synth.int_matrix(seed + 50, 1, d, "fp32")
    static = np.sort(rng.choice(V, 12, replace=False)).astype(np.int32)
    seeds = rng.choice(V, 4, replace=False).astype(np.int32)
    rows = {}
    for u in range(V):
        k = int(rng.integers(0, 5))
        rows[str(u)] = [int(x) for x in rng.choice(V, k, replace=False)]
    row_ptr, col = csr_from_rows(V, rows)
    n_sem, ngs, per, n_dyn = 10, 3, 2, int(rng.integers(3, 20))
    r = oracle_mod.build_subset(E, q, static, seeds, row_ptr, col, n_sem=n_sem,
                                n_graph_sem_seeds=ngs, per_seed=per, n_dyn=n_dyn)
    bS, bsem, bdyn = brute.build_subset(E.tolist(), q[0].tolist(), static.tolist(), seeds.tolist(),
                                        {int(k): v for k, v in rows.items()}, n_sem, ngs, per, n_dyn)
    assert r["sem"].tolist() == bsem
    assert r["dyn"].tolist() == bdyn
    assert r["S"].tolist() == bS
    # invariants: sorted unique, in range, static subset, budget
    S = r["S"]
    assert np.all(np.diff(S) > 0) and S.min() >= 0 and S.max() < V
    assert set(static.tolist()) <= set(S.tolist())
    assert len(set(S.tolist()) - set(static.tolist())) <= n_dyn


def test_build_subset_rejects_unsorted_static(oracle_mod):
    E = np.zeros((10, 1), np.float32)
    with pytest.raises(ValueError):
        oracle_mod.build_subset(E, f32([1.0]), [3, 1], [], None, None, n_sem=0,
                                n_graph_sem_seeds=0, per_seed=0, n_dyn=2)


# ------------------------------------------------------------ a8 merge
def test_merge_worked_example(oracle_mod):
    g = GOLD["merge"]
    z = np.array([g["z"]], np.float64)
    R, k = g["R"], g["k"]
    trip = []
    for r in range(R):
        Sr = np.array([v for v in range(6) if v % R == r], np.int32)
        trip.append(oracle_mod.softmax_topk(z[:, Sr], Sr, k))
    for r in range(R):
        assert abs(trip[r]["m"][0] - g["m"][r]) < g["tol"]
        assert abs(trip[r]["s"][0] - g["s"][r]) < g["tol"]
    out = oracle_mod.merge(np.stack([t["ids"] for t in trip]), np.stack([t["vals"] for t in trip]),
                           np.stack([t["m"] for t in trip]), np.stack([t["s"] for t in trip]), k)
    assert out["ids"][0].tolist() == g["ids"]
    assert abs(out["lse"][0] - g["lse"]) < g["tol"]
    np.testing.assert_allclose(out["probs"][0], g["probs"], atol=g["tol"])


@pytest.mark.parametrize("R", [1, 2, 3, 4])
def test_merge_of_split_equals_unsplit(oracle_mod, R):
    V, d, n_h, k = 211, 16, 3, 7
    W = synth.int_matrix(20, V, d, "fp32")       # integer data: real ties across shards
    H = synth.int_matrix(21, n_h, d, "fp32")
    S = np.sort(np.random.default_rng(3).choice(V, 90, replace=False)).astype(np.int32)
    ref = oracle_mod.subset_logits_topk(W, H, S, k)
    parts = [oracle_mod.subset_logits_topk(np.ascontiguousarray(W[r::R]), H, S[S % R == r], k, R=R)
             for r in range(R)]
    st = lambda key: np.stack([p[key] for p in parts])
    out = oracle_mod.merge(st("ids"), st("vals"), st("m"), st("s"), k)
    np.testing.assert_array_equal(out["ids"], ref["ids"])
    np.testing.assert_allclose(out["lse"], ref["lse"], rtol=1e-12)
    np.testing.assert_allclose(out["probs"], ref["probs"], atol=1e-12)
    # shard order invariance
    perm = np.random.default_rng(4).permutation(R)
    out2 = oracle_mod.merge(st("ids")[perm], st("vals")[perm], st("m")[perm], st("s")[perm], k)
    np.testing.assert_array_equal(out2["ids"], out["ids"])
    np.testing.assert_allclose(out2["lse"], out["lse"], rtol=1e-12)


def test_merge_skips_empty_shard_and_pads(oracle_mod):
    z = np.array([[0.5, 1.5]])
    a = oracle_mod.softmax_topk(z, [2, 4], 3)
    empty = oracle_mod.softmax_topk(np.zeros((1, 0)), [], 3)
    assert empty["m"][0] == -np.inf and empty["s"][0] == 0 and empty["ids"][0].tolist() == [-1, -1, -1]
    st = lambda key: np.stack([a[key], empty[key]])
    out = oracle_mod.merge(st("ids"), st("vals"), st("m"), st("s"), 3)
    assert out["ids"][0].tolist() == [4, 2, -1]
    assert abs(out["lse"][0] - logsumexp([0.5, 1.5])) < 1e-12


# ------------------------------------------------ batched serving (config Bt)
def test_batched_build_worked_example(oracle_mod):
    """Two sequences on the worked formation example (golden "formation"): sequence 0
    keeps its seeds [5, 2]; sequence 1 has none, so by the same rules (C4, C6, C7)
    G = S_sem[:2] = [7, 5], S_graph = [1, 10, 6, 7], C = [7, 5, 9, 1, 10, 6, 7] and,
    skipping static 1, dyn = [7, 5, 9, 10] at N_dyn = 4 (derived by hand)."""
    g = GOLD["formation"]
    E, q = _onehot_sem(g["V"], g["sem_order"])
    row_ptr, col = csr_from_rows(g["V"], g["rows"])
    Q = np.stack([q, q])
    dyn, offs = oracle_mod.build_subset_batched(
        E, Q, g["static"], g["seeds"], [0, len(g["seeds"]), len(g["seeds"])], row_ptr, col,
        n_sem=len(g["sem_order"]), n_graph_sem_seeds=g["n_graph_sem_seeds"], per_seed=g["per_seed"], n_dyn=4)
    assert offs.tolist() == [0, 4, 8]
    assert dyn[0:4].tolist() == sorted(g["dyn_ndyn4"])
    assert dyn[4:8].tolist() == [5, 7, 9, 10]


@pytest.mark.parametrize("seed", range(3))
def test_batched_build_bruteforce(oracle_mod, seed):
    """Every sequence of a batch equals the pure-Python brute force of its own build,
    restricted to the dynamic part (static excluded, sorted)."""
    rng = np.random.default_rng(300 + seed)
    V, d, B = 64, 6, 4
    E = synth.int_matrix(seed + 7, V, d, "fp32")
    Q = synth.int_matrix(seed + 70, B, d, "fp32")
    static = np.sort(rng.choice(V, 10, replace=False)).astype(np.int32)
    n_seed = rng.integers(0, 5, B)
    offs = np.concatenate([[0], np.cumsum(n_seed)]).astype(np.int64)
    seeds = rng.choice(V, int(offs[-1]), replace=True).astype(np.int32)
    rows = {str(u): [int(x) for x in rng.choice(V, int(rng.integers(0, 5)), replace=False)] for u in range(V)}
    row_ptr, col = csr_from_rows(V, rows)
    n_sem, ngs, per, n_dyn = 8, 3, 2, 9
    dyn, doff = oracle_mod.build_subset_batched(E, Q, static, seeds, offs, row_ptr, col, n_sem=n_sem,
                                                n_graph_sem_seeds=ngs, per_seed=per, n_dyn=n_dyn)
    for b in range(B):
        _, _, bdyn = brute.build_subset(E.tolist(), Q[b].tolist(), static.tolist(),
                                        seeds[offs[b]:offs[b + 1]].tolist(),
                                        {int(k): v for k, v in rows.items()}, n_sem, ngs, per, n_dyn)
        assert dyn[doff[b]:doff[b + 1]].tolist() == sorted(bdyn)
        assert not set(bdyn) & set(static.tolist())


def test_ragged_equals_brute_force_per_sequence(oracle_mod):
    """Each row's triple over its own V_b = static u dyn_b equals the brute-force
    restricted softmax / ordering on that support."""
    V, d, k = 48, 5, 4
    W = synth.int_matrix(40, V, d, "fp32")
    H = synth.int_matrix(41, 7, d, "fp32")
    static = np.array([1, 4, 9, 16, 25, 36], np.int32)
    dyn_lists = [[0, 2, 3], [], [40, 41, 47, 5]]
    h_off = [0, 3, 4, 7]
    dyn = np.array(sum(dyn_lists, []), np.int32)
    doff = np.concatenate([[0], np.cumsum([len(x) for x in dyn_lists])])
    out = oracle_mod.subset_logits_topk_ragged(W, H, h_off, static, dyn, doff, k)
    for b, dl in enumerate(dyn_lists):
        supp = sorted(set(static.tolist()) | set(dl))
        for r in range(h_off[b], h_off[b + 1]):
            logits = [float(brute.dot(H[r], W[v])) for v in supp]
            order = brute.order_desc(logits, supp)[:k]
            assert out["ids"][r].tolist() == order
            p = brute.restricted_softmax(logits, supp)
            np.testing.assert_allclose(out["probs"][r], [p[v] for v in order], rtol=1e-12)
            assert abs(out["m"][r] - max(logits)) == 0.0


def test_ragged_equals_merge_of_static_and_dynamic_parts(oracle_mod):
    """static and dyn_b are disjoint, so the ragged result is the two-part merge
    (the shard merge, pinned above) of the static triple and the dyn_b triple."""
    V, d, k = 300, 12, 6
    W = synth.matrix(50, V, d, 0.5, "fp32")
    H = synth.matrix(51, 9, d, 1.0, "fp32")
    rng = np.random.default_rng(52)
    perm = rng.permutation(V)
    static = np.sort(perm[:80]).astype(np.int32)
    dyn_lists = [np.sort(perm[80:110]), np.sort(perm[110:111]), np.sort(perm[111:200])]
    h_off = [0, 4, 5, 9]
    dyn = np.concatenate(dyn_lists).astype(np.int32)
    doff = np.concatenate([[0], np.cumsum([x.size for x in dyn_lists])])
    out = oracle_mod.subset_logits_topk_ragged(W, H, h_off, static, dyn, doff, k)
    st = oracle_mod.subset_logits_topk(W, H, static, k)
    for b in range(3):
        rows = slice(h_off[b], h_off[b + 1])
        dy = oracle_mod.subset_logits_topk(W, H[rows], dyn_lists[b].astype(np.int32), k)
        mg = oracle_mod.merge(np.stack([st["ids"][rows], dy["ids"]]), np.stack([st["vals"][rows], dy["vals"]]),
                              np.stack([st["m"][rows], dy["m"]]), np.stack([st["s"][rows], dy["s"]]), k)
        np.testing.assert_array_equal(out["ids"][rows], mg["ids"])
        np.testing.assert_allclose(out["lse"][rows], mg["lse"], rtol=1e-12)
        np.testing.assert_allclose(out["probs"][rows], mg["probs"], atol=1e-12)


# ---------------------------------------------------------------- N2 verification
# Pins for oracle.verify_chain (eo_verify_chain): the SPEC worked example
# (S:385), the losslessness theorem (the first emitted token is
# distributed exactly as the target, for any draft q supported on V_t) and
# greedy equivalence. The acceptance probability and the draw's CDF are
# recovered from the oracle as a black box by bisection on the uniforms (its
# decisions are monotone in u and w), never from its formulas.

def _bisect(pred, lo=0.0, hi=1.0, it=60):
    """largest x in [lo, hi) with pred(x) true, pred monotone (true then false)"""
    for _ in range(it):
        mid = 0.5 * (lo + hi)
        if pred(mid):
            lo = mid
        else:
            hi = mid
    return lo


def _draw_intervals(fn, V):
    """{token: length of the set of w in [0, 1) that emits it}, fn(w) monotone in w"""
    out = {}
    w0 = 0.0
    while w0 < 1.0:
        t = fn(w0)
        w1 = _bisect(lambda w: fn(w) == t, w0, 1.0)
        if fn(w1) != t:       # numeric guard
            w1 = w0
        nxt = w1 + 1e-15
        out[t] = out.get(t, 0.0) + (min(1.0, nxt) - w0)
        w0 = nxt
    return out


def test_verify_spec_worked_example():
    """p = (0.6, 0.4), q = (0.5, 0.5), proposal 1 -> accept prob 0.8; on a
    rejection the residual is the point mass on token 0."""
    import oracle
    z = np.log(np.array([[0.6, 0.4], [0.5, 0.5]], np.float32))
    q = np.array([[0.5, 0.5]], np.float32)
    acc = lambda u: oracle.verify_chain(z, [1], [0, 1], q, greedy=False, u=[u], w=[0.5, 0.5])[1] == 1
    assert abs(_bisect(acc) - 0.8) < 1e-6
    for w in (0.0, 0.3, 0.999):
        tok, n = oracle.verify_chain(z, [1], [0, 1], q, greedy=False, u=[0.95], w=[w, 0.5])
        assert n == 0 and tok.tolist() == [0]


@pytest.mark.parametrize("seed", range(3))
def test_verify_lossless_first_token(seed):
    """Losslessness: with x ~ q_0 (q supported on a subset S of V),
    u, w uniform, the first emitted token has the target law p_0 exactly:
    sum_x q(x) [a(x) 1{v = x} + (1 - a(x)) P(draw = v | x)] = p(v), within 1e-9.
    a(x) and the draw's law come from the oracle by bisection on u and w."""
    import oracle
    rng = np.random.default_rng(100 + seed)
    V = 7
    S = np.sort(rng.choice(V, 4, replace=False)).astype(np.int32)
    q = rng.dirichlet(np.ones(S.size)).astype(np.float32)
    q = (q / q.astype(np.float64).sum()).astype(np.float32)
    z = rng.normal(size=(2, V)).astype(np.float32)
    p = np.exp(z[0].astype(np.float64) - z[0].max())
    p /= p.sum()
    law = np.zeros(V)
    qd = q.astype(np.float64)
    qd /= qd.sum()
    for i, x in enumerate(S):
        run = lambda u, w: oracle.verify_chain(z, [x], S, q[None, :], greedy=False, u=[u], w=[w, 0.5])
        a = _bisect(lambda u: run(u, 0.5)[1] == 1)
        law[x] += qd[i] * a
        for t, length in _draw_intervals(lambda w: int(run(0.999999999, w)[0][0]) if a < 0.999999999 else x, V).items():
            law[t] += qd[i] * (1.0 - a) * length
    # q sums to 1 only up to fp32 rounding: compare against p with that slack
    assert np.abs(law - p).max() < 1e-6, (law, p)
    # where q(x) > p(x) the proposal is accepted with probability exactly p/q
    i = int(np.argmax(qd / p[S]))
    x = S[i]
    a = _bisect(lambda u: oracle.verify_chain(z, [x], S, q[None, :], greedy=False, u=[u], w=[0.5, 0.5])[1] == 1)
    assert abs(a - min(1.0, p[x] / float(q[i]))) < 1e-9


def test_verify_bonus_draw_is_target_law():
    """All proposals accepted (u = 0): the bonus token is drawn from p_g -- the
    w-intervals of the draw have the lengths p_g(v) (inverse CDF in id order)."""
    import oracle
    rng = np.random.default_rng(7)
    V = 9
    z = rng.normal(size=(2, V)).astype(np.float32)
    S = np.arange(V, dtype=np.int32)
    q = np.full((1, V), 1.0 / V, np.float32)
    x = 3
    fn = lambda w: int(oracle.verify_chain(z, [x], S, q, greedy=False, u=[0.0], w=[0.5, w])[0][1])
    law = _draw_intervals(fn, V)
    p = np.exp(z[1].astype(np.float64) - z[1].max())
    p /= p.sum()
    got = np.array([law.get(v, 0.0) for v in range(V)])
    assert np.abs(got - p).max() < 1e-9
    # id order: the emitted token is non-decreasing in w
    toks = [fn(w) for w in np.linspace(0, 0.999, 50)]
    assert toks == sorted(toks)


def test_verify_greedy_equivalence_and_ties():
    """T = 0 reproduces target greedy decoding token for token; ties of the
    target maximum go to the lower id; a mismatch at j stops with argmax p_j."""
    import oracle
    rng = np.random.default_rng(3)
    g, V = 5, 50
    z = rng.normal(size=(g + 1, V)).astype(np.float32)
    z[2, 11] = z[2, 40] = z[2].max() + 1.0          # a tie: 11 wins
    am = np.argmax(z, axis=1)                        # numpy argmax: first (lower) index
    assert am[2] == 11
    tok, n = oracle.verify_chain(z, am[:g].astype(np.int32), None, None, greedy=True)
    assert n == g and tok.tolist() == am.tolist()
    x = am[:g].copy()
    x[3] = (x[3] + 1) % V
    tok, n = oracle.verify_chain(z, x.astype(np.int32), None, None, greedy=True)
    assert n == 3 and tok.tolist() == am[:4].tolist()


def test_verify_rejects_proposal_outside_support():
    """a proposal with q = 0 is an invariant violation."""
    import oracle
    z = np.zeros((2, 4), np.float32)
    with pytest.raises(ValueError):
        oracle.verify_chain(z, [2], np.array([0, 1], np.int32), np.array([[0.5, 0.5]], np.float32),
                            greedy=False, u=[0.1], w=[0.1, 0.1])


# ---------------------------------------------------------------- N4 coverage
# Pins for oracle.coverage (eo_coverage): SPEC S:173-175 worked examples, an
# independent numpy implementation (scipy softmax in fp64, np.lexsort top-k with
# the smallest-id tie rule of S:171), and the insertion monotonicity of S:178.

def test_coverage_spec_examples():
    import oracle
    z = np.log(np.array([[0.5, 0.3, 0.2]], np.float32))
    m, r = oracle.coverage(z, [0, 2], [2])
    assert abs(m[0] - 0.7) < 1e-7 and r[0, 0] == 0.5
    m, r = oracle.coverage(z, [0, 1, 2], [1, 2, 3])
    assert abs(m[0] - 1.0) < 1e-12 and np.all(r == 1.0)
    z2 = np.array([[0.0, 0.0, -np.inf, -np.inf]], np.float32)   # support {0, 1}
    m, _ = oracle.coverage(z2, [2, 3], [1])
    assert m[0] == 0.0


@pytest.mark.parametrize("integer", [False, True])
def test_coverage_matches_numpy(integer):
    import oracle
    from scipy.special import softmax
    rng = np.random.default_rng(5)
    n, V = 4, 3000
    z = (rng.integers(-3, 4, size=(n, V)) if integer else rng.normal(size=(n, V)) * 1.3).astype(np.float32)
    S = np.sort(rng.choice(V, 700, replace=False)).astype(np.int32)
    ks = [1, 10, 50, 100, 2999]
    m, r = oracle.coverage(z, S, ks, inv_temp=1 / 0.7)
    inS = np.zeros(V, bool)
    inS[S] = True
    for i in range(n):
        p = softmax(z[i].astype(np.float64) / 0.7)
        assert abs(m[i] - p[S].sum()) < 1e-12
        order = np.lexsort((np.arange(V), -z[i]))      # (z desc, id asc)
        for t, k in enumerate(ks):
            assert r[i, t] == inS[order[:k]].sum() / k


def test_coverage_monotone_under_insertion():
    import oracle
    rng = np.random.default_rng(9)
    V = 500
    z = rng.normal(size=(3, V)).astype(np.float32)
    S = np.sort(rng.choice(V, 50, replace=False)).astype(np.int32)
    m0, r0 = oracle.coverage(z, S, [5, 20])
    S2 = np.union1d(S, rng.choice(V, 40, replace=False)).astype(np.int32)
    m1, r1 = oracle.coverage(z, S2, [5, 20])
    assert np.all(m1 >= m0) and np.all(r1 >= r0)


# ---------------------------------------------------------------- N3 KD objective
# Pins for oracle.kd_loss (eo_kd_loss): Eq. curriculum_weight and
# Eq. lora_objective against an independent scipy implementation
# (softmax, rel_entr), the KL's zero / positivity, the gradient by central
# finite differences of J (weights held fixed, reading K1), and the limits the
# paper names: beta = 0 (no curriculum, equal weights) and a confident first
# step (L_base -> 0: the horizon flattens).

def test_kd_matches_scipy():
    import oracle
    from scipy.special import log_softmax, rel_entr, softmax
    rng = np.random.default_rng(21)
    B, g, K, T, beta = 3, 6, 64, 1.7, 0.3
    zp = (rng.normal(size=(B, g, K)) * 2).astype(np.float32)
    zq = (rng.normal(size=(B, g, K)) * 2).astype(np.float32)
    v = rng.integers(0, K, size=B).astype(np.int32)
    J, _, w = oracle.kd_loss(zp, zq, v, T=T, beta=beta)
    for b in range(B):
        Lb = -log_softmax(zq[b, 0].astype(np.float64))[v[b]]
        wj = np.exp(-beta * Lb * np.arange(g))
        kl = [rel_entr(softmax(zp[b, j].astype(np.float64) / T), softmax(zq[b, j].astype(np.float64) / T)).sum()
              for j in range(g)]
        assert abs(J[b] - (wj * T * T * np.array(kl)).sum()) < 1e-12 * max(1.0, J[b])
        np.testing.assert_allclose(w[b], wj, rtol=1e-13)


def test_kd_zero_positive_and_gradient_fd():
    import oracle
    rng = np.random.default_rng(22)
    B, g, K, T = 2, 4, 16, 1.3
    zp = rng.normal(size=(B, g, K)).astype(np.float32)
    zq = rng.normal(size=(B, g, K)).astype(np.float32)
    v = np.array([2, 5], np.int32)
    J0, g0, w0 = oracle.kd_loss(zp, zp, v, T=T)
    assert np.all(J0 == 0.0) and np.all(g0 == 0.0)
    J, grad, w = oracle.kd_loss(zp, zq, v, T=T)
    assert np.all(J > 0.0)
    # central differences of J_b with the weights held at w (beta = 0 keeps them fixed)
    J, grad, _ = oracle.kd_loss(zp, zq, v, T=T, beta=0.0)
    h = 1e-2
    for (b, j, i) in [(0, 0, 3), (1, 2, 7), (1, 3, 15)]:
        zqp, zqm = zq.copy(), zq.copy()
        zqp[b, j, i] += h
        zqm[b, j, i] -= h
        fd = (oracle.kd_loss(zp, zqp, v, T=T, beta=0.0)[0][b] - oracle.kd_loss(zp, zqm, v, T=T, beta=0.0)[0][b]) / (2 * h)
        assert abs(fd - grad[b, j, i]) < 1e-4 * max(1.0, abs(fd))
    # the gradient of each step sums to zero (softmax shift invariance)
    assert np.abs(grad.sum(-1)).max() < 1e-12


def test_kd_curriculum_limits():
    import oracle
    rng = np.random.default_rng(23)
    B, g, K = 1, 6, 32
    zp = rng.normal(size=(B, g, K)).astype(np.float32)
    zq = rng.normal(size=(B, g, K)).astype(np.float32)
    _, _, w = oracle.kd_loss(zp, zq, [0], beta=0.0)
    assert np.all(w == 1.0)                         # beta = 0: no curriculum
    zq[0, 0, 0] = 60.0                              # the verified token dominates: L_base ~ 0
    _, _, w = oracle.kd_loss(zp, zq, [0], beta=0.3)
    assert np.all(w > 0.999999)                     # the horizon flattens
    zq[0, 0, 0] = -60.0                             # very unconfident: weights decay fast
    _, _, w = oracle.kd_loss(zp, zq, [0], beta=0.3)
    assert w[0, 0] == 1.0 and w[0, 1] < 1e-7


# ---------------------------------------------------------------- N1 ARC + update
# Pins for oracle.Arc (eo_arc_*): the SPEC worked examples, the
# invariants of S:295-299 / S:332-337 on random traces, and operation-for-
# operation equality with an independently written simulator (tests/brute.py
# ArcSim); oracle.subset_update against numpy set operations.

def test_arc_spec_examples():
    import oracle
    a = oracle.Arc(4, p0=0, min_res=0, warmup=0)
    assert a.admit([7], 0) == [] and a.state()["T1"] == [7]
    a = oracle.Arc(2, p0=0, min_res=0, warmup=0)                                  # S:319 (canonical p0 = 0)
    x, y, z = 10, 20, 30
    assert a.admit([x], 0) == [] and a.admit([y], 1) == []
    assert a.touch(x, 2)
    assert a.admit([z], 3) == [y]
    st = a.state()
    assert st["T1"] == [z] and st["T2"] == [x] and st["B1"] == [y]
    p_before = st["p"]                                                            # ghost re-admit
    assert a.admit([y], 4) != []
    st = a.state()
    assert y in st["T2"] and st["p"] > p_before
    b = oracle.Arc(8, min_res=0, warmup=0)
    b.admit([3, 9], 0)
    assert b.members() == [3, 9]
    assert not oracle.Arc(2).touch(5, 0)


@pytest.mark.parametrize("seed", range(4))
def test_arc_invariants_and_independent_simulator(seed):
    import oracle
    rng = np.random.default_rng(40 + seed)
    c, V = 16, 60
    kw = dict(p0=8, b1cap=10, b2cap=7, min_res=3 if seed % 2 else 0, warmup=5 if seed >= 2 else 0)
    a = oracle.Arc(c, **kw)
    sim = brute.ArcSim(c, kw["p0"], kw["b1cap"], kw["b2cap"], kw["min_res"], kw["warmup"])
    admitted_at = {}
    for step in range(300):
        if rng.random() < 0.5:
            t = int(rng.integers(V))
            assert a.touch(t, step) == sim.touch(t)
        else:
            toks = [int(t) for t in rng.choice(V, int(rng.integers(1, 6)), replace=False)]
            ev = a.admit(toks, step)
            assert ev == sim.admit(toks, step)
            for t in toks:
                admitted_at.setdefault(t, step)
            for t in ev:
                # min residency unless every resident was under-resident
                if step - admitted_at[t] < kw["min_res"]:
                    st = a.state()
                    assert all(step - admitted_at.get(u, step) < kw["min_res"] for u in st["T1"] + st["T2"])
                admitted_at.pop(t, None)
            for t in toks:
                admitted_at.setdefault(t, step)
        st = a.state()
        assert st == sim.state()
        res = st["T1"] + st["T2"]
        assert len(res) <= c and len(set(res)) == len(res)
        assert not (set(res) & set(st["B1"] + st["B2"]))
        assert len(st["B1"]) <= kw["b1cap"] and len(st["B2"]) <= kw["b2cap"]
        assert 0 <= st["p"] <= c


def test_arc_warmup_freezes_p():
    import oracle
    a = oracle.Arc(2, p0=1, min_res=0, warmup=100)
    for s, t in enumerate([1, 2, 3, 4, 1, 2, 3, 4, 1, 2]):
        a.admit([t], s)
    assert a.state()["p"] == 1


def test_subset_update_matches_set_ops():
    import oracle
    rng = np.random.default_rng(8)
    S = np.sort(rng.choice(10000, 3000, replace=False)).astype(np.int32)
    rem = np.sort(rng.choice(S, 40, replace=False)).astype(np.int32)
    add = np.sort(rng.choice(np.setdiff1d(np.arange(10000), S), 25, replace=False)).astype(np.int32)
    out = oracle.subset_update(S, rem, add)
    np.testing.assert_array_equal(out, np.union1d(np.setdiff1d(S, rem), add))
    with pytest.raises(ValueError):
        oracle.subset_update(S, [], S[:1])                                        # not disjoint
