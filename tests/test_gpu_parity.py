"""GPU parity: the CUDA path through the C ABI vs the oracle, element by element.

Bar (BASELINE.json north_star): subset ids and top-k ids bit-exact (ties to
the lower id); logits / LSE |d| <= 2e-3 (1 + |z|); probabilities |d| <= 1e-4.
Sizes span several CTA tiles and ragged tails; the full Llama-3 config
(V=128256, d=4096, n_S=36,864, n_h=60) runs in the launch configuration
bench.py times.
"""
import numpy as np
import pytest

import oracle
from tests import gpu_helpers as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_27390_b200 as es  # noqa: E402

DEV = "cuda:0"


def ctx_for(P, **kw):
    cfg = dict(V=P["V"], d=P["d"], w_dtype=G.torch_dtype(P["dtype"]), h_dtype=G.torch_dtype(P["dtype"]),
               max_subset=P["static"].size + P["n_dyn"], max_rows=max(P["n_h"], 1), max_k=64,
               max_sem=max(P["n_sem"], 1), max_seeds=64, debug_checks=True)
    cfg.update(kw)
    return es.Context(**cfg)


def run_path(P, ctx=None, inv_temp=1.0, logits=False):
    ctx = ctx or ctx_for(P)
    W = G.to_dev(P["W"], DEV)
    ctx.prepare_weights(W)
    ids, n, _, _ = ctx.build_subset(W, G.to_dev(P["q"], DEV), G.to_dev(P["static"], DEV),
                                    G.to_dev(P["seeds"], DEV), G.to_dev(P["row_ptr"], DEV),
                                    G.to_dev(P["col"], DEV), n_sem=P["n_sem"], n_dyn=P["n_dyn"],
                                    n_graph_sem_seeds=P["n_graph_sem_seeds"], per_seed=P["per_seed"])
    nmax = P["static"].size + P["n_dyn"]
    lo = torch.full((P["n_h"], max(nmax, 1)), float("nan"), device=DEV) if logits else None
    tri = ctx.subset_logits_topk(W, G.to_dev(P["H"], DEV), ids, n, nmax, P["k"], inv_temp, logits_out=lo)
    mrg = ctx.merge_shards(*tri, n_h=P["n_h"], k=P["k"])
    sem = ctx.last_semantic(P["n_sem"])
    torch.cuda.synchronize()
    nS = int(n.item())
    out = dict(S=ids[:nS].cpu().numpy(), sem=sem.cpu().numpy(),
               tri=[t.cpu().numpy() for t in tri], mrg=[t.cpu().numpy() for t in mrg],
               flags=ctx.get_flags())
    if logits:
        out["logits"] = lo[:, :nS].cpu().numpy()
    return out


def check(P, got, ref, k):
    np.testing.assert_array_equal(np.sort(got["sem"]), np.sort(ref["sem"]))
    np.testing.assert_array_equal(got["S"], ref["S"])
    G.assert_triple_close(*got["tri"], ref["triple"], k)
    oi, ov, ol, op = got["mrg"]
    np.testing.assert_array_equal(oi, ref["triple"]["ids"])
    fin = np.isfinite(ref["triple"]["lse"])
    assert np.all(np.abs(ol[fin] - ref["triple"]["lse"][fin]) <= G.LOGIT_TOL * (1 + np.abs(ref["triple"]["lse"][fin])))
    assert np.max(np.abs(op - ref["triple"]["probs"]), initial=0) <= G.PROB_TOL
    assert got["flags"] == 0, got["flags"]


TINY = dict(V=1024, d=64, n_static=128, n_sem=32, n_dyn=64, n_h=4, k=8, w_std=1.0, h_std=0.125)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_tiny(seed, dtype):
    P = G.make_problem(seed, dtype=dtype, **TINY)
    got = run_path(P, logits=True)
    ref = G.oracle_step(oracle, P)
    check(P, got, ref, P["k"])
    z = oracle.subset_logits(P["W"], P["H"], ref["S"])
    assert np.all(np.abs(got["logits"] - z) <= G.LOGIT_TOL * (1 + np.abs(z)))


@pytest.mark.parametrize("seed", range(3))
def test_integer_family_exact_ties(seed):
    """Integer data: every sum exact, many exact ties in scores and logits."""
    P = G.make_problem(seed, dtype="bf16", integer=True, V=3000, d=72 * 8, n_static=300, n_sem=200,
                       n_dyn=150, n_h=5, k=16)
    got = run_path(P, logits=True)
    ref = G.oracle_step(oracle, P)
    check(P, got, ref, P["k"])
    z = oracle.subset_logits(P["W"], P["H"], ref["S"])
    np.testing.assert_array_equal(got["logits"], z)   # exact


@pytest.mark.parametrize("n_h,k,inv_temp", [(1, 1, 1.0), (3, 10, 1.0), (4, 64, 1 / 0.7), (10, 10, 1.0)])
def test_medium_ragged(n_h, k, inv_temp):
    P = G.make_problem(11, dtype="bf16", V=20011, d=512, n_static=2999, n_sem=700, n_dyn=517,
                       n_h=n_h, k=k, avg_deg=16)
    got = run_path(P, inv_temp=inv_temp)
    ref = G.oracle_step(oracle, P, inv_temp=inv_temp)
    check(P, got, ref, k)


def test_duplicate_rows_tie_to_lower_id():
    P = G.make_problem(5, dtype="bf16", V=8192, d=256, n_static=1000, n_sem=400, n_dyn=300,
                       n_h=4, k=12, dup_rows=2000)
    got = run_path(P)
    ref = G.oracle_step(oracle, P)
    check(P, got, ref, P["k"])


@pytest.mark.parametrize("regime", ["tie_block", "sign_span", "narrow_span", "multipass"])
def test_union_selection_regimes(regime):
    """The union's three exact selections (S_sem, the budget of new candidates, the
    graph-seed prefix) in the regimes their key-linear binning treats differently:
    tie_block -- 3000 identical rows scoring near the top, so the S_sem and budget
    boundaries fall inside a block of > 1024 equal keys (ranked by id: the id-digit
    fallback); sign_span -- N_sem = 70% of V, candidates of both signs, so the key
    range spans the sign flip and the boundary bin is narrowed over several passes;
    narrow_span -- all scores within a few ulps of each other (one row plus ulp-level
    perturbations), so one bin covers single keys from the first pass; multipass --
    20,000 copies of the best row at V = 40,000: the candidate superset of the scan's
    histogram (>= 20,000 equal keys) exceeds the union's capacity (~16k), so the
    candidate kernel runs its further passes down to the id digits (grid barriers)."""
    if regime == "multipass":
        P = G.make_problem(64, dtype="fp32", V=40000, d=64, n_static=3000, n_sem=2000, n_dyn=1500, n_h=2, k=8,
                           w_std=1.0)
        sc = oracle.sem_scores(P["W"], P["q"])
        top = int(np.argmax(sc))
        rng = np.random.default_rng(5)
        dst = rng.choice(P["V"], 20000, replace=False)
        P["W"][dst] = P["W"][top]
    elif regime == "tie_block":
        P = G.make_problem(61, dtype="bf16", V=8192, d=256, n_static=1000, n_sem=1500, n_dyn=1200, n_h=2, k=8)
        sc = oracle.sem_scores(P["W"], P["q"])
        top = int(np.argsort(-sc)[20])
        rng = np.random.default_rng(3)
        dst = rng.choice(P["V"], 3000, replace=False)
        P["W"][dst] = P["W"][top]
    elif regime == "sign_span":
        P = G.make_problem(62, dtype="fp32", V=6000, d=64, n_static=500, n_sem=4200, n_dyn=3000, n_h=2, k=8,
                           w_std=1.0)
    else:
        P = G.make_problem(63, dtype="fp32", V=5000, d=64, n_static=300, n_sem=900, n_dyn=700, n_h=2, k=8,
                           w_std=1.0)
        base = P["W"][7].copy()
        rng = np.random.default_rng(4)
        P["W"][:] = base
        # ulp-level perturbations of 8 coordinates: thousands of distinct scores within
        # a relative range of ~1e-6
        for c in range(8):
            step = rng.integers(-1, 2, P["V"])
            up, dn = np.nextafter(base[c], np.float32(np.inf)), np.nextafter(base[c], np.float32(-np.inf))
            P["W"][:, c] = np.where(step > 0, up, np.where(step < 0, dn, base[c]))
    got = run_path(P)
    ref = G.oracle_step(oracle, P)
    if regime == "narrow_span":
        # the logits of rows equal up to ulps are closer than the LM head's tolerance, so
        # their top-k order is not fixed by the north star: the selections alone here
        np.testing.assert_array_equal(np.sort(got["sem"]), np.sort(ref["sem"]))
        np.testing.assert_array_equal(got["S"], ref["S"])
        assert got["flags"] & ~2 == 0   # (UNCERTIFIED: the head reports the unresolvable order)
    else:
        check(P, got, ref, P["k"])


def test_cap_not_reached_graph_and_seeds_fill():
    """Paper-default formation: N_sem = 10, graph top-8 per seed, cap binds inside S_graph."""
    P = G.make_problem(2, dtype="bf16", V=50000, d=256, n_static=5000, n_sem=10, n_dyn=100,
                       n_seed=10, per_seed=8, n_h=2, k=10, avg_deg=32)
    got = run_path(P)
    ref = G.oracle_step(oracle, P)
    check(P, got, ref, P["k"])


def test_empty_subset_and_k_gt_nS():
    P = G.make_problem(3, dtype="fp32", V=512, d=64, n_static=0, n_sem=3, n_dyn=3, n_seed=0,
                       n_graph_sem_seeds=0, n_h=2, k=8, w_std=1.0)
    got = run_path(P)
    ref = G.oracle_step(oracle, P)
    assert got["S"].size == 3
    check(P, got, ref, 8)
    assert (got["tri"][0][:, 3:] == -1).all()
    P0 = dict(P, n_sem=0, n_dyn=0)
    got0 = run_path(P0)
    assert got0["S"].size == 0
    assert np.all(got0["tri"][2] == -np.inf) and np.all(got0["tri"][3] == 0)
    assert np.all(got0["mrg"][0] == -1)


def test_vocab_shards_on_one_gpu():
    """T3: R interleaved W slices, one triple per shard, stacked merge == unsplit oracle."""
    P = G.make_problem(7, dtype="bf16", V=30000, d=256, n_static=3000, n_sem=600, n_dyn=400, n_h=6, k=10)
    ref = G.oracle_step(oracle, P)
    S = ref["S"]
    for R in (2, 3, 4):
        trips = []
        for r in range(R):
            Sr = S[S % R == r].astype(np.int32)
            Wr = np.ascontiguousarray(P["W"][r::R])
            ctx = ctx_for(P, n_shards=R, shard_rank=r)
            Wd = G.to_dev(Wr, DEV)
            ctx.prepare_weights(Wd)
            Sd = G.to_dev(Sr, DEV) if Sr.size else torch.zeros(1, dtype=torch.int32, device=DEV)
            nd = torch.tensor([Sr.size], dtype=torch.int32, device=DEV)
            trips.append(ctx.subset_logits_topk(Wd, G.to_dev(P["H"], DEV), Sd, nd, S.size, P["k"]))
            assert ctx.get_flags() == 0
        mctx = ctx_for(P, n_shards=R, shard_rank=0)
        st = [torch.stack([t[i] for t in trips]) for i in range(4)]
        oi, ov, ol, op = mctx.merge_shards(*st, n_h=P["n_h"], k=P["k"])
        torch.cuda.synchronize()
        np.testing.assert_array_equal(oi.cpu().numpy(), ref["triple"]["ids"])
        assert np.max(np.abs(op.cpu().numpy() - ref["triple"]["probs"])) <= G.PROB_TOL
        lse = ref["triple"]["lse"]
        assert np.all(np.abs(ol.cpu().numpy() - lse) <= G.LOGIT_TOL * (1 + np.abs(lse)))


def test_draft_step_host_io_equals_device_path():
    P = G.make_problem(9, dtype="bf16", V=16000, d=256, n_static=2000, n_sem=300, n_dyn=250, n_h=3, k=10)
    ctx = ctx_for(P)
    W = G.to_dev(P["W"], DEV)
    ctx.prepare_weights(W)
    kw = dict(E=W, W_local=W, static_ids=G.to_dev(P["static"], DEV), csr_row_ptr=G.to_dev(P["row_ptr"], DEV),
              csr_col=G.to_dev(P["col"], DEV), k=P["k"], n_sem=P["n_sem"], n_dyn=P["n_dyn"])
    H = G.to_dev(P["H"], "cpu").pin_memory()
    q = G.to_dev(P["q"], "cpu").pin_memory()
    seeds = torch.from_numpy(P["seeds"]).pin_memory()
    out_h = ctx.draft_step(q=q, H=H, seeds=seeds, **kw)
    torch.cuda.synchronize()
    out_d = ctx.draft_step(q=q.to(DEV), H=H.to(DEV), seeds=seeds.to(DEV), **kw)
    torch.cuda.synchronize()
    ref = G.oracle_step(oracle, P)
    for a, b in zip(out_h, out_d):
        np.testing.assert_array_equal(a.numpy(), b.cpu().numpy())
    np.testing.assert_array_equal(out_h[0].numpy(), ref["triple"]["ids"])
    assert np.max(np.abs(out_h[3].numpy() - ref["triple"]["probs"])) <= G.PROB_TOL


def test_prepared_draft_step_refilled_host_buffers():
    """Context.prepare_draft_step (the serving-loop call bench.py's e2e times): the
    caller refills the pinned host H / q in place between runs; every run equals the
    oracle for the current contents."""
    Ps = [G.make_problem(s, dtype="bf16", V=16000, d=256, n_static=2000, n_sem=300, n_dyn=250, n_h=3, k=10)
          for s in (9, 10)]
    P0 = Ps[0]
    ctx = ctx_for(P0)
    W = G.to_dev(P0["W"], DEV)
    ctx.prepare_weights(W)
    kw = dict(E=W, W_local=W, static_ids=G.to_dev(P0["static"], DEV), csr_row_ptr=G.to_dev(P0["row_ptr"], DEV),
              csr_col=G.to_dev(P0["col"], DEV), k=P0["k"], n_sem=P0["n_sem"], n_dyn=P0["n_dyn"])
    H = G.to_dev(P0["H"], "cpu").pin_memory()
    q = G.to_dev(P0["q"], "cpu").pin_memory()
    seeds = torch.from_numpy(P0["seeds"]).pin_memory()
    step = ctx.prepare_draft_step(q=q, H=H, seeds=seeds, **kw)
    for P in Ps + Ps[:1]:
        Q = dict(P0, H=P["H"], q=P["q"])       # same weights / graph / static set, new H and q
        H.copy_(G.to_dev(Q["H"], "cpu"))
        q.copy_(G.to_dev(Q["q"], "cpu"))
        out = step.run()
        torch.cuda.synchronize()
        ref = G.oracle_step(oracle, Q)
        np.testing.assert_array_equal(out[0].numpy(), ref["triple"]["ids"])
        assert np.max(np.abs(out[3].numpy() - ref["triple"]["probs"])) <= G.PROB_TOL


@pytest.mark.parametrize("dup", [0, 3000])
def test_draft_step_llama_full_size(dup):
    """Config L through evospec_draft_step (the bench's call; with EVOSPEC_OVERLAP the
    static / dynamic two-list LM head), against the oracle; dup > 0 duplicates W rows so
    that exact logit ties cross the static and dynamic lists (ties to the lower id)."""
    import synth
    c = dict(synth.CONFIGS["llama"])
    P = G.make_problem(1, dup_rows=dup, **c)
    ctx = ctx_for(P)
    W = G.to_dev(P["W"], DEV)
    ctx.prepare_weights(W)
    kw = dict(E=W, W_local=W, static_ids=G.to_dev(P["static"], DEV), csr_row_ptr=G.to_dev(P["row_ptr"], DEV),
              csr_col=G.to_dev(P["col"], DEV), k=P["k"], n_sem=P["n_sem"], n_dyn=P["n_dyn"])
    out = ctx.draft_step(q=G.to_dev(P["q"], DEV), H=G.to_dev(P["H"], DEV), seeds=G.to_dev(P["seeds"], DEV), **kw)
    torch.cuda.synchronize()
    ref = G.oracle_step(oracle, P)
    np.testing.assert_array_equal(out[0].cpu().numpy(), ref["triple"]["ids"])
    vals, lse = out[1].cpu().numpy().astype(np.float64), out[2].cpu().numpy().astype(np.float64)
    rv, rl = ref["triple"]["vals"], ref["triple"]["lse"]
    assert np.all(np.abs(vals - rv) <= G.LOGIT_TOL * (1 + np.abs(rv))), np.abs(vals - rv).max()
    assert np.all(np.abs(lse - rl) <= G.LOGIT_TOL * (1 + np.abs(rl))), np.abs(lse - rl).max()
    assert np.max(np.abs(out[3].cpu().numpy() - ref["triple"]["probs"])) <= G.PROB_TOL
    assert ctx.get_flags() == 0


@pytest.mark.parametrize("d", [4096, 8192])
def test_tc_error_envelope_at_bench_shapes(d):
    """The tcgen05 certification band (kTcGamma = 2^-16 of ||h|| max||W_v||, api.cu) at the
    bench's hidden sizes: the measured accumulation error of every logit of a 60-row tree
    against the exact fp64 value stays below 1/8 of the band (values drawn as in the
    bench: W ~ N(0, 0.02^2) bf16, H ~ N(0, 1) bf16)."""
    import synth
    V, n_h, n_S = 12000, 60, 6000
    W = synth.matrix(70 + d, V, d, 0.02, "bf16")
    H = synth.matrix(71 + d, n_h, d, 1.0, "bf16")
    S = np.sort(np.random.default_rng(d).choice(V, n_S, replace=False)).astype(np.int32)
    ctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=n_S, max_rows=n_h,
                     max_k=10, max_sem=1)
    Wd = G.to_dev(W, DEV)
    ctx.prepare_weights(Wd)
    lo = torch.full((n_h, n_S), float("nan"), device=DEV)
    nd = torch.tensor([n_S], dtype=torch.int32, device=DEV)
    ctx.subset_logits_topk(Wd, G.to_dev(H, DEV), G.to_dev(S, DEV), nd, n_S, 10, logits_out=lo)
    torch.cuda.synchronize()
    assert ctx.get_flags() == 0
    z = oracle.subset_logits(W, H, S)
    Wf = (W.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    Hf = (H.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    wmax = np.sqrt((Wf ** 2).sum(1)).max()
    hn = np.sqrt((Hf ** 2).sum(1))
    err = np.abs(lo.cpu().numpy().astype(np.float64) - z).max(1)
    assert np.all(err <= 2.0 ** -16 * hn * wmax / 8), (err / (hn * wmax)).max() * 2.0 ** 16


@pytest.mark.parametrize("n_h,k,n_dyn,dup,n_static", [(5, 1, 3000, 0, 40000), (17, 10, 3000, 400, 40000),
                                                        (60, 24, 5000, 0, 40000), (60, 10, 100, 0, 40000),
                                                        (60, 10, 12000, 0, 10000)])
def test_draft_step_two_list_shapes(n_h, k, n_dyn, dup, n_static):
    """draft_step's two-list LM head (static rows before the wait, dynamic rows after;
    DESIGN §5.0) across tree widths, k and dynamic-list sizes (whole and partial
    second-list tiles), with cross-list exact ties (dup), against the oracle."""
    P = G.make_problem(40 + n_h, dtype="bf16", V=60000, d=256, n_static=n_static, n_sem=max(6000, n_dyn),
                       n_dyn=n_dyn, n_h=n_h, k=k, dup_rows=dup)   # (~12k dynamic rows: most CTAs hold one)
    ctx = ctx_for(P)
    W = G.to_dev(P["W"], DEV)
    ctx.prepare_weights(W)
    kw = dict(E=W, W_local=W, static_ids=G.to_dev(P["static"], DEV), csr_row_ptr=G.to_dev(P["row_ptr"], DEV),
              csr_col=G.to_dev(P["col"], DEV), k=P["k"], n_sem=P["n_sem"], n_dyn=P["n_dyn"])
    out = ctx.draft_step(q=G.to_dev(P["q"], DEV), H=G.to_dev(P["H"], DEV), seeds=G.to_dev(P["seeds"], DEV), **kw)
    torch.cuda.synchronize()
    ref = G.oracle_step(oracle, P)
    np.testing.assert_array_equal(out[0].cpu().numpy(), ref["triple"]["ids"])
    np.testing.assert_allclose(out[2].cpu().numpy(), ref["triple"]["lse"], rtol=2e-3, atol=2e-3)
    assert np.max(np.abs(out[3].cpu().numpy() - ref["triple"]["probs"])) <= G.PROB_TOL
    assert ctx.get_flags() == 0


@pytest.mark.parametrize("seed,n_h,k,n_dyn", [(0, 10, 10, 2500), (1, 60, 24, 2500), (2, 3, 1, 2500),
                                               (3, 60, 10, 600), (4, 17, 24, 800)])
def test_draft_step_two_list_integer_ties(seed, n_h, k, n_dyn):
    """The two-list LM head on integer data ({-3..3}: every logit an exact integer, massive
    ties inside and across the static and dynamic lists, whose subset positions do not
    follow id order): the candidate buffers order ties by vocabulary id (DESIGN §5.3,
    keys), so the top-k ids equal the oracle's lower-id-first order. n_dyn = 2500 (~1000
    new semantic members: the graph walk adds the rest, the head waits for the union's
    end); n_dyn <= 800: the semantic part fills the budget and the head takes the union's
    early, unsorted copy of the dynamic list."""
    P = G.make_problem(70 + seed, dtype="bf16", integer=True, V=30000, d=128, n_static=20000, n_sem=3000,
                       n_dyn=n_dyn, n_h=n_h, k=k)
    ctx = ctx_for(P)
    W = G.to_dev(P["W"], DEV)
    ctx.prepare_weights(W)
    kw = dict(E=W, W_local=W, static_ids=G.to_dev(P["static"], DEV), csr_row_ptr=G.to_dev(P["row_ptr"], DEV),
              csr_col=G.to_dev(P["col"], DEV), k=P["k"], n_sem=P["n_sem"], n_dyn=P["n_dyn"])
    out = ctx.draft_step(q=G.to_dev(P["q"], DEV), H=G.to_dev(P["H"], DEV), seeds=G.to_dev(P["seeds"], DEV), **kw)
    torch.cuda.synchronize()
    ref = G.oracle_step(oracle, P)
    np.testing.assert_array_equal(out[0].cpu().numpy(), ref["triple"]["ids"])
    np.testing.assert_allclose(out[1].cpu().numpy(), ref["triple"]["vals"], rtol=0, atol=1e-6)
    assert ctx.get_flags() == 0


def test_input_errors():
    P = G.make_problem(0, dtype="fp32", **TINY)
    ctx = ctx_for(P)
    W = G.to_dev(P["W"], DEV)
    H = G.to_dev(P["H"], DEV)
    S = torch.arange(10, dtype=torch.int32, device=DEV)
    n = torch.tensor([10], dtype=torch.int32, device=DEV)
    for kw in [dict(k=0), dict(k=65), dict(inv_temp=0.0), dict(inv_temp=float("inf"))]:
        args = dict(k=4, inv_temp=1.0)
        args.update(kw)
        with pytest.raises(es.EvospecError) as ei:
            ctx.subset_logits_topk(W, H, S, n, 10, args["k"], args["inv_temp"])
        assert ei.value.status == es.EINPUT


def test_invariant_fault_fixture_returns_einvariant():
    """Product-path fault fixture (SPEC S:621-628 mirrored): with
    debug_checks, an unsorted subset and an out-of-range id make the LM-head call
    return EVOSPEC_EINVARIANT; without debug_checks, evospec_sync_status reports the
    same verdict for an invariant flag, and a clean context reports OK."""
    P = G.make_problem(0, dtype="bf16", **TINY)
    W = G.to_dev(P["W"], DEV)
    H = G.to_dev(P["H"], DEV)
    n = torch.tensor([10], dtype=torch.int32, device=DEV)
    bad_sets = [torch.tensor([0, 5, 3, 7, 9, 11, 13, 20, 30, 40], dtype=torch.int32, device=DEV),   # unsorted
                torch.tensor([0, 1, 2, 3, 4, 5, 6, 7, 8, P["V"] + 5], dtype=torch.int32, device=DEV)]  # id >= V
    for S in bad_sets:
        ctx = ctx_for(P)   # debug_checks=True
        ctx.prepare_weights(W)
        with pytest.raises(es.EvospecError) as ei:
            ctx.subset_logits_topk(W, H, S, n, 10, 4)
        assert ei.value.status == es.EINVARIANT
        assert ctx.get_flags() & es.FLAG_BAD_IDS
    ctx = ctx_for(P, debug_checks=False)
    ctx.prepare_weights(W)
    ctx.subset_logits_topk(W, H, torch.arange(10, dtype=torch.int32, device=DEV), n, 10, 4)
    ctx.sync_status()   # clean: no exception
    flags = torch.zeros(1, dtype=torch.int32, device=DEV)
    es.subset_update(torch.arange(10, dtype=torch.int32, device=DEV), torch.tensor([50], dtype=torch.int32, device=DEV),
                     torch.tensor([], dtype=torch.int32, device=DEV), flags=flags)   # removed id not in the set
    torch.cuda.synchronize()
    assert int(flags.item()) & es.FLAG_BAD_IDS


@pytest.mark.slow
def test_llama_full_size():
    """Config L at full size: V=128256, d=4096, static 32768 + 4096 retrieved, n_h=60, k=10."""
    import synth
    c = dict(synth.CONFIGS["llama"])
    P = G.make_problem(0, **c)
    got = run_path(P)
    ref = G.oracle_step(oracle, P)
    assert got["S"].size == 36864
    # C10: the selections' boundaries are not near-ties in fp64 (so "bit-exact" is
    # tested on boundaries the GPU must resolve, not ones it could order either way)
    s = oracle.sem_scores(P["W"], P["q"])
    assert G.near_tie_count(s, c["n_sem"]) == 0
    z = oracle.subset_logits(P["W"], P["H"], ref["S"])
    assert G.near_tie_count(z, c["k"]) == 0
    check(P, got, ref, c["k"])


@pytest.fixture
def lmh_path(monkeypatch):
    def set_path(p):
        monkeypatch.setenv("EVOSPEC_LMH", p)
    return set_path


@pytest.mark.parametrize("path", ["tc", "gemv"])
@pytest.mark.parametrize("n_h,k", [(5, 10), (16, 1), (60, 10), (60, 24), (60, 25), (128, 64)])
def test_lmh_paths(lmh_path, path, n_h, k):
    """Both LM-head kernels (tcgen05 and FFMA) against the oracle, same inputs."""
    lmh_path(path)
    P = G.make_problem(21, dtype="bf16", V=40000, d=1024, n_static=5000, n_sem=900, n_dyn=777,
                       n_h=n_h, k=k, avg_deg=16)
    got = run_path(P, logits=True)
    ref = G.oracle_step(oracle, P)
    check(P, got, ref, k)
    z = oracle.subset_logits(P["W"], P["H"], ref["S"])
    # accumulation error stays well inside the certification envelope (1/8 of delta)
    gamma = 2.0 ** -16 if path == "tc" else 1.01 * (1024 / 32 + 6) * 2.0 ** -24
    W64 = P["W"].astype(np.uint32) << 16
    wmax = np.sqrt((W64.view(np.float32).astype(np.float64) ** 2).sum(1)).max()
    hn = np.sqrt((((P["H"].astype(np.uint32) << 16).view(np.float32).astype(np.float64)) ** 2).sum(1))
    err = np.abs(got["logits"] - z).max(1)
    assert np.all(err <= gamma * hn * wmax / 8), (err / (hn * wmax)).max()


@pytest.mark.parametrize("k,integer", [(1, False), (10, False), (24, False), (10, True)])
def test_tc_multitile_thread_parallel_fold(lmh_path, k, integer):
    """Subsets longer than two 128-row tiles per CTA (n_S > 2 * 128 * 148): the tensor-core
    kernel's thread-parallel fold for every bound width (J = 3 / 5 / 8 for k + 8 <= 12 / 20 /
    32), and with integer inputs (massive exact ties) its overflow fallback to the warp fold."""
    lmh_path("tc")
    P = G.make_problem(31, dtype="bf16", integer=integer, V=60000, d=256, n_static=40000, n_sem=6000,
                       n_dyn=5000, n_h=8, k=k)
    got = run_path(P)
    ref = G.oracle_step(oracle, P)
    assert got["S"].size > 2 * 128 * 148
    check(P, got, ref, k)


def test_tc_integer_exact(lmh_path):
    """Integer inputs: tcgen05 fp32 accumulation is exact (sums < 2^24)."""
    lmh_path("tc")
    P = G.make_problem(4, dtype="bf16", integer=True, V=6000, d=512, n_static=700, n_sem=300,
                       n_dyn=260, n_h=37, k=12)
    got = run_path(P, logits=True)
    ref = G.oracle_step(oracle, P)
    check(P, got, ref, P["k"])
    np.testing.assert_array_equal(got["logits"], oracle.subset_logits(P["W"], P["H"], ref["S"]))


def test_ctx_count_source():
    """Reading C5: context-count source (count >= min, (count desc, id asc), first n_ctx_max)."""
    import synth
    P = G.make_problem(13, dtype="bf16", V=30000, d=256, n_static=3000, n_sem=40, n_dyn=120, n_h=3, k=10)
    ctx_ids = synth.ctx_tokens(14, P["V"], 900)
    ctx = ctx_for(P, max_ctx=1024)
    W = G.to_dev(P["W"], DEV)
    ctx.prepare_weights(W)
    ids, n, _, _ = ctx.build_subset(W, G.to_dev(P["q"], DEV), G.to_dev(P["static"], DEV),
                                    G.to_dev(P["seeds"], DEV), G.to_dev(P["row_ptr"], DEV),
                                    G.to_dev(P["col"], DEV), n_sem=P["n_sem"], n_dyn=P["n_dyn"],
                                    n_graph_sem_seeds=2, per_seed=1,
                                    ctx_ids=G.to_dev(ctx_ids, DEV), ctx_min_count=2, n_ctx_max=64)
    torch.cuda.synchronize()
    ref = oracle.build_subset(P["W"], P["q"], P["static"], P["seeds"], P["row_ptr"], P["col"],
                              n_sem=P["n_sem"], n_dyn=P["n_dyn"], n_graph_sem_seeds=2, per_seed=1,
                              ctx_ids=ctx_ids, ctx_min_count=2, n_ctx_max=64)
    np.testing.assert_array_equal(ids[:int(n.item())].cpu().numpy(), ref["S"])
    # the ctx source contributed (cap not reached by seeds + sem + graph alone)
    ref0 = oracle.build_subset(P["W"], P["q"], P["static"], P["seeds"], P["row_ptr"], P["col"],
                               n_sem=P["n_sem"], n_dyn=P["n_dyn"], n_graph_sem_seeds=2, per_seed=1)
    assert ref["S"].size > ref0["S"].size
    assert ctx.get_flags() == 0


@pytest.mark.slow
def test_qwen_full_size():
    """Config Q (Qwen2.5-7B head): V=152064, d=3584, static 32768 + 4096, n_h=60."""
    import synth
    c = dict(synth.CONFIGS["qwen"])
    P = G.make_problem(1, **c)
    got = run_path(P)
    ref = G.oracle_step(oracle, P)
    assert got["S"].size == 32768 + 4096
    check(P, got, ref, c["k"])


# ------------------------------------------------ batched serving (config Bt)
def _ragged_problem(seed, *, V, d, n_static, n_rows_per_seq, dyn_sizes, k, dtype="bf16"):
    rng = np.random.default_rng(seed)
    W = synth_matrix(seed, V, d, 0.02, dtype)
    h_off = np.concatenate([[0], np.cumsum(n_rows_per_seq)]).astype(np.int64)
    H = synth_matrix(seed + 1, int(h_off[-1]), d, 1.0, dtype)
    perm = rng.permutation(V)
    static = np.sort(perm[:n_static]).astype(np.int32)
    pool = perm[n_static:]
    dyn_lists = [np.sort(rng.choice(pool, n, replace=False)).astype(np.int32) for n in dyn_sizes]
    dyn = np.concatenate(dyn_lists).astype(np.int32) if dyn_lists else np.zeros(0, np.int32)
    d_off = np.concatenate([[0], np.cumsum([x.size for x in dyn_lists])]).astype(np.int64)
    return dict(W=W, H=H, h_off=h_off, static=static, dyn=dyn, d_off=d_off, k=k, V=V, d=d, dtype=dtype)


def synth_matrix(seed, rows, d, std, dtype):
    import synth
    return synth.matrix(seed, rows, d, std, dtype)


def _run_ragged(R, max_rows=None):
    ctx = es.Context(V=R["V"], d=R["d"], w_dtype=G.torch_dtype(R["dtype"]), h_dtype=G.torch_dtype(R["dtype"]),
                     max_subset=max(R["static"].size, int(np.diff(R["d_off"]).max(initial=0)), 1),
                     max_rows=max_rows or int(R["h_off"][-1]), max_k=64, max_sem=1, max_seeds=16, debug_checks=True)
    W = G.to_dev(R["W"], DEV)
    ctx.prepare_weights(W)
    dyn = G.to_dev(R["dyn"], DEV) if R["dyn"].size else torch.zeros(1, dtype=torch.int32, device=DEV)
    max_dyn = int(np.diff(R["d_off"]).max(initial=0))
    out = ctx.subset_logits_topk_ragged(W, G.to_dev(R["H"], DEV), R["h_off"].tolist(), G.to_dev(R["static"], DEV),
                                        dyn, G.to_dev(R["d_off"].astype(np.int32), DEV), max_dyn, R["k"])
    torch.cuda.synchronize()
    assert ctx.get_flags() == 0
    return [t.cpu().numpy() for t in out]


@pytest.mark.parametrize("case", ["mixed", "many_rows"])
def test_ragged_lmh(case):
    """Per-sequence V_b = static u dyn_b: row groups on the tensor-core path (n_b >= 5)
    and on the FFMA path (n_b < 5), an empty dyn_b, a sequence without rows, and
    (many_rows) more than 128 rows so the static block runs in several row groups."""
    if case == "mixed":
        R = _ragged_problem(60, V=20000, d=256, n_static=2500, n_rows_per_seq=[10, 1, 0, 6, 3, 12],
                            dyn_sizes=[300, 17, 40, 0, 900, 256], k=10)
    else:
        R = _ragged_problem(61, V=12000, d=128, n_static=1000, n_rows_per_seq=[40, 60, 50, 7],
                            dyn_sizes=[100, 0, 500, 33], k=8)
    ids, vals, m, s = _run_ragged(R)
    ref = oracle.subset_logits_topk_ragged(R["W"], R["H"], R["h_off"], R["static"], R["dyn"], R["d_off"], R["k"])
    G.assert_triple_close(ids, vals, m, s, ref, R["k"])


def test_batched_build_then_ragged():
    """Batched build (per-sequence seeds, shared static) feeds the ragged LM head
    through device offsets; both stages equal the oracle."""
    P = G.make_problem(62, dtype="bf16", V=9000, d=128, n_static=900, n_sem=120, n_dyn=80, n_h=1, k=8)
    B = 5
    Q = synth_matrix(63, B, P["d"], 1.0, "bf16")
    rng = np.random.default_rng(64)
    n_seed = [0, 3, 10, 1, 6]
    s_off = np.concatenate([[0], np.cumsum(n_seed)]).astype(np.int64)
    seeds = rng.choice(P["V"], int(s_off[-1]), replace=True).astype(np.int32)
    ctx = es.Context(V=P["V"], d=P["d"], w_dtype=torch.bfloat16, h_dtype=torch.bfloat16,
                     max_subset=P["static"].size + P["n_dyn"], max_rows=40, max_k=64, max_sem=P["n_sem"],
                     max_seeds=64, debug_checks=True)
    W = G.to_dev(P["W"], DEV)
    ctx.prepare_weights(W)
    dyn, d_off = ctx.build_subset_batched(W, G.to_dev(Q, DEV), G.to_dev(P["static"], DEV), G.to_dev(seeds, DEV),
                                          s_off.tolist(), G.to_dev(P["row_ptr"], DEV), G.to_dev(P["col"], DEV),
                                          n_sem=P["n_sem"], n_dyn=P["n_dyn"], n_graph_sem_seeds=5, per_seed=4)
    ref_dyn, ref_off = oracle.build_subset_batched(P["W"], Q, P["static"], seeds, s_off, P["row_ptr"], P["col"],
                                                   n_sem=P["n_sem"], n_dyn=P["n_dyn"], n_graph_sem_seeds=5,
                                                   per_seed=4)
    torch.cuda.synchronize()
    got_off = d_off.cpu().numpy()
    np.testing.assert_array_equal(got_off, ref_off)
    np.testing.assert_array_equal(dyn[:int(got_off[-1])].cpu().numpy(), ref_dyn)
    assert ctx.get_flags() == 0
    rows = [8, 2, 5, 0, 9]
    h_off = np.concatenate([[0], np.cumsum(rows)]).astype(np.int64)
    H = synth_matrix(65, int(h_off[-1]), P["d"], 1.0, "bf16")
    out = ctx.subset_logits_topk_ragged(W, G.to_dev(H, DEV), h_off.tolist(), G.to_dev(P["static"], DEV), dyn, d_off,
                                        P["n_dyn"], 8)
    torch.cuda.synchronize()
    ref = oracle.subset_logits_topk_ragged(P["W"], H, h_off, P["static"], ref_dyn, ref_off, 8)
    G.assert_triple_close(*[t.cpu().numpy() for t in out], ref, 8)
    assert ctx.get_flags() == 0


@pytest.mark.slow
def test_batched_full_size_sampled():
    """Config Bt at full size (V=128256, d=4096, 64 sequences x 10 rows, static 32768,
    dyn_b ~ U[256, 4096]) in the launch configuration bench.py times; the oracle
    checks three sampled sequences (first, middle, last) element by element."""
    n_seq, n_b = 64, 10
    sizes = np.random.default_rng(66).integers(256, 4097, n_seq)
    R = _ragged_problem(66, V=128256, d=4096, n_static=32768, n_rows_per_seq=[n_b] * n_seq,
                        dyn_sizes=sizes.tolist(), k=10)
    ids, vals, m, s = _run_ragged(R)
    for b in (0, 31, 63):
        h0, h1 = int(R["h_off"][b]), int(R["h_off"][b + 1])
        S_b = np.union1d(R["static"], R["dyn"][R["d_off"][b]:R["d_off"][b + 1]]).astype(np.int32)
        ref = oracle.subset_logits_topk(R["W"], R["H"][h0:h1], S_b, R["k"])
        G.assert_triple_close(ids[h0:h1], vals[h0:h1], m[h0:h1], s[h0:h1], ref, R["k"])


def test_merged_single_shard_equals_oracle():
    """evospec_subset_logits_topk_merged (R = 1: merge fused into the finalisation)
    returns merge_shards' outputs: ids exact, LSE and probabilities within tolerance."""
    P = G.make_problem(70, dtype="bf16", V=30000, d=256, n_static=3000, n_sem=500, n_dyn=700, n_h=12, k=10)
    ref = G.oracle_step(oracle, P)
    S = ref["S"]
    ctx = ctx_for(P)
    W = G.to_dev(P["W"], DEV)
    ctx.prepare_weights(W)
    Sd = G.to_dev(S, DEV)
    nd = torch.tensor([S.size], dtype=torch.int32, device=DEV)
    ids, vals, lse, probs = ctx.subset_logits_topk_merged(W, G.to_dev(P["H"], DEV), Sd, nd, S.size, P["k"])
    torch.cuda.synchronize()
    t = ref["triple"]
    np.testing.assert_array_equal(ids.cpu().numpy(), t["ids"])
    assert np.all(np.abs(lse.cpu().numpy() - t["lse"]) <= G.LOGIT_TOL * (1 + np.abs(t["lse"])))
    assert np.max(np.abs(probs.cpu().numpy() - t["probs"])) <= G.PROB_TOL
    assert np.all(np.abs(vals.cpu().numpy() - t["vals"]) <= G.LOGIT_TOL * (1 + np.abs(t["vals"])))
    assert ctx.get_flags() == 0


def test_draft_step_graph_replay_matches_direct():
    """evospec_draft_step replays a captured CUDA graph while the I/O descriptor is
    unchanged; its results equal the direct path's and the oracle's, also after the
    inputs behind the same pointers change."""
    import os
    P = G.make_problem(71, dtype="bf16", V=16000, d=256, n_static=2000, n_sem=300, n_dyn=250, n_h=8, k=10)
    ctx = ctx_for(P, debug_checks=False)
    W = G.to_dev(P["W"], DEV)
    ctx.prepare_weights(W)
    kw = dict(E=W, W_local=W, static_ids=G.to_dev(P["static"], DEV), csr_row_ptr=G.to_dev(P["row_ptr"], DEV),
              csr_col=G.to_dev(P["col"], DEV), k=P["k"], n_sem=P["n_sem"], n_dyn=P["n_dyn"])
    H = G.to_dev(P["H"], DEV)
    q = G.to_dev(P["q"], DEV)
    seeds = G.to_dev(P["seeds"], DEV)
    n_h, k = P["n_h"], P["k"]
    out = (torch.empty((n_h, k), dtype=torch.int32, device=DEV), torch.empty((n_h, k), device=DEV),
           torch.empty(n_h, device=DEV), torch.empty((n_h, k), device=DEV))
    l0 = ctx.read_stats()["launches"]
    outs = []
    for _ in range(3):                                   # capture, replay, replay
        o = ctx.draft_step(q=q, H=H, seeds=seeds, out=out, **kw)
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy().copy() for t in o])
    per_step = (ctx.read_stats()["launches"] - l0) / 3
    assert per_step >= 4                                 # replays still count the graph's kernels
    ref = G.oracle_step(oracle, P)
    for o in outs:
        np.testing.assert_array_equal(o[0], ref["triple"]["ids"])
        assert np.max(np.abs(o[3] - ref["triple"]["probs"])) <= G.PROB_TOL
    # new data behind the same pointers: the replay must see it
    P2 = dict(P)
    P2["H"] = synth_matrix(72, P["n_h"], P["d"], 1.0, "bf16")
    H.copy_(G.to_dev(P2["H"], DEV))
    o = ctx.draft_step(q=q, H=H, seeds=seeds, out=out, **kw)
    torch.cuda.synchronize()
    ref2 = G.oracle_step(oracle, P2)
    np.testing.assert_array_equal(o[0].cpu().numpy(), ref2["triple"]["ids"])
    assert ctx.get_flags() == 0


@pytest.mark.parametrize("V,d,n_dyn", [(12345, 192, 0), (12345, 192, 77), (4099, 320, 500)])
def test_odd_shapes_static_only_and_ragged_vocab(V, d, n_dyn):
    """V not a multiple of 32, d not a multiple of 256 (the LDG scan variant; d = 192 / 320
    still on the tensor-core head), a static-only subset (N_dyn = 0), and a dynamic budget
    larger than the non-static pool can fill."""
    P = G.make_problem(80 + n_dyn, dtype="bf16", V=V, d=d, n_static=1500, n_sem=200, n_dyn=n_dyn, n_h=7, k=10)
    got = run_path(P)
    ref = G.oracle_step(oracle, P)
    check(P, got, ref, P["k"])


@pytest.mark.parametrize("case", [
    dict(seed=90, integer=False, V=20000, d=256, n_static=2000, n_sem=300, n_dyn=500, n_h=20, k=10),
    dict(seed=91, integer=True, V=3000, d=576, n_static=300, n_sem=200, n_dyn=150, n_h=5, k=16),
    dict(seed=92, integer=True, V=60000, d=128, n_static=50000, n_sem=300, n_dyn=500, n_h=60, k=24),
    dict(seed=93, integer=False, V=90000, d=192, n_static=80000, n_sem=300, n_dyn=900, n_h=33, k=1)])
def test_tc_head_ties_tiles_and_lists(case):
    """The tensor-core head + the lean finalisation (fin64.cuh) on integer data with
    massive exact ties (candidate buffers overflowing, more than 1024 entries at the
    threshold: the finalisation's tie merge), several tiles per CTA, k = 1 and k = 24,
    called twice on one context (stale partials must not leak into the second call)."""
    c = dict(case)
    seed = c.pop("seed")
    integer = c.pop("integer")
    P = G.make_problem(seed, dtype="bf16", integer=integer, **c)
    ref = G.oracle_step(oracle, P)
    S = ref["S"]
    ctx = es.Context(V=P["V"], d=P["d"], w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=S.size,
                     max_rows=P["n_h"], max_k=32, max_sem=P["n_sem"])
    W = G.to_dev(P["W"])
    ctx.prepare_weights(W)
    nd = torch.tensor([S.size], dtype=torch.int32, device="cuda")
    for _ in range(2):
        ids, vals, m, s = ctx.subset_logits_topk(W, G.to_dev(P["H"]), G.to_dev(S), nd, S.size, P["k"])
        torch.cuda.synchronize()
        G.assert_triple_close(ids.cpu().numpy(), vals.cpu().numpy(), m.cpu().numpy(), s.cpu().numpy(),
                              ref["triple"], P["k"])
    assert ctx.get_flags() == 0


@pytest.mark.slow
def test_sharded_d8192_full_vocab_sampled():
    """Config Sh (d = 8192, V = 128256) at the full vocabulary in the launch configuration
    the bench times: R = 1 (merged call) and R = 2 interleaved shards on one GPU merged
    with merge_shards. The oracle checks 3 sampled rows of the 60 (63 G MAC for all)."""
    V, d, n_h, k = 128256, 8192, 60, 10
    W = synth_matrix(40, V, d, 0.02, "bf16")
    H = synth_matrix(41, n_h, d, 1.0, "bf16")
    S = np.arange(V, dtype=np.int32)
    rows = [0, 29, 59]
    ref = oracle.subset_logits_topk(W, H[rows], S, k)
    Wd, Hd = G.to_dev(W, DEV), G.to_dev(H, DEV)
    ctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=V, max_rows=n_h,
                     max_k=k, max_sem=1, max_seeds=1)
    ctx.prepare_weights(Wd)
    nd = torch.tensor([V], dtype=torch.int32, device=DEV)
    ids, vals, lse, probs = ctx.subset_logits_topk_merged(Wd, Hd, G.to_dev(S, DEV), nd, V, k)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ids.cpu().numpy()[rows], ref["ids"])
    assert np.all(np.abs(lse.cpu().numpy()[rows] - ref["lse"]) <= G.LOGIT_TOL * (1 + np.abs(ref["lse"])))
    assert np.max(np.abs(probs.cpu().numpy()[rows] - ref["probs"])) <= G.PROB_TOL
    del Wd
    trips = []
    for r in range(2):
        Wr = G.to_dev(np.ascontiguousarray(W[r::2]), DEV)
        cr = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, n_shards=2, shard_rank=r,
                        max_subset=V, max_rows=n_h, max_k=k, max_sem=1, max_seeds=1)
        cr.prepare_weights(Wr)
        Sr = S[S % 2 == r]
        ndr = torch.tensor([Sr.size], dtype=torch.int32, device=DEV)
        trips.append(cr.subset_logits_topk(Wr, Hd, G.to_dev(Sr, DEV), ndr, Sr.size, k))
        torch.cuda.synchronize()
        assert cr.get_flags() == 0
        del Wr
    mctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, n_shards=2, shard_rank=0,
                      max_subset=V, max_rows=n_h, max_k=k, max_sem=1, max_seeds=1)
    st = [torch.stack([t[i] for t in trips]) for i in range(4)]
    oi, ov, ol, op = mctx.merge_shards(*st, n_h=n_h, k=k)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(oi.cpu().numpy()[rows], ref["ids"])
    assert np.max(np.abs(op.cpu().numpy()[rows] - ref["probs"])) <= G.PROB_TOL


def test_draft_step_two_list_several_second_list_tiles():
    """The two-list head with 16-row second-list tiles (EVOSPEC_DYN_TILE=16, read once per
    process: run in a subprocess) -- several second-list tiles per CTA -- against the oracle."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, torch, oracle\n"
        "from tests import gpu_helpers as G\n"
        "import paper_2605_27390_b200 as es\n"
        "P = G.make_problem(77, dtype='bf16', V=60000, d=256, n_static=30000, n_sem=6000, n_dyn=5000, n_h=60, k=10)\n"
        "ctx = es.Context(V=P['V'], d=P['d'], w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=35000,\n"
        "                 max_rows=60, max_k=10, max_sem=6000)\n"
        "W = G.to_dev(P['W'], 'cuda:0'); ctx.prepare_weights(W)\n"
        "kw = dict(E=W, W_local=W, static_ids=G.to_dev(P['static'], 'cuda:0'), csr_row_ptr=G.to_dev(P['row_ptr'], 'cuda:0'),\n"
        "          csr_col=G.to_dev(P['col'], 'cuda:0'), k=10, n_sem=6000, n_dyn=5000)\n"
        "out = ctx.draft_step(q=G.to_dev(P['q'], 'cuda:0'), H=G.to_dev(P['H'], 'cuda:0'), seeds=G.to_dev(P['seeds'], 'cuda:0'), **kw)\n"
        "torch.cuda.synchronize()\n"
        "ref = G.oracle_step(oracle, P)\n"
        "assert np.array_equal(out[0].cpu().numpy(), ref['triple']['ids'])\n"
        "assert np.max(np.abs(out[3].cpu().numpy() - ref['triple']['probs'])) <= G.PROB_TOL\n"
        "assert ctx.get_flags() == 0\n"
        "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, EVOSPEC_DYN_TILE="16", EVOSPEC_OVERLAP="1")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr
