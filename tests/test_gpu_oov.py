"""N1 end to end on the GPU: a sequence of OOV events through
evospec_oov_event_begin / _end -- the event's candidate formation on the side
stream (exact semantic top-10 of the target-side hidden state, graph top-8 of
target top-10 u semantic top-10, the first 32 new non-static ids: P:458),
LM-head calls on the current subset while it runs, then the ARC admission
(capacity 256, p0 128, ghosts 256 / 256, min residency 8, warm-up 50: P:433-437)
and the incremental device update -- against the oracle pipeline event by event:
oracle.build_subset with the same parameters (its dynamic part = the candidates),
the oracle ARC, oracle.subset_update. The subset after every event is bit-exact and
equals sorted(static u ARC members); the LM head on it matches the oracle."""
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


def test_oov_event_sequence_matches_oracle_pipeline():
    import synth
    V, d, n_static = 20011, 256, 3000
    P = G.make_problem(81, dtype="bf16", V=V, d=d, n_static=n_static, n_sem=10, n_dyn=32, n_h=6, k=10,
                       avg_deg=16)
    W = G.to_dev(P["W"], DEV)
    static = np.sort(P["static"]).astype(np.int32)
    rp, col = G.to_dev(P["row_ptr"], DEV), G.to_dev(P["col"], DEV)
    ctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=n_static + 256 + 32,
                     max_rows=6, max_k=16, max_sem=16, max_seeds=64)
    ctx.prepare_weights(W)
    arc = es.Arc(256)
    oarc = oracle.Arc(256)
    S = torch.from_numpy(static).to(DEV)
    n = static.size
    H = G.to_dev(P["H"], DEV)
    rng = np.random.default_rng(5)
    for ev in range(24):
        q = synth.matrix(500 + ev, 1, d, 1.0, "bf16")[0]
        seeds = np.sort(rng.choice(V, 10, replace=False)).astype(np.int32)
        step = 8 * ev
        ctx.oov_event_begin(W, G.to_dev(q, DEV), G.to_dev(static, DEV), G.to_dev(seeds, DEV), rp, col, n_sem=10,
                            n_dyn=32, n_graph_sem_seeds=10, per_seed=8)
        nd = torch.tensor([n], dtype=torch.int32, device=DEV)
        for _ in range(2):   # drafting on the current subset while the event forms (other stream)
            ctx.subset_logits_topk(W, H, S, nd, n, 10)
        S2, n2, add, rem = ctx.oov_event_end(arc, step, S, n)
        torch.cuda.synchronize()
        # oracle pipeline for the same event
        b = oracle.build_subset(P["W"], q, static, seeds, P["row_ptr"], P["col"], n_sem=10, n_graph_sem_seeds=10,
                                per_seed=8, n_dyn=32)
        cand = np.setdiff1d(b["S"], static)
        before = set(oarc.members())
        oarc.admit(cand.tolist(), step)
        after = set(oarc.members())
        assert add == sorted(after - before) and rem == sorted(before - after), ev
        ref = oracle.subset_update(S.cpu().numpy()[:n], np.asarray(rem, np.int32), np.asarray(add, np.int32))
        np.testing.assert_array_equal(S2.cpu().numpy(), ref)
        np.testing.assert_array_equal(ref, np.union1d(static, np.asarray(sorted(after), np.int32)))
        assert int(n2.item()) == ref.size
        assert arc.state() == oarc.state()
        S, n = S2.clone(), ref.size
    # the LM head on the evolved subset
    nd = torch.tensor([n], dtype=torch.int32, device=DEV)
    ids, vals, m, s = ctx.subset_logits_topk(W, H, S, nd, n, 10)
    torch.cuda.synchronize()
    G.assert_triple_close(ids.cpu().numpy(), vals.cpu().numpy(), m.cpu().numpy(), s.cpu().numpy(),
                          oracle.subset_logits_topk(P["W"], P["H"], S.cpu().numpy()[:n], 10), 10)
    assert ctx.get_flags() == 0


def test_oov_event_protocol_errors():
    P = G.make_problem(82, dtype="bf16", V=4000, d=64, n_static=300, n_sem=10, n_dyn=32, n_h=2, k=4)
    W = G.to_dev(P["W"], DEV)
    ctx = es.Context(V=4000, d=64, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=400, max_rows=2,
                     max_k=8, max_sem=16, max_seeds=64)
    arc = es.Arc(64)
    S = G.to_dev(np.sort(P["static"]).astype(np.int32), DEV)
    with pytest.raises(es.EvospecError):   # _end without _begin
        ctx.oov_event_end(arc, 0, S, S.numel())
    args = (W, G.to_dev(P["q"], DEV), S, G.to_dev(P["seeds"], DEV), G.to_dev(P["row_ptr"], DEV),
            G.to_dev(P["col"], DEV))
    ctx.oov_event_begin(*args)
    with pytest.raises(es.EvospecError):   # a second event in flight
        ctx.oov_event_begin(*args)
    out, n, add, rem = ctx.oov_event_end(arc, 0, S, S.numel())
    torch.cuda.synchronize()
    assert int(n.item()) == S.numel() + len(add) - len(rem) and len(add) > 0
