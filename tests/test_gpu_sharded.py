"""The vocab-sharded path on one GPU, through the C ABI, against
the unsharded oracle: R interleaved shards (shard r owns ids v = r mod R, local
row v / R), each running
  1. its exact local semantic top-N over its rows of E (evospec_build_local_candidates),
  2. the global selection + formation / union over the R candidate lists stacked in
     rank order (evospec_build_subset_from_candidates; the NCCL path all-gathers the
     same lists) -> the same sorted S on every shard and the shard's owned slice,
  3. its LM head over its slice (evospec_subset_logits_topk on W_local, exact top-k
     values because the triple feeds a cross-shard merge),
and the R triples merged (evospec_merge_shards, stacked mode). S, the semantic set and
the merged ids are bit-exact; LSE and probabilities within the north-star tolerances.
The multi-GPU run of the same calls with the NCCL exchanges is tests/test_dist_gpu.py.
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


def sharded_chain(P, R, inv_temp=1.0):
    nmax = P["static"].size + P["n_dyn"]
    dev = lambda a: G.to_dev(np.ascontiguousarray(a), DEV)
    ctxs, Ws, cands = [], [], []
    q, H = dev(P["q"]), dev(P["H"])
    for r in range(R):
        ctx = es.Context(V=P["V"], d=P["d"], w_dtype=G.torch_dtype(P["dtype"]), h_dtype=G.torch_dtype(P["dtype"]),
                         n_shards=R, shard_rank=r, max_subset=nmax, max_rows=P["n_h"], max_k=64,
                         max_sem=P["n_sem"], max_seeds=64, debug_checks=True)
        Wr = dev(P["W"][r::R])
        ctx.prepare_weights(Wr)
        cands.append(ctx.build_local_candidates(Wr, q, P["n_sem"]))
        ctxs.append(ctx)
        Ws.append(Wr)
    cs = torch.cat([c[0] for c in cands])
    ci = torch.cat([c[1] for c in cands])
    out = []
    for r, ctx in enumerate(ctxs):
        ids, n, lids, ln = ctx.build_subset_from_candidates(
            cs, ci, dev(P["static"]), dev(P["seeds"]), dev(P["row_ptr"]), dev(P["col"]), n_sem=P["n_sem"],
            n_dyn=P["n_dyn"], n_graph_sem_seeds=P["n_graph_sem_seeds"], per_seed=P["per_seed"])
        sem = ctx.last_semantic(P["n_sem"])
        trip = ctx.subset_logits_topk(Ws[r], H, lids, ln, nmax, P["k"], inv_temp)
        out.append(dict(ids=ids, n=n, lids=lids, ln=ln, sem=sem, trip=trip, ctx=ctx))
    st = [torch.stack([o["trip"][i] for o in out]) for i in range(4)]
    merged = ctxs[0].merge_shards(*st, n_h=P["n_h"], k=P["k"])
    torch.cuda.synchronize()
    return out, merged


@pytest.mark.parametrize("R", [2, 3, 4])
def test_sharded_build_lmh_merge_on_one_gpu(R):
    P = G.make_problem(31 + R, dtype="bf16", V=20011, d=512, n_static=2999, n_sem=700, n_dyn=517, n_h=12, k=10,
                       avg_deg=16)
    ref = G.oracle_step(oracle, P)
    S = ref["S"]
    out, (oi, ov, ol, op) = sharded_chain(P, R)
    for r, o in enumerate(out):
        n = int(o["n"].item())
        np.testing.assert_array_equal(o["ids"][:n].cpu().numpy(), S)            # the same S on every shard
        ln = int(o["ln"].item())
        np.testing.assert_array_equal(o["lids"][:ln].cpu().numpy(), S[S % R == r])   # the owned slice
        np.testing.assert_array_equal(np.sort(o["sem"].cpu().numpy()), np.sort(ref["sem"]))
        assert o["ctx"].get_flags() == 0
    np.testing.assert_array_equal(oi.cpu().numpy(), ref["triple"]["ids"])
    lse = ref["triple"]["lse"]
    assert np.all(np.abs(ol.cpu().numpy() - lse) <= G.LOGIT_TOL * (1 + np.abs(lse)))
    assert np.max(np.abs(op.cpu().numpy() - ref["triple"]["probs"])) <= G.PROB_TOL


def test_sharded_chain_ties_and_temperature():
    """Duplicated W rows put exact score / logit ties across shards (ties to the lower
    id through the candidate exchange and the merge); inv_temp != 1."""
    P = G.make_problem(44, dtype="bf16", V=12000, d=256, n_static=1500, n_sem=400, n_dyn=300, n_h=7, k=16,
                       dup_rows=500, avg_deg=12)
    it = float(np.float32(1 / 0.7))
    ref = G.oracle_step(oracle, P, inv_temp=it)
    out, (oi, ov, ol, op) = sharded_chain(P, 4, inv_temp=it)
    n = int(out[0]["n"].item())
    np.testing.assert_array_equal(out[0]["ids"][:n].cpu().numpy(), ref["S"])
    np.testing.assert_array_equal(oi.cpu().numpy(), ref["triple"]["ids"])
    assert np.max(np.abs(op.cpu().numpy() - ref["triple"]["probs"])) <= G.PROB_TOL


def test_local_candidates_are_the_shard_top_n():
    """Step 1 alone: a shard's list is its exact top-N of s_v = q . E_v over the ids it
    owns, ordered (s desc, id asc), global ids, against the oracle's fp64 scores."""
    P = G.make_problem(50, dtype="bf16", V=9001, d=128, n_static=100, n_sem=300, n_dyn=10, n_h=1, k=1)
    s = oracle.sem_scores(P["W"], P["q"])
    R, r = 3, 1
    ctx = es.Context(V=P["V"], d=P["d"], w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, n_shards=R, shard_rank=r,
                     max_subset=1000, max_rows=1, max_k=1, max_sem=300)
    cs, ci = ctx.build_local_candidates(G.to_dev(np.ascontiguousarray(P["W"][r::R]), DEV), G.to_dev(P["q"], DEV), 300)
    torch.cuda.synchronize()
    own = np.arange(r, P["V"], R)
    order = np.lexsort((own, -s[own]))[:300]
    ids = ci.cpu().numpy()
    np.testing.assert_array_equal(np.sort(ids), np.sort(own[order]))
    # (fp64 sums in a different order than the oracle's sequential one: relative 1e-12)
    np.testing.assert_allclose(cs.cpu().numpy()[np.argsort(ids)], s[np.sort(own[order])], rtol=1e-12, atol=1e-12)
