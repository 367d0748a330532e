"""Worker of tests/test_dist_gpu.py: one rank per GPU (torchrun), the library's own
NCCL communicator. Each rank holds its interleaved W / E shard; the sharded build
(local scan, candidate all-gather, global selection), the LM head over the owned
slice, the triple all-gather + merge (evospec_merge_shards), then the sharded
evospec_draft_step (CUDA-graph replay on the second call) -- every rank checks its
replicated result against the unsharded oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist

    import oracle
    import paper_2605_27390_b200 as es
    from tests import gpu_helpers as G

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    dist.init_process_group("nccl", device_id=torch.device(dev))
    P = G.make_problem(61, dtype="bf16", V=30011, d=512, n_static=3000, n_sem=800, n_dyn=600, n_h=16, k=10,
                       avg_deg=16, dup_rows=200)
    ref = G.oracle_step(oracle, P)
    S = ref["S"]
    nmax = P["static"].size + P["n_dyn"]
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev) if a.dtype != np.uint16 else \
        torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    ctx = es.Context(V=P["V"], d=P["d"], w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, n_shards=world,
                     shard_rank=rank, max_subset=nmax, max_rows=P["n_h"], max_k=16, max_sem=P["n_sem"],
                     max_seeds=64, device=local)
    ctx.comm_init()
    W_loc = t(P["W"][rank::world])
    ctx.prepare_weights(W_loc)
    ids, n, lids, ln = ctx.build_subset(W_loc, t(P["q"]), t(P["static"]), t(P["seeds"]), t(P["row_ptr"]),
                                        t(P["col"]), n_sem=P["n_sem"], n_dyn=P["n_dyn"],
                                        n_graph_sem_seeds=P["n_graph_sem_seeds"], per_seed=P["per_seed"])
    tri = ctx.subset_logits_topk(W_loc, t(P["H"]), lids, ln, nmax, P["k"])
    oi, ov, ol, op = ctx.merge_shards(*tri, n_h=P["n_h"], k=P["k"])
    torch.cuda.synchronize()
    nn = int(n.item())
    assert np.array_equal(ids[:nn].cpu().numpy(), S), "subset differs from the oracle"
    assert np.array_equal(lids[:int(ln.item())].cpu().numpy(), S[S % world == rank]), "owned slice"
    assert np.array_equal(oi.cpu().numpy(), ref["triple"]["ids"]), "merged ids"
    lse = ref["triple"]["lse"]
    assert np.all(np.abs(ol.cpu().numpy() - lse) <= G.LOGIT_TOL * (1 + np.abs(lse))), "LSE"
    assert np.max(np.abs(op.cpu().numpy() - ref["triple"]["probs"])) <= G.PROB_TOL, "probs"
    kw = dict(E=W_loc, W_local=W_loc, static_ids=t(P["static"]), csr_row_ptr=t(P["row_ptr"]),
              csr_col=t(P["col"]), k=P["k"], n_sem=P["n_sem"], n_dyn=P["n_dyn"])
    for _ in range(3):   # first call captures the graph, the next replay it
        out = ctx.draft_step(q=t(P["q"]), H=t(P["H"]), seeds=t(P["seeds"]), **kw)
        torch.cuda.synchronize()
        assert np.array_equal(out[0].cpu().numpy(), ref["triple"]["ids"]), "draft_step ids"
        assert np.max(np.abs(out[3].cpu().numpy() - ref["triple"]["probs"])) <= G.PROB_TOL, "draft_step probs"
    assert ctx.get_flags() == 0
    dist.barrier()
    print(f"rank {rank} ok", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
