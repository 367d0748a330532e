"""World-size-2 gloo tests of the N>1 host logic (CPU only).

The vocab-sharded path: interleaved ownership (v mod R), local rows v // R,
the stacked [R, n_h, k] / [R, n_h] triple layout that evospec_merge_shards
consumes after its all-gather, and the unique-id broadcast helper that
Context.comm_init uses. Compute on each rank is the oracle (CPU); the
exchange is torch.distributed over gloo with the same layout as the library's
NCCL all-gather.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        from paper_2605_27390_b200 import dist as esd

        # unique-id broadcast (Context.comm_init's plumbing)
        payload = bytes(range(128)) if rank == 0 else None
        got = esd.broadcast_bytes(payload)
        assert got == bytes(range(128))

        V, d, n_h, k = 4099, 32, 5, 9
        W = synth.int_matrix(30, V, d, "fp32")     # integer data: exact cross-shard ties
        H = synth.int_matrix(31, n_h, d, "fp32")
        S = np.sort(np.random.default_rng(7).choice(V, 1500, replace=False)).astype(np.int32)
        # this rank's shard, exactly as bench.py / the C ABI lay it out
        W_loc = np.ascontiguousarray(esd.shard_rows(W, world, rank))
        assert W_loc.shape[0] == esd.n_local_rows(V, world, rank)
        S_loc = S[np.array([esd.owner(int(v), world) == rank for v in S], dtype=bool)]
        for v in S_loc[:50]:
            assert np.array_equal(W_loc[esd.local_row(int(v), world)], W[v])
        tri = oracle.subset_logits_topk(W_loc, H, S_loc, k, R=world)
        # all-gather into the stacked layout evospec_merge_shards consumes
        def gather(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t)
            return np.stack([o.numpy() for o in out])
        ids, vals, m, s = gather(tri["ids"]), gather(tri["vals"]), gather(tri["m"]), gather(tri["s"])
        assert ids.shape == (world, n_h, k) and m.shape == (world, n_h)
        merged = oracle.merge(ids, vals, m, s, k)
        ref = oracle.subset_logits_topk(W, H, S, k)
        assert np.array_equal(merged["ids"], ref["ids"])
        assert np.allclose(merged["lse"], ref["lse"], rtol=1e-12)
        assert np.allclose(merged["probs"], ref["probs"], atol=1e-12)
        # every rank holds the identical merged result
        h = torch.from_numpy(merged["ids"].astype(np.int64)).sum()
        hs = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        assert all(int(x) == int(h) for x in hs)
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2])
def test_vocab_shard_merge_gloo(world):
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}: {msg}"
