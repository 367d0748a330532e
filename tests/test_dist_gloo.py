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


def _cand_worker(rank, world, port, q):
    """The sharded build's candidate exchange (what evospec_build_subset
    all-gathers over NCCL and evospec_build_subset_from_candidates consumes): each rank's
    exact local top-N over its owned ids (global id = local row * R + r), N (s, id) pairs
    per rank stacked in rank order; the global top-N of the R * N gathered pairs equals
    the unsharded top-N, and every rank resolves the same set."""
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        from paper_2605_27390_b200 import dist as esd

        V, d, N = 5003, 48, 257
        E = synth.matrix(40, V, d, 0.5, "bf16")
        E[100:140] = E[600:640]           # duplicated rows: exact score ties across shards
        qv = synth.matrix(41, 1, d, 1.0, "bf16")[0]
        E_loc = np.ascontiguousarray(esd.shard_rows(E, world, rank))
        s_loc = oracle.sem_scores(E_loc, qv)
        top = oracle.topn(s_loc, min(N, s_loc.size))          # local rows, (s desc, row asc)
        ids = (top * world + rank).astype(np.int32)            # local row -> global id
        s = s_loc[top]
        ids = np.concatenate([ids, np.full(N - ids.size, -1, np.int32)])
        s = np.concatenate([s, np.full(N - s.size, -np.inf)])

        def gather(a):
            tt = torch.from_numpy(np.ascontiguousarray(a))
            out = [torch.empty_like(tt) for _ in range(world)]
            dist.all_gather(out, tt)
            return np.concatenate([o.numpy() for o in out])
        gs, gi = gather(s), gather(ids)
        ok = gi >= 0
        order = np.lexsort((gi[ok], -gs[ok]))[:N]            # the global selection, (s desc, id asc)
        got = np.sort(gi[ok][order])
        ref = np.sort(oracle.topn(oracle.sem_scores(E, qv), N))
        assert np.array_equal(got, ref), "gathered global top-N differs from the unsharded one"
        h = torch.tensor(int(got.astype(np.int64).sum()))
        hs = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        assert all(int(x) == int(h) for x in hs)
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world", [2, 3])
def test_candidate_exchange_gloo(world):
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cand_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for rank, msg in res:
        assert msg == "ok", f"rank {rank}: {msg}"
