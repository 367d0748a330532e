"""Host-side plumbing for vocab sharding; no compute here.

Shard r of R owns the token ids v with v mod R == r and stores id v at local
row v // R of its W / E slice. The library's own NCCL communicator carries the
data-path exchange (candidate pairs in evospec_build_subset, (top-k, m, s)
triples in evospec_merge_shards); torch.distributed is only used to broadcast
the 128-byte NCCL unique id at setup.
"""
from __future__ import annotations


def owner(v: int, R: int) -> int:
    return v % R


def local_row(v: int, R: int) -> int:
    return v // R


def shard_rows(W, R: int, r: int):
    """The rows of W (numpy or torch, [V, d]) owned by shard r, in local-row order."""
    return W[r::R]


def n_local_rows(V: int, R: int, r: int) -> int:
    return (V - r + R - 1) // R


def broadcast_bytes(payload, group=None, src_rank: int = 0, nbytes: int = 128) -> bytes:
    """Broadcast `nbytes` bytes from src_rank over a torch.distributed group
    (gloo: host tensor; nccl: device tensor)."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(nbytes, dtype=torch.uint8)
    if dist.get_rank(group) == src_rank:
        t = torch.tensor(list(bytes(payload))[:nbytes], dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    src = dist.get_global_rank(group, src_rank) if group is not None else src_rank
    dist.broadcast(t, src=src, group=group)
    return bytes(t.cpu().tolist())
