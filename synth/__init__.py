"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the EvoSpec method (no dot products, no
selection, no union, no softmax): it only draws random numbers and lays them
out in the byte formats both sides read. Both `oracle/` and the product path
consume exactly the arrays returned here; neither imports the other.

Workload recipe:
  * W (the LM head, also the semantic index E, reading C1) ~ N(0, 0.02^2)
    rounded to bf16, the HF init std of Llama/Qwen heads; H ~ N(0, 1) so the
    logits have std ~= 0.02*sqrt(d) (1.28 at d=4096).
  * static core = the first n_static ids of a seeded permutation of the
    vocabulary ("top-K frequent" of a Zipf corpus over a permuted vocab),
    returned sorted ascending (tab:hyperparams P:417).
  * co-occurrence CSR: per-row out-degree drawn from a truncated geometric
    law with the requested mean, capped at max_deg = 64; successors
    distinct, each row ordered (p desc, id asc).
  * seeds = synthetic "target top-10 at the rejection step".
  * an integer family with entries in {-3..3}: every partial sum is an
    integer < 2^24, exact in fp32 in any order, so ties are real.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "bf16_bits", "bf16_to_f32", "matrix", "int_matrix", "static_ids",
    "csr_graph", "seed_ids", "ctx_tokens", "CONFIGS", "domain_matrix",
]


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bit patterns (uint16), round-to-nearest-even."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32)
    r = (u >> 16) & 1          # finite inputs: u + 0x7FFF + 1 never wraps uint32
    r += 0x7FFF
    r += u
    r >>= 16
    return r.astype(np.uint16)


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) -> fp32 (exact)."""
    return (np.ascontiguousarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32)


def _normal(rng: np.random.Generator, shape, std: float) -> np.ndarray:
    out = rng.standard_normal(size=shape, dtype=np.float32)
    if std != 1.0:
        out *= np.float32(std)
    return out


_CHUNK_ROWS = 4096


def matrix(seed: int, rows: int, cols: int, std: float, dtype: str) -> np.ndarray:
    """Gaussian matrix; dtype 'bf16' returns uint16 bit patterns, 'fp32' float32.

    Large matrices are drawn in fixed chunks of 4096 rows, chunk i from the
    i-th child of SeedSequence(seed) (deterministic, thread-parallel)."""
    if dtype not in ("bf16", "fp32"):
        raise ValueError(dtype)
    if rows <= _CHUNK_ROWS:
        x = _normal(np.random.default_rng(seed), (rows, cols), std)
        return bf16_bits(x) if dtype == "bf16" else x
    from concurrent.futures import ThreadPoolExecutor
    n_chunks = (rows + _CHUNK_ROWS - 1) // _CHUNK_ROWS
    kids = np.random.SeedSequence(seed).spawn(n_chunks)
    out = np.empty((rows, cols), dtype=np.uint16 if dtype == "bf16" else np.float32)

    def work(i):
        r0, r1 = i * _CHUNK_ROWS, min(rows, (i + 1) * _CHUNK_ROWS)
        x = _normal(np.random.default_rng(kids[i]), (r1 - r0, cols), std)
        out[r0:r1] = bf16_bits(x) if dtype == "bf16" else x

    import os
    with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
        list(ex.map(work, range(n_chunks)))
    return out


def int_matrix(seed: int, rows: int, cols: int, dtype: str, lo: int = -3, hi: int = 3) -> np.ndarray:
    """Integer-valued matrix with entries in {lo..hi} (exact in bf16 and fp32)."""
    rng = np.random.default_rng(seed)
    x = rng.integers(lo, hi + 1, size=(rows, cols)).astype(np.float32)
    return bf16_bits(x) if dtype == "bf16" else x


def domain_matrix(seed: int, rows: int, cols: int, std: float, n_domains: int,
                  hot: int, alpha: float, dtype: str):
    """W with n_domains 'hot blocks' of `hot` ids each shifted along a domain mean.

    Mirrors the paper's specialised domains (Code/Law/Med) for the
    topic-switch config: rows in domain j's block get + alpha*mu_j/|mu_j|.
    Returns (W, mus, blocks) where mus [n_domains, cols] fp32 are the domain
    means (queries for domain j are mu_j + 0.5*xi).
    """
    rng = np.random.default_rng(seed)
    w = _normal(rng, (rows, cols), std)
    mus = rng.standard_normal(size=(n_domains, cols)).astype(np.float32)
    perm = rng.permutation(rows)
    blocks = []
    for j in range(n_domains):
        ids = np.sort(perm[j * hot:(j + 1) * hot])
        blocks.append(ids.astype(np.int32))
        w[ids] += np.float32(alpha) * (mus[j] / np.linalg.norm(mus[j]))[None, :]
    return (bf16_bits(w) if dtype == "bf16" else w), mus, blocks


def static_ids(seed: int, V: int, n_static: int) -> np.ndarray:
    """Sorted unique int32 ids: the first n_static of a seeded permutation."""
    rng = np.random.default_rng(seed)
    return np.sort(rng.permutation(V)[:n_static]).astype(np.int32)


def csr_graph(seed: int, V: int, avg_deg: float, max_deg: int = 64):
    """Random co-occurrence CSR (row_ptr int32[V+1], col int32[nnz], prob fp32[nnz]).

    Rows are sorted by (prob desc, id asc); successors within a row are
    distinct and != the source. Probabilities are a random normalised split
    of each row's mass (they only fix the row order on the hot path).
    """
    rng = np.random.default_rng(seed)
    p_geo = 1.0 / (1.0 + avg_deg)
    deg = np.minimum(rng.geometric(p_geo, size=V) - 1, max_deg).astype(np.int64)
    row_ptr = np.zeros(V + 1, dtype=np.int64)
    np.cumsum(deg, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    src = np.repeat(np.arange(V, dtype=np.int64), deg)
    # distinct successors != src: offsets start + k*step with
    # 1 <= start and start + max_deg*step < V, so every offset lies in
    # [1, V-1] and the offsets of one row are pairwise distinct.
    step = rng.integers(1, max(2, V // (max_deg + 1)), size=V, dtype=np.int64)
    span = np.maximum(V - max_deg * step - 1, 1)
    start = 1 + (rng.random(size=V) * span).astype(np.int64)
    k = np.arange(nnz, dtype=np.int64) - row_ptr[src]
    col = (src + start[src] + k * step[src]) % V
    w = rng.exponential(size=nnz)
    # normalise per row
    sums = np.zeros(V)
    np.add.at(sums, src, w)
    prob = (w / sums[src]).astype(np.float32)
    # order each row by (prob desc, id asc)
    order = np.lexsort((col, -prob.astype(np.float64), src))
    col = col[order]
    prob = prob[order]
    return row_ptr.astype(np.int32), col.astype(np.int32), prob


def seed_ids(seed: int, V: int, n: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.choice(V, size=n, replace=False).astype(np.int32)


def ctx_tokens(seed: int, V: int, n: int, vocab_window: int = 512) -> np.ndarray:
    """Context token stream with repeats (draws from a small window of ids)."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, max(1, V - vocab_window))
    return (base + rng.zipf(1.3, size=n) % vocab_window).astype(np.int32)


# The five BASELINE.json configs (SURVEY.md §8 top, §8(d)).
CONFIGS = {
    "tiny": dict(V=1024, d=64, dtype="fp32", n_static=128, n_sem=32, n_dyn=64,
                 n_seed=10, n_graph_sem_seeds=10, per_seed=8, n_h=4, k=8,
                 avg_deg=8.0, w_std=1.0, h_std=1.0 / 8.0),
    "llama": dict(V=128256, d=4096, dtype="bf16", n_static=32768, n_sem=8192,
                  n_dyn=4096, n_seed=10, n_graph_sem_seeds=10, per_seed=8,
                  n_h=60, k=10, avg_deg=32.0, w_std=0.02, h_std=1.0),
    "qwen": dict(V=152064, d=3584, dtype="bf16", n_static=32768, n_sem=8192,
                 n_dyn=4096, n_seed=10, n_graph_sem_seeds=10, per_seed=8,
                 n_h=60, k=10, avg_deg=32.0, w_std=0.02, h_std=1.0),
    "sharded": dict(V=128256, d=8192, dtype="bf16", n_static=128256 - 4096,
                    n_sem=8192, n_dyn=4096, n_seed=10, n_graph_sem_seeds=10,
                    per_seed=8, n_h=60, k=10, avg_deg=32.0, w_std=0.02, h_std=1.0),
}


def verify_problem(seed: int, *, V: int, g: int, n_S: int, inv_temp: float = 1.0, s_range: int = 0) -> dict:
    """Inputs of the N2 verification step, seeded: target logits z
    [g+1, V] fp32 (N(0, 1.28^2): the llama head's logit scale, §8(d)), a sorted
    random subset S of n_S ids, the draft's restricted distribution q on S
    ([g, n_S] fp32; a draft whose logits are the target's on S plus N(0, 0.5^2)
    noise, normalised on S -- an input, not the method's arithmetic), proposals
    x_j drawn from q_j, uniforms u [g] and w [g+1] (fp64, [0, 1)). s_range > 0: the
    subset is drawn from ids [0, s_range) only (a subset concentrated in one part of
    the vocabulary)."""
    rng = np.random.default_rng(seed)
    z = (rng.normal(size=(g + 1, V)) * 1.28).astype(np.float32)
    n_S = min(n_S, V)
    S = np.sort(rng.choice(s_range if s_range > 0 else V, n_S, replace=False)).astype(np.int32)
    dl = z[:g, S].astype(np.float64) * inv_temp + rng.normal(size=(g, n_S)) * 0.5
    q = np.exp(dl - dl.max(axis=1, keepdims=True))
    q /= q.sum(axis=1, keepdims=True)
    q = q.astype(np.float32)
    x = np.array([S[rng.choice(n_S, p=q[j].astype(np.float64) / q[j].astype(np.float64).sum())]
                  for j in range(g)], np.int32)
    u = rng.random(g)
    w = rng.random(g + 1)
    return dict(z=z, S=S, q=q, x=x, u=u, w=w, V=V, g=g, inv_temp=inv_temp)
