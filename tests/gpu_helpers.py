"""Shared helpers for the GPU parity tests, smoke() and bench.py.

Builds seeded inputs with synth/ (numpy), moves them to the device for the
CUDA path, and runs the oracle (oracle/) on the same numpy arrays. The CUDA
path and the oracle never exchange values: both consume the generator output.
"""
from __future__ import annotations

import numpy as np

import synth

# north-star tolerances (BASELINE.json north_star)
LOGIT_TOL = 2e-3      # |dz| <= 2e-3 * (1 + |z|)
PROB_TOL = 1e-4       # |dp| <= 1e-4


def to_dev(a: np.ndarray, device="cuda"):
    import torch
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).to(device)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def torch_dtype(code: str):
    import torch
    return torch.bfloat16 if code == "bf16" else torch.float32


def make_problem(seed: int, *, V: int, d: int, dtype: str, n_static: int, n_sem: int, n_dyn: int,
                 n_seed: int = 10, n_graph_sem_seeds: int = 10, per_seed: int = 8, n_h: int = 4,
                 k: int = 8, avg_deg: float = 8.0, w_std: float = 0.02, h_std: float = 1.0,
                 integer: bool = False, dup_rows: int = 0, **_):
    """Seeded synthetic problem in numpy (host); integer=True draws {-3..3}."""
    if integer:
        W = synth.int_matrix(seed, V, d, dtype)
        H = synth.int_matrix(seed + 1, n_h, d, dtype)
        q = synth.int_matrix(seed + 2, 1, d, dtype)[0]
    else:
        W = synth.matrix(seed, V, d, w_std, dtype)
        H = synth.matrix(seed + 1, n_h, d, h_std, dtype)
        q = synth.matrix(seed + 2, 1, d, 1.0, dtype)[0]
    if dup_rows:
        # duplicate rows -> exact ties in both the semantic scores and the logits
        rng = np.random.default_rng(seed + 7)
        src = rng.choice(V, dup_rows, replace=False)
        dst = rng.choice(V, dup_rows, replace=False)
        W[dst] = W[src]
    static = synth.static_ids(seed + 3, V, n_static)
    row_ptr, col, _prob = synth.csr_graph(seed + 4, V, avg_deg)
    seeds = synth.seed_ids(seed + 5, V, n_seed) if n_seed else np.zeros(0, np.int32)
    return dict(W=W, H=H, q=q, static=static, row_ptr=row_ptr, col=col, seeds=seeds,
                n_sem=n_sem, n_dyn=n_dyn, n_graph_sem_seeds=n_graph_sem_seeds,
                per_seed=per_seed, k=k, V=V, d=d, dtype=dtype, n_h=n_h)


def oracle_step(oracle, P, *, R: int = 1, inv_temp: float = 1.0, S=None):
    """Oracle reference for one step: subset, unsplit triple, merged outputs."""
    if S is None:
        b = oracle.build_subset(P["W"], P["q"], P["static"], P["seeds"], P["row_ptr"], P["col"],
                                n_sem=P["n_sem"], n_graph_sem_seeds=P["n_graph_sem_seeds"],
                                per_seed=P["per_seed"], n_dyn=P["n_dyn"])
        S = b["S"]
        sem = b["sem"]
    else:
        sem = None
    t = oracle.subset_logits_topk(P["W"], P["H"], S, P["k"], inv_temp=inv_temp)
    return dict(S=S, sem=sem, triple=t)


def assert_triple_close(ids, vals, m, s, ref, k: int):
    ids = np.asarray(ids)
    vals = np.asarray(vals, np.float64)
    np.testing.assert_array_equal(ids, ref["ids"][:, :k])
    fin = np.isfinite(ref["vals"][:, :k])
    np.testing.assert_array_equal(np.isfinite(vals), fin)
    dv = np.abs(vals[fin] - ref["vals"][:, :k][fin])
    assert np.all(dv <= LOGIT_TOL * (1 + np.abs(ref["vals"][:, :k][fin]))), dv.max()
    lse = np.asarray(m, np.float64) + np.log(np.asarray(s, np.float64))
    fin = np.isfinite(ref["lse"])
    assert np.all(np.abs(lse[fin] - ref["lse"][fin]) <= LOGIT_TOL * (1 + np.abs(ref["lse"][fin])))


def near_tie_count(scores, n: int, rel: float = 1e-12) -> int:
    """SURVEY §8(c) C10 near-tie counter: 1 if the oracle's fp64 values ranked n and
    n + 1 (descending) differ by less than rel (relative) without being equal -- a
    boundary where a reassociated fp64 sum on the GPU could legitimately order the
    two the other way. Rows: a 2-D array counts per row."""
    a = np.atleast_2d(np.asarray(scores, np.float64))
    if a.shape[1] <= n:
        return 0
    part = -np.partition(-a, n, axis=1)[:, : n + 1]
    srt = -np.sort(-part, axis=1)
    x, y = srt[:, n - 1], srt[:, n]
    gap = np.abs(x - y)
    return int(np.sum((gap > 0) & (gap <= rel * np.maximum(np.abs(x), np.abs(y)))))
