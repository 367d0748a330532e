"""ctypes wrapper over oracle/evospec_oracle.c.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package
(paper_2605_27390_b200/). The C source shares no code with the CUDA path.

Every function here is argument marshalling; the arithmetic is in the C file,
each function there citing the PAPER.md / SPEC.md passage it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "evospec_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

BF16, FP32 = 0, 1


def build(force: bool = False) -> str:
    """Compile the oracle with g++/gcc -O2 (no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _L():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_LIB)
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _dt(a: np.ndarray) -> int:
    if a.dtype == np.uint16:
        return BF16
    if a.dtype == np.float32:
        return FP32
    raise TypeError(f"oracle inputs are bf16 bits (uint16) or float32, got {a.dtype}")


def _check(rc: int, what: str):
    if rc != 0:
        raise ValueError(f"oracle {what}: input error (rc={rc})")


def _i32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int32)


def sem_scores(E: np.ndarray, q: np.ndarray) -> np.ndarray:
    E = np.ascontiguousarray(E)
    q = np.ascontiguousarray(q).reshape(-1)
    n, d = E.shape
    out = np.empty(n, dtype=np.float64)
    f = _L().eo_sem_scores
    f.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_void_p, C.c_int, C.c_void_p]
    _check(f(_p(E), _dt(E), n, d, _p(q), _dt(q), _p(out)), "sem_scores")
    return out


def topn(s: np.ndarray, N: int) -> np.ndarray:
    s = np.ascontiguousarray(s, dtype=np.float64)
    out = np.empty(N, dtype=np.int32)
    f = _L().eo_topn
    f.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p]
    _check(f(_p(s), s.size, N, _p(out)), "topn")
    return out


def graph_expand(G, row_ptr, col, per_seed: int) -> np.ndarray:
    G = _i32(G)
    row_ptr = _i32(row_ptr)
    col = _i32(col)
    out = np.empty(max(1, G.size * per_seed), dtype=np.int32)
    n = C.c_int(0)
    f = _L().eo_graph_expand
    f.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    _check(f(_p(G), G.size, _p(row_ptr), _p(col), per_seed, _p(out), C.byref(n)), "graph_expand")
    return out[:n.value].copy()


def ctx_tokens(ctx, V: int, min_count: int, n_max: int) -> np.ndarray:
    ctx = _i32(ctx) if ctx is not None else np.zeros(0, np.int32)
    out = np.empty(max(1, n_max), dtype=np.int32)
    n = C.c_int(0)
    f = _L().eo_ctx_tokens
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
    _check(f(_p(ctx), ctx.size, V, min_count, n_max, _p(out), C.byref(n)), "ctx_tokens")
    return out[:n.value].copy()


def build_subset(E, q, static_ids, seed_ids, row_ptr, col, *, n_sem: int,
                 n_graph_sem_seeds: int = 10, per_seed: int = 8, n_dyn: int,
                 ctx_ids=None, ctx_min_count: int = 0, n_ctx_max: int = 0):
    """Returns dict(S, sem, dyn) per SURVEY §8(c) steps 2-8."""
    E = np.ascontiguousarray(E)
    q = np.ascontiguousarray(q).reshape(-1)
    V, d = E.shape
    static_ids = _i32(static_ids)
    seed_ids = _i32(seed_ids) if seed_ids is not None else np.zeros(0, np.int32)
    ctx = _i32(ctx_ids) if ctx_ids is not None else np.zeros(0, np.int32)
    row_ptr = _i32(row_ptr)
    col = _i32(col)
    S = np.empty(static_ids.size + n_dyn + 1, dtype=np.int32)
    nS = C.c_int32(0)
    sem = np.empty(max(1, n_sem), dtype=np.int32)
    dyn = np.empty(max(1, n_dyn), dtype=np.int32)
    nd = C.c_int32(0)
    f = _L().eo_build_subset
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                  C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                  C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    rc = f(_p(E), _dt(E), V, d, _p(q), _dt(q), _p(static_ids), static_ids.size,
           _p(seed_ids), seed_ids.size, _p(row_ptr), _p(col), _p(ctx), ctx.size,
           n_sem, n_graph_sem_seeds, per_seed, ctx_min_count, n_ctx_max, n_dyn,
           _p(S), C.byref(nS), _p(sem), _p(dyn), C.byref(nd))
    _check(rc, "build_subset")
    return dict(S=S[:nS.value].copy(), sem=sem[:n_sem].copy(), dyn=dyn[:nd.value].copy())


def subset_logits(W, H, S, *, R: int = 1, inv_temp: float = 1.0) -> np.ndarray:
    """z [n_h, n_S] (float64) for a shard's W_local (rows v // R)."""
    W = np.ascontiguousarray(W)
    H = np.ascontiguousarray(H)
    S = _i32(S)
    n_rows, d = W.shape
    n_h = H.shape[0]
    out = np.empty((n_h, S.size), dtype=np.float64)
    f = _L().eo_subset_logits
    f.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int, C.c_void_p, C.c_int, C.c_int,
                  C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_void_p]
    _check(f(_p(W), _dt(W), n_rows, d, _p(H), _dt(H), n_h, _p(S), S.size, R,
             float(inv_temp), _p(out)), "subset_logits")
    return out


def softmax_topk(z: np.ndarray, S, k: int):
    """Returns dict(ids, vals, m, s, lse, probs) per §8(c) steps 10-11."""
    z = np.ascontiguousarray(z, dtype=np.float64)
    S = _i32(S)
    n_h = z.shape[0]
    ids = np.empty((n_h, k), np.int32)
    vals = np.empty((n_h, k), np.float64)
    probs = np.empty((n_h, k), np.float64)
    m = np.empty(n_h, np.float64)
    s = np.empty(n_h, np.float64)
    lse = np.empty(n_h, np.float64)
    f = _L().eo_softmax_topk
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int] + [C.c_void_p] * 6
    _check(f(_p(z), n_h, S.size, _p(S), k, _p(ids), _p(vals), _p(m), _p(s), _p(lse),
             _p(probs)), "softmax_topk")
    return dict(ids=ids, vals=vals, m=m, s=s, lse=lse, probs=probs)


def subset_logits_topk(W, H, S, k: int, *, R: int = 1, inv_temp: float = 1.0):
    """The shard triple (ids, vals, m, s) plus lse/probs of the shard alone."""
    z = subset_logits(W, H, S, R=R, inv_temp=inv_temp)
    return softmax_topk(z, S, k)


def merge(ids, vals, m, s, k: int):
    """Stacked [R, n_h, k] / [R, n_h] shard triples -> dict(ids, vals, lse, probs)."""
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.float64)
    m = np.ascontiguousarray(m, dtype=np.float64)
    s = np.ascontiguousarray(s, dtype=np.float64)
    R, n_h = m.shape
    oi = np.empty((n_h, k), np.int32)
    ov = np.empty((n_h, k), np.float64)
    ol = np.empty(n_h, np.float64)
    op = np.empty((n_h, k), np.float64)
    f = _L().eo_merge
    f.argtypes = [C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 8
    _check(f(R, n_h, k, _p(ids), _p(vals), _p(m), _p(s), _p(oi), _p(ov), _p(ol), _p(op)), "merge")
    return dict(ids=oi, vals=ov, lse=ol, probs=op)


def shard_subset(S, R: int, r: int) -> np.ndarray:
    """S_r = [v in S : v mod R = r] (§8(c) step 12, interleaved ownership)."""
    S = np.asarray(S)
    return S[S % R == r].astype(np.int32)


def shard_rows(W, R: int, r: int):
    """W_local for shard r: global rows v = r (mod R), local row v // R."""
    return np.ascontiguousarray(W[r::R])


def build_subset_batched(E, Q, static_ids, seed_ids, seed_offsets, row_ptr, col, *, n_sem: int,
                         n_dyn: int, n_graph_sem_seeds: int = 10, per_seed: int = 8, ctx_ids=None,
                         ctx_offsets=None, ctx_min_count: int = 0, n_ctx_max: int = 0):
    """Batched serving build (SURVEY §8(a) a4, config Bt): for each sequence b the
    single-query build (§8(c) steps 2-8) with q = Q[b], its own seeds / context
    tokens and the shared static set; returns (dyn_ids concatenated, offsets [B+1])
    with dyn_b = sorted(dyn) -- the dynamic part only (static excluded)."""
    Q = np.ascontiguousarray(Q)
    seed_ids = np.zeros(0, np.int32) if seed_ids is None else _i32(seed_ids)
    out, offs = [], [0]
    for b in range(Q.shape[0]):
        seeds_b = seed_ids[seed_offsets[b]:seed_offsets[b + 1]]
        ctx_b = None if ctx_ids is None else _i32(ctx_ids)[ctx_offsets[b]:ctx_offsets[b + 1]]
        r = build_subset(E, Q[b], static_ids, seeds_b, row_ptr, col, n_sem=n_sem,
                         n_graph_sem_seeds=n_graph_sem_seeds, per_seed=per_seed, n_dyn=n_dyn,
                         ctx_ids=ctx_b, ctx_min_count=ctx_min_count, n_ctx_max=n_ctx_max)
        dyn_b = np.sort(r["dyn"]).astype(np.int32)
        out.append(dyn_b)
        offs.append(offs[-1] + dyn_b.size)
    dyn = np.concatenate(out) if out else np.zeros(0, np.int32)
    return dyn.astype(np.int32), np.asarray(offs, dtype=np.int64)


def subset_logits_topk_ragged(W, H, h_offsets, static_ids, dyn_ids, dyn_offsets, k: int, *,
                              inv_temp: float = 1.0):
    """Ragged batched LM head (config Bt): the rows of sequence b against its own
    V_b = sort(static u dyn_b) (Eq. 1 P:47 restricted per sequence; §8(c) steps
    9-11 per sequence). Returns dict(ids, vals, m, s, lse, probs) over all rows."""
    static_ids = _i32(static_ids)
    dyn_ids = _i32(dyn_ids)
    parts = []
    for b in range(len(h_offsets) - 1):
        h0, h1 = int(h_offsets[b]), int(h_offsets[b + 1])
        if h1 == h0:
            continue
        S_b = np.union1d(static_ids, dyn_ids[int(dyn_offsets[b]):int(dyn_offsets[b + 1])]).astype(np.int32)
        parts.append(subset_logits_topk(W, H[h0:h1], S_b, k, inv_temp=inv_temp))
    return {key: np.concatenate([p[key] for p in parts]) for key in ("ids", "vals", "m", "s", "lse", "probs")}


def verify_chain(z, x, S, qS, *, inv_temp: float = 1.0, greedy: bool, u=None, w=None):
    """N2: lossless verification of a draft chain (eo_verify_chain). z float32 [g+1, V] target
    logits, x int32 [g] proposals, S sorted int32 subset, qS float32 [g, n_S] draft
    probabilities on S (None in greedy mode), u [g] / w [g+1] uniforms (float64).
    Returns (tokens int32[n_acc + 1], n_acc)."""
    z = np.ascontiguousarray(z, dtype=np.float32)
    g1, V = z.shape
    g = g1 - 1
    x = _i32(np.asarray(x if x is not None else [], dtype=np.int32).reshape(-1))
    S = _i32(np.asarray(S if S is not None else [], dtype=np.int32).reshape(-1))
    qS = None if qS is None else np.ascontiguousarray(qS, dtype=np.float32)
    u = None if u is None else np.ascontiguousarray(u, dtype=np.float64)
    w = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    tokens = np.full(g + 1, -1, np.int32)
    n_acc = np.zeros(1, np.int32)
    f = _L().eo_verify_chain
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_double,
                  C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
    rc = f(_p(z), V, g, _p(x), _p(S), int(S.size), _p(qS), float(inv_temp), int(bool(greedy)), _p(u), _p(w),
           _p(tokens), _p(n_acc))
    if rc == 3:
        raise ValueError("oracle verify_chain: a proposal has draft probability 0 (S:383)")
    _check(rc, "verify_chain")
    n = int(n_acc[0])
    return tokens[:n + 1].copy(), n


def coverage(z, S, ks, *, inv_temp: float = 1.0):
    """N4: covered mass and Recall@k of the subset S against the target rows z (eo_coverage).
    z float32 [n_rows, V] logits; S sorted int32; ks list of k. Returns (mass [n_rows],
    recall [n_rows, len(ks)]) as float64."""
    z = np.ascontiguousarray(np.atleast_2d(z), dtype=np.float32)
    n_rows, V = z.shape
    S = _i32(np.asarray(S, dtype=np.int32).reshape(-1))
    ks = _i32(np.asarray(ks, dtype=np.int32).reshape(-1))
    mass = np.zeros(n_rows, np.float64)
    rec = np.zeros((n_rows, max(1, ks.size)), np.float64)
    f = _L().eo_coverage
    f.restype = C.c_int
    f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_int,
                  C.c_void_p, C.c_void_p]
    _check(f(_p(z), n_rows, V, _p(S), int(S.size), float(inv_temp), _p(ks), int(ks.size), _p(mass), _p(rec)),
           "coverage")
    return mass, rec[:, :ks.size]


def kd_loss(zp, zq, verified, *, T: float = 1.0, beta: float = 0.3):
    """N3: curriculum-weighted KD objective (eo_kd_loss). zp, zq float32 [B, g, K] target /
    draft logits on the retained support, verified int32 [B] (support index of the verified
    first token). Returns (J [B], grad [B, g, K], w [B, g]) as float64."""
    zp = np.ascontiguousarray(zp, dtype=np.float32)
    zq = np.ascontiguousarray(zq, dtype=np.float32)
    B, g, K = zp.shape
    v = _i32(np.asarray(verified, dtype=np.int32).reshape(-1))
    J = np.zeros(B, np.float64)
    grad = np.zeros((B, g, K), np.float64)
    w = np.zeros((B, g), np.float64)
    f = _L().eo_kd_loss
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, C.c_double,
                  C.c_void_p, C.c_void_p, C.c_void_p]
    _check(f(B, g, K, _p(zp), _p(zq), _p(v), float(T), float(beta), _p(J), _p(grad), _p(w)), "kd_loss")
    return J, grad, w


class Arc:
    """N1: the oracle ARC dynamic buffer (eo_arc_*), one instance = one cache state."""

    def __init__(self, c: int, *, p0: int = 128, b1cap: int = 256, b2cap: int = 256, min_res: int = 8,
                 warmup: int = 50):
        L = _L()
        L.eo_arc_size.restype = C.c_size_t
        self._buf = C.create_string_buffer(int(L.eo_arc_size()))
        L.eo_arc_init.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        _check(L.eo_arc_init(self._buf, c, p0, b1cap, b2cap, min_res, warmup), "arc_init")
        self.c = c

    def touch(self, token: int, step: int) -> bool:
        f = _L().eo_arc_touch
        f.argtypes = [C.c_void_p, C.c_int32, C.c_int64]
        return bool(f(self._buf, int(token), int(step)))

    def admit(self, tokens, step: int) -> list:
        t = _i32(np.asarray(tokens, dtype=np.int32).reshape(-1))
        ev = np.zeros(max(1, t.size), np.int32)
        ne = C.c_int(0)
        f = _L().eo_arc_admit
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_void_p, C.c_void_p]
        _check(f(self._buf, _p(t), int(t.size), int(step), _p(ev), C.byref(ne)), "arc_admit")
        return ev[:ne.value].tolist()

    def state(self) -> dict:
        out = np.zeros(5 + 4 * 4096, np.int32)
        f = _L().eo_arc_state
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        _check(f(self._buf, _p(out), int(out.size)), "arc_state")
        n1, n2, nb1, nb2, p = (int(x) for x in out[:5])
        o = 5
        lists = []
        for n in (n1, n2, nb1, nb2):
            lists.append(out[o:o + n].tolist())
            o += n
        return dict(T1=lists[0], T2=lists[1], B1=lists[2], B2=lists[3], p=p)

    def members(self) -> list:
        s = self.state()
        return sorted(s["T1"] + s["T2"])


def subset_update(S, remove, add):
    """N1: S' = sort((S minus remove) union add) (eo_subset_update)."""
    S, r, a = (_i32(np.asarray(x, dtype=np.int32).reshape(-1)) for x in (S, remove, add))
    out = np.zeros(S.size + a.size, np.int32)
    n = C.c_int(0)
    f = _L().eo_subset_update
    f.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    _check(f(_p(S), int(S.size), _p(r), int(r.size), _p(a), int(a.size), _p(out), C.byref(n)), "subset_update")
    return out[:n.value].copy()
