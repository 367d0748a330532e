"""Thin Python binding over libevospec.so (include/evospec.h).

Argument marshalling only: every step of the EvoSpec subset LM-head path runs
in the library's CUDA kernels. torch supplies device memory, streams and
process groups. There is no CPU fallback: importing this package without the
built library, or calling it without a CUDA device, raises.

Names follow the C ABI: build_subset, subset_logits_topk, merge_shards,
draft_step (PAPER.md Eq. projection, Eq. vocab_union P:88-93,
runtime formation P:458).
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libevospec.so")

BF16, FP32 = 0, 1
OK, EINPUT, EINVARIANT, ECUDA, ENCCL, ENOMEM = 0, 2, 3, 10, 11, 12
FLAG_BAD_IDS, FLAG_UNCERTIFIED, FLAG_SELECT_OVERFLOW, FLAG_BUDGET = 0x1, 0x2, 0x4, 0x8

EXPORTED = [
    "evospec_create", "evospec_destroy", "evospec_status_string", "evospec_last_error",
    "evospec_version", "evospec_prepare_weights", "evospec_get_flags",
    "evospec_comm_unique_id", "evospec_comm_init", "evospec_build_subset",
    "evospec_last_semantic", "evospec_subset_logits_topk", "evospec_merge_shards",
    "evospec_draft_step", "evospec_set_timing", "evospec_read_stats", "evospec_read_trace",
    "evospec_build_subset_batched", "evospec_subset_logits_topk_ragged", "evospec_subset_logits_topk_merged",
    "evospec_verify_chain", "evospec_coverage", "evospec_kd_loss",
    "evospec_arc_create", "evospec_arc_destroy", "evospec_arc_touch", "evospec_arc_admit", "evospec_arc_state",
    "evospec_subset_update",
    "evospec_sync_status",
    "evospec_build_local_candidates", "evospec_build_subset_from_candidates",
    "evospec_arc_admit_delta", "evospec_oov_event_begin", "evospec_oov_event_end", "evospec_last_scores",
]

STAGES = ["scan", "select", "union", "lmh", "finalize", "merge", "copy"]


class EvospecError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"evospec status {status}: {detail}")
        self.status = status


class Config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "V", "d", "w_dtype", "h_dtype", "n_shards", "shard_rank", "max_subset", "max_rows",
        "max_k", "max_sem", "max_seeds", "max_ctx", "debug_checks")]


class BuildParams(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "n_sem", "n_graph_sem_seeds", "per_seed", "ctx_min_count", "n_ctx_max", "n_dyn")]


class Stats(C.Structure):
    _fields_ = [("launches", C.c_int64), ("calls", C.c_int32 * 7), ("stage_ms", C.c_float * 7)]


class StepIO(C.Structure):
    _fields_ = [
        ("E", C.c_void_p), ("n_e_rows", C.c_int64),
        ("W_local", C.c_void_p), ("n_w_rows", C.c_int64),
        ("static_ids", C.c_void_p), ("n_static", C.c_int32),
        ("csr_row_ptr", C.c_void_p), ("csr_col", C.c_void_p),
        ("build", BuildParams),
        ("n_h", C.c_int32), ("k", C.c_int32), ("inv_temp", C.c_float),
        ("q", C.c_void_p), ("H", C.c_void_p),
        ("seeds", C.c_void_p), ("n_seed", C.c_int32),
        ("ctx_ids", C.c_void_p), ("n_ctx", C.c_int32),
        ("out_ids", C.c_void_p), ("out_vals", C.c_void_p), ("out_lse", C.c_void_p),
        ("out_probs", C.c_void_p), ("host_io", C.c_int32),
    ]


_lib = None


def lib() -> C.CDLL:
    """Loads libevospec.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2605_27390_b200._build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        sig = {
            "evospec_create": ([C.POINTER(vp), C.POINTER(Config), C.c_int], i32),
            "evospec_destroy": ([vp], i32),
            "evospec_status_string": ([i32], C.c_char_p),
            "evospec_last_error": ([], C.c_char_p),
            "evospec_version": ([], C.c_char_p),
            "evospec_prepare_weights": ([vp, vp, i64, vp], i32),
            "evospec_get_flags": ([vp, C.POINTER(i32), C.c_int, vp], i32),
            "evospec_comm_unique_id": ([vp], i32),
            "evospec_comm_init": ([vp, vp], i32),
            "evospec_build_subset": ([vp, vp, i64, vp, vp, i32, vp, i32, vp, vp, vp, i32,
                                      C.POINTER(BuildParams), vp, vp, vp, vp, vp], i32),
            "evospec_build_local_candidates": ([vp, vp, i64, vp, i32, vp, vp, vp], i32),
            "evospec_build_subset_from_candidates": ([vp, vp, vp, i32, vp, i32, vp, i32, vp, vp, vp, i32,
                                                      C.POINTER(BuildParams), vp, vp, vp, vp, vp], i32),
            "evospec_last_semantic": ([vp, vp, i32, vp], i32),
            "evospec_subset_logits_topk": ([vp, vp, i64, vp, i32, vp, vp, i32, i32, C.c_float,
                                            vp, vp, vp, vp, vp, vp], i32),
            "evospec_merge_shards": ([vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp], i32),
            "evospec_verify_chain": ([vp, vp, i32, i32, vp, vp, i32, vp, C.c_float, i32, vp, vp, vp, vp, vp], i32),
            "evospec_coverage": ([vp, vp, i32, i32, vp, i32, C.c_float, vp, i32, vp, vp, vp], i32),
            "evospec_kd_loss": ([vp, i32, i32, i32, vp, vp, vp, C.c_float, C.c_float, vp, vp, vp, vp], i32),
            "evospec_arc_create": ([vp, i32, i32, i32, i32, i32, i32], i32),
            "evospec_arc_destroy": ([vp], i32),
            "evospec_arc_touch": ([vp, i32, i64], i32),
            "evospec_arc_admit": ([vp, vp, i32, i64, vp, vp], i32),
            "evospec_arc_state": ([vp, vp, i32, vp], i32),
            "evospec_arc_admit_delta": ([vp, vp, i32, i64, vp, vp, vp, vp], i32),
            "evospec_last_scores": ([vp, vp, i64, vp], i32),
            "evospec_oov_event_begin": ([vp, vp, i64, vp, vp, i32, vp, i32, vp, vp, C.POINTER(BuildParams), vp], i32),
            "evospec_oov_event_end": ([vp, vp, i64, vp, i32, vp, vp, vp, vp, vp, vp, vp], i32),
            "evospec_subset_update": ([vp, i32, vp, i32, vp, i32, vp, vp, vp, vp], i32),
            "evospec_sync_status": ([vp, vp], i32),
            "evospec_draft_step": ([vp, C.POINTER(StepIO), vp], i32),
            "evospec_set_timing": ([vp, C.c_int], i32),
            "evospec_read_stats": ([vp, C.POINTER(Stats)], i32),
            "evospec_read_trace": ([vp, vp, i32], i32),
            "evospec_build_subset_batched": ([vp, vp, i64, vp, i32, vp, i32, vp, vp, vp, vp, vp, vp,
                                              C.POINTER(BuildParams), vp, vp, vp], i32),
            "evospec_subset_logits_topk_ragged": ([vp, vp, i64, vp, vp, i32, vp, i32, vp, vp, i32, i32,
                                                   C.c_float, vp, vp, vp, vp, vp], i32),
            "evospec_subset_logits_topk_merged": ([vp, vp, i64, vp, i32, vp, vp, i32, i32, C.c_float,
                                                   vp, vp, vp, vp, vp, vp, vp], i32),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(st: int):
    if st != OK:
        raise EvospecError(st, lib().evospec_last_error().decode())


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def version() -> str:
    return lib().evospec_version().decode()


def _dtype_code(t) -> int:
    import torch
    if t == torch.bfloat16:
        return BF16
    if t == torch.float32:
        return FP32
    raise TypeError(f"unsupported dtype {t} (bf16 or fp32)")


class Arc:
    """N1: the dynamic buffer's ARC (evospec_arc_*; host-side, no GPU needed). Paper defaults:
    capacity 256, p0 128, ghost caps 256 / 256, min residency 8 steps, warm-up 50 events."""

    def __init__(self, capacity: int = 256, *, p0: int = 128, b1_cap: int = 256, b2_cap: int = 256,
                 min_residency: int = 8, warmup_events: int = 50):
        h = C.c_void_p()
        _check(lib().evospec_arc_create(C.byref(h), capacity, p0, b1_cap, b2_cap, min_residency, warmup_events))
        self._h = h
        self.capacity = capacity

    _h = None   # (set only once creation succeeded)

    def close(self):
        if self._h:
            lib().evospec_arc_destroy(self._h)
            self._h = None

    __del__ = close

    def touch(self, token: int, step: int) -> bool:
        return bool(lib().evospec_arc_touch(self._h, int(token), int(step)))

    def admit(self, tokens, step: int) -> list:
        import numpy as np
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32).reshape(-1))
        ev = np.zeros(max(1, t.size), np.int32)
        ne = C.c_int32(0)
        _check(lib().evospec_arc_admit(self._h, t.ctypes.data_as(C.c_void_p), int(t.size), int(step),
                                       ev.ctypes.data_as(C.c_void_p), C.byref(ne)))
        return ev[:ne.value].tolist()

    def admit_delta(self, tokens, step: int):
        """One OOV event as the net membership change: (added, removed), ascending."""
        import numpy as np
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32).reshape(-1))
        add = np.zeros(max(1, t.size), np.int32)
        rem = np.zeros(max(1, t.size), np.int32)
        na, nr = C.c_int32(0), C.c_int32(0)
        _check(lib().evospec_arc_admit_delta(self._h, t.ctypes.data_as(C.c_void_p), int(t.size), int(step),
                                             add.ctypes.data_as(C.c_void_p), C.byref(na),
                                             rem.ctypes.data_as(C.c_void_p), C.byref(nr)))
        return add[:na.value].tolist(), rem[:nr.value].tolist()

    def state(self) -> dict:
        import numpy as np
        out = np.zeros(5 + 4 * max(self.capacity, 1) + 2 * 65536, np.int32)
        n = C.c_int32(0)
        _check(lib().evospec_arc_state(self._h, out.ctypes.data_as(C.c_void_p), int(out.size), C.byref(n)))
        n1, n2, nb1, nb2, p = (int(x) for x in out[:5])
        o, lists = 5, []
        for k in (n1, n2, nb1, nb2):
            lists.append(out[o:o + k].tolist())
            o += k
        return dict(T1=lists[0], T2=lists[1], B1=lists[2], B2=lists[3], p=p)

    def members(self) -> list:
        s = self.state()
        return sorted(s["T1"] + s["T2"])


def subset_update(subset, removed, added, *, out=None, flags=None, stream=None):
    """N1: out = sort((subset minus removed) union added) on the device (evospec_subset_update).
    All int32 device tensors, removed / added sorted. flags: optional int32 [1] device tensor,
    OR-ed with FLAG_BAD_IDS on a contract violation. Returns (out, n_out)."""
    import torch
    n_new = subset.numel() - removed.numel() + added.numel()
    if out is None:
        out = (torch.empty(max(1, n_new), dtype=torch.int32, device=subset.device),
               torch.empty(1, dtype=torch.int32, device=subset.device))
    o, n = out
    _check(lib().evospec_subset_update(_ptr(subset), int(subset.numel()), _ptr(removed), int(removed.numel()),
                                       _ptr(added), int(added.numel()), _ptr(o), _ptr(n),
                                       _ptr(flags) if flags is not None else None, _stream(stream)))
    return o[:n_new], n


class DraftStep:
    """A prepared evospec_draft_step (Context.prepare_draft_step): one ctypes call per run()."""

    def __init__(self, ctx, kw, out, stream):
        self.ctx, self.out, self._keep = ctx, out, (kw, out)
        io = StepIO()
        E, W, st = kw["E"], kw["W_local"], kw["static_ids"]
        io.E, io.n_e_rows = E.data_ptr(), E.shape[0]
        io.W_local, io.n_w_rows = W.data_ptr(), W.shape[0]
        io.static_ids, io.n_static = st.data_ptr(), st.numel()
        rp, col = kw.get("csr_row_ptr"), kw.get("csr_col")
        io.csr_row_ptr = None if rp is None else rp.data_ptr()
        io.csr_col = None if col is None else col.data_ptr()
        io.build = BuildParams(kw["n_sem"], kw.get("n_graph_sem_seeds", 10), kw.get("per_seed", 8),
                               kw.get("ctx_min_count", 0), kw.get("n_ctx_max", 0), kw["n_dyn"])
        H, q, seeds, cx = kw["H"], kw["q"], kw.get("seeds"), kw.get("ctx_ids")
        io.n_h, io.k, io.inv_temp = H.shape[0], kw["k"], float(kw.get("inv_temp", 1.0))
        io.q, io.H = q.data_ptr(), H.data_ptr()
        io.seeds = None if seeds is None else seeds.data_ptr()
        io.n_seed = 0 if seeds is None else seeds.numel()
        io.ctx_ids = None if cx is None else cx.data_ptr()
        io.n_ctx = 0 if cx is None else cx.numel()
        io.out_ids, io.out_vals, io.out_lse, io.out_probs = (t.data_ptr() for t in out)
        io.host_io = int(not H.is_cuda)
        self._io, self._ref = io, C.byref(io)
        self._st = _stream(stream)
        self._fn = lib().evospec_draft_step

    def run(self):
        st = self._fn(self.ctx._h, self._ref, self._st)
        if st != OK:
            _check(st)
        return self.out


class Context:
    """Owns an evospec_ctx (device workspace + optional NCCL communicator)."""

    def __init__(self, *, V: int, d: int, w_dtype, h_dtype, n_shards: int = 1, shard_rank: int = 0,
                 max_subset: int, max_rows: int, max_k: int = 64, max_sem: int = 8192,
                 max_seeds: int = 64, max_ctx: int = 0, debug_checks: bool = False, device: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("evospec needs a CUDA device (B200, sm_100a); there is no CPU path")
        self.cfg = Config(V, d, _dtype_code(w_dtype), _dtype_code(h_dtype), n_shards, shard_rank,
                          max_subset, max_rows, max_k, max_sem, max_seeds, max_ctx, int(debug_checks))
        self.device = device
        h = C.c_void_p()
        _check(lib().evospec_create(C.byref(h), C.byref(self.cfg), device))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib().evospec_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- setup
    def prepare_weights(self, W, stream=None):
        _check(lib().evospec_prepare_weights(self._h, _ptr(W), W.shape[0], _stream(stream)))

    def set_timing(self, enable: bool = True):
        _check(lib().evospec_set_timing(self._h, int(enable)))

    def read_stats(self) -> dict:
        st = Stats()
        _check(lib().evospec_read_stats(self._h, C.byref(st)))
        return dict(launches=st.launches,
                    calls={n: st.calls[i] for i, n in enumerate(STAGES)},
                    ms={n: st.stage_ms[i] for i, n in enumerate(STAGES)})

    def read_trace(self, n: int = 2 * 148 * 8 + 16):
        """Flat int64 profiling stamps (EVOSPEC_TRACE=1); see include/evospec.h."""
        import numpy as np
        out = np.zeros(n, dtype=np.int64)
        _check(lib().evospec_read_trace(self._h, out.ctypes.data_as(C.c_void_p), out.size))
        return out

    def sync_status(self, stream=None):
        """evospec_sync_status: synchronizes the stream; raises EvospecError(EINVARIANT)
        when an invariant flag (bad ids, budget) is set."""
        _check(lib().evospec_sync_status(self._h, _stream(stream)))

    def get_flags(self, clear: bool = True, stream=None) -> int:
        out = C.c_int32(0)
        _check(lib().evospec_get_flags(self._h, C.byref(out), int(clear), _stream(stream)))
        return out.value

    def comm_init(self, group=None):
        """Creates the library's NCCL communicator; the 128-byte unique id is
        broadcast from rank 0 over the given torch.distributed group."""
        import torch.distributed as dist
        from . import dist as esd
        buf = (C.c_char * 128)()
        if dist.get_rank(group) == 0:
            _check(lib().evospec_comm_unique_id(buf))
        raw = esd.broadcast_bytes(bytes(buf), group)
        _check(lib().evospec_comm_init(self._h, C.c_char_p(raw)))

    # ---- a1-a4
    def build_subset(self, E, q, static_ids, seed_ids, csr_row_ptr, csr_col, *, n_sem: int,
                     n_dyn: int, n_graph_sem_seeds: int = 10, per_seed: int = 8, ctx_ids=None,
                     ctx_min_count: int = 0, n_ctx_max: int = 0, out=None, stream=None):
        """Returns (ids, n_dev, local_ids, local_n_dev): device tensors; n stays on the device."""
        import torch
        dev = E.device
        cap = static_ids.numel() + n_dyn
        if out is None:
            out = (torch.empty(max(cap, 1), dtype=torch.int32, device=dev),
                   torch.empty(1, dtype=torch.int32, device=dev),
                   torch.empty(max(cap, 1), dtype=torch.int32, device=dev),
                   torch.empty(1, dtype=torch.int32, device=dev))
        ids, n, lids, ln = out
        p = BuildParams(n_sem, n_graph_sem_seeds, per_seed, ctx_min_count, n_ctx_max, n_dyn)
        n_ctx = 0 if ctx_ids is None else ctx_ids.numel()
        _check(lib().evospec_build_subset(
            self._h, _ptr(E), E.shape[0], _ptr(q), _ptr(static_ids), static_ids.numel(),
            _ptr(seed_ids) if seed_ids is not None else None,
            0 if seed_ids is None else seed_ids.numel(),
            _ptr(csr_row_ptr), _ptr(csr_col), _ptr(ctx_ids), n_ctx, C.byref(p),
            _ptr(ids), _ptr(n), _ptr(lids), _ptr(ln), _stream(stream)))
        return ids, n, lids, ln

    def oov_event_begin(self, E, q, static_ids, seed_ids, csr_row_ptr, csr_col, *, n_sem: int = 10,
                        n_dyn: int = 32, n_graph_sem_seeds: int = 10, per_seed: int = 8, stream=None):
        """N1: enqueue an OOV event's candidate formation on the context's side stream
        (evospec_oov_event_begin) and return at once."""
        p = BuildParams(n_sem, n_graph_sem_seeds, per_seed, 0, 0, n_dyn)
        self._oov_cap = n_dyn
        _check(lib().evospec_oov_event_begin(
            self._h, _ptr(E), E.shape[0], _ptr(q), _ptr(static_ids), static_ids.numel(),
            _ptr(seed_ids) if seed_ids is not None else None, 0 if seed_ids is None else seed_ids.numel(),
            _ptr(csr_row_ptr), _ptr(csr_col), C.byref(p), _stream(stream)))

    def oov_event_end(self, arc, step: int, subset, n: int, *, out=None, stream=None):
        """N1: admit the event's candidates into `arc` and update the subset on the device
        (evospec_oov_event_end). subset: the current sorted V_t ([>= n] int32 device).
        Returns (out [n'] device, n_out device, added list, removed list)."""
        import numpy as np
        import torch
        cap = getattr(self, "_oov_cap", 32)
        if out is None:
            out = (torch.empty(n + cap, dtype=torch.int32, device=subset.device),
                   torch.empty(1, dtype=torch.int32, device=subset.device))
        o, no = out
        add = np.zeros(max(1, cap), np.int32)
        rem = np.zeros(max(1, cap), np.int32)
        na, nr = C.c_int32(0), C.c_int32(0)
        _check(lib().evospec_oov_event_end(self._h, arc._h, int(step), _ptr(subset), int(n), _ptr(o), _ptr(no),
                                           add.ctypes.data_as(C.c_void_p), C.byref(na),
                                           rem.ctypes.data_as(C.c_void_p), C.byref(nr), _stream(stream)))
        n_new = n - nr.value + na.value
        return o[:n_new], no, add[:na.value].tolist(), rem[:nr.value].tolist()

    def build_local_candidates(self, E_local, q, n_sem: int, out=None, stream=None):
        """Sharded build, step 1 (evospec_build_local_candidates): this shard's exact
        semantic top-n_sem over its rows of E. Returns (s fp64 [n_sem], ids int32 [n_sem])."""
        import torch
        dev = E_local.device
        if out is None:
            out = (torch.empty(n_sem, dtype=torch.float64, device=dev), torch.empty(n_sem, dtype=torch.int32, device=dev))
        cs, ci = out
        _check(lib().evospec_build_local_candidates(self._h, _ptr(E_local), E_local.shape[0], _ptr(q), int(n_sem),
                                                    _ptr(cs), _ptr(ci), _stream(stream)))
        return cs, ci

    def build_subset_from_candidates(self, cand_s, cand_id, static_ids, seed_ids, csr_row_ptr, csr_col, *,
                                     n_sem: int, n_dyn: int, n_graph_sem_seeds: int = 10, per_seed: int = 8,
                                     ctx_ids=None, ctx_min_count: int = 0, n_ctx_max: int = 0, out=None,
                                     stream=None):
        """Sharded build, step 2 (evospec_build_subset_from_candidates): the R shards'
        candidates stacked in rank order -> (ids, n_dev, local_ids, local_n_dev), as
        build_subset."""
        import torch
        dev = cand_s.device
        cap = static_ids.numel() + n_dyn
        if out is None:
            out = (torch.empty(max(cap, 1), dtype=torch.int32, device=dev),
                   torch.empty(1, dtype=torch.int32, device=dev),
                   torch.empty(max(cap, 1), dtype=torch.int32, device=dev),
                   torch.empty(1, dtype=torch.int32, device=dev))
        ids, n, lids, ln = out
        p = BuildParams(n_sem, n_graph_sem_seeds, per_seed, ctx_min_count, n_ctx_max, n_dyn)
        n_ctx = 0 if ctx_ids is None else ctx_ids.numel()
        _check(lib().evospec_build_subset_from_candidates(
            self._h, _ptr(cand_s), _ptr(cand_id), cand_s.numel(), _ptr(static_ids), static_ids.numel(),
            _ptr(seed_ids) if seed_ids is not None else None, 0 if seed_ids is None else seed_ids.numel(),
            _ptr(csr_row_ptr), _ptr(csr_col), _ptr(ctx_ids), n_ctx, C.byref(p),
            _ptr(ids), _ptr(n), _ptr(lids), _ptr(ln), _stream(stream)))
        return ids, n, lids, ln

    def build_subset_batched(self, E, Q, static_ids, seed_ids, seed_offsets, csr_row_ptr, csr_col, *,
                             n_sem: int, n_dyn: int, n_graph_sem_seeds: int = 10, per_seed: int = 8,
                             ctx_ids=None, ctx_offsets=None, ctx_min_count: int = 0, n_ctx_max: int = 0,
                             out=None, stream=None):
        """Q [B, d]; seed_offsets / ctx_offsets: host int sequences [B+1].
        Returns (dyn_ids [B*n_dyn], dyn_offsets [B+1]) device tensors (per-sequence
        sorted dynamic lists, compacted)."""
        import torch
        B = Q.shape[0]
        dev = E.device
        if out is None:
            out = (torch.empty(max(B * n_dyn, 1), dtype=torch.int32, device=dev),
                   torch.empty(B + 1, dtype=torch.int32, device=dev))
        dyn, offs = out
        so = (C.c_int32 * (B + 1))(*[int(x) for x in seed_offsets])
        co = None if ctx_offsets is None else (C.c_int32 * (B + 1))(*[int(x) for x in ctx_offsets])
        p = BuildParams(n_sem, n_graph_sem_seeds, per_seed, ctx_min_count, n_ctx_max, n_dyn)
        _check(lib().evospec_build_subset_batched(
            self._h, _ptr(E), E.shape[0], _ptr(Q), B, _ptr(static_ids), static_ids.numel(),
            _ptr(seed_ids), C.cast(so, C.c_void_p), _ptr(csr_row_ptr), _ptr(csr_col), _ptr(ctx_ids),
            None if co is None else C.cast(co, C.c_void_p), C.byref(p), _ptr(dyn), _ptr(offs),
            _stream(stream)))
        return dyn, offs

    def last_scores(self, n: int, stream=None):
        """The last full-index scan's fp64 scores of rows [0, n) (evospec_last_scores)."""
        import torch
        out = torch.empty(max(n, 1), dtype=torch.float64, device=f"cuda:{self.device}")
        _check(lib().evospec_last_scores(self._h, _ptr(out), int(n), _stream(stream)))
        return out[:n]

    def last_semantic(self, n: int, stream=None):
        import torch
        out = torch.empty(max(n, 1), dtype=torch.int32, device=f"cuda:{self.device}")
        _check(lib().evospec_last_semantic(self._h, _ptr(out), n, _stream(stream)))
        return out[:n]

    # ---- a5-a7
    def subset_logits_topk(self, W_local, H, subset, n_subset_dev, n_subset_max: int, k: int,
                           inv_temp: float = 1.0, logits_out=None, out=None, stream=None):
        """Returns this shard's triple (topk_ids, topk_vals, row_max, row_sumexp)."""
        import torch
        n_h = H.shape[0]
        dev = H.device
        if out is None:
            out = (torch.empty((n_h, k), dtype=torch.int32, device=dev),
                   torch.empty((n_h, k), dtype=torch.float32, device=dev),
                   torch.empty(n_h, dtype=torch.float32, device=dev),
                   torch.empty(n_h, dtype=torch.float32, device=dev))
        ids, vals, m, s = out
        _check(lib().evospec_subset_logits_topk(
            self._h, _ptr(W_local), W_local.shape[0], _ptr(H), n_h, _ptr(subset), _ptr(n_subset_dev),
            n_subset_max, k, float(inv_temp), _ptr(ids), _ptr(vals), _ptr(m), _ptr(s),
            _ptr(logits_out), _stream(stream)))
        return ids, vals, m, s

    def subset_logits_topk_merged(self, W_local, H, subset, n_subset_dev, n_subset_max: int, k: int,
                                  inv_temp: float = 1.0, out=None, stream=None):
        """Single shard (R = 1): returns (ids, vals, lse, probs) -- merge_shards' outputs,
        written by the LM head's finalisation."""
        import torch
        n_h = H.shape[0]
        dev = H.device
        if out is None:
            out = (torch.empty((n_h, k), dtype=torch.int32, device=dev),
                   torch.empty((n_h, k), dtype=torch.float32, device=dev),
                   torch.empty(n_h, dtype=torch.float32, device=dev),
                   torch.empty((n_h, k), dtype=torch.float32, device=dev))
        ids, vals, lse, probs = out
        _check(lib().evospec_subset_logits_topk_merged(
            self._h, _ptr(W_local), W_local.shape[0], _ptr(H), n_h, _ptr(subset), _ptr(n_subset_dev),
            n_subset_max, k, float(inv_temp), _ptr(ids), _ptr(vals), _ptr(lse), _ptr(probs), None, None,
            _stream(stream)))
        return ids, vals, lse, probs

    def subset_logits_topk_ragged(self, W_local, H, h_offsets, static_ids, dyn_ids, dyn_offsets, max_dyn: int,
                                  k: int, inv_temp: float = 1.0, out=None, stream=None):
        """h_offsets: host ints [B+1]; dyn_offsets: device int32 [B+1]. Returns the
        per-row triple (topk_ids, topk_vals, row_max, row_sumexp) over static u dyn_b."""
        import torch
        B = len(h_offsets) - 1
        n_rows = int(h_offsets[-1])
        dev = H.device
        if out is None:
            out = (torch.empty((n_rows, k), dtype=torch.int32, device=dev),
                   torch.empty((n_rows, k), dtype=torch.float32, device=dev),
                   torch.empty(n_rows, dtype=torch.float32, device=dev),
                   torch.empty(n_rows, dtype=torch.float32, device=dev))
        ids, vals, m, s = out
        ho = (C.c_int32 * (B + 1))(*[int(x) for x in h_offsets])
        n_static = 0 if static_ids is None else static_ids.numel()
        _check(lib().evospec_subset_logits_topk_ragged(
            self._h, _ptr(W_local), W_local.shape[0], _ptr(H), C.cast(ho, C.c_void_p), B, _ptr(static_ids),
            n_static, _ptr(dyn_ids), _ptr(dyn_offsets), int(max_dyn), k, float(inv_temp), _ptr(ids), _ptr(vals),
            _ptr(m), _ptr(s), _stream(stream)))
        return ids, vals, m, s

    # ---- a8
    def merge_shards(self, ids, vals, m, s, *, n_h: int, k: int, out=None, stream=None):
        """Returns (ids, vals, lse, probs) merged over the shards."""
        import torch
        dev = ids.device
        if out is None:
            out = (torch.empty((n_h, k), dtype=torch.int32, device=dev),
                   torch.empty((n_h, k), dtype=torch.float32, device=dev),
                   torch.empty(n_h, dtype=torch.float32, device=dev),
                   torch.empty((n_h, k), dtype=torch.float32, device=dev))
        oi, ov, ol, op = out
        _check(lib().evospec_merge_shards(self._h, n_h, k, _ptr(ids), _ptr(vals), _ptr(m), _ptr(s),
                                          _ptr(oi), _ptr(ov), _ptr(ol), _ptr(op), _stream(stream)))
        return oi, ov, ol, op

    # ---- N2: verification of a draft chain
    def verify_chain(self, z, proposals, *, subset=None, draft_probs=None, inv_temp: float = 1.0,
                     greedy: bool, u=None, w=None, out=None, stream=None):
        """Lossless verification (evospec_verify_chain). z: fp32 [g+1, V] target logits,
        proposals int32 [g], subset int32 sorted [n_S], draft_probs fp32 [g, n_S], u / w fp64
        [g] / [g+1] uniforms (device tensors). Returns (tokens int32 [g+1], n_accepted int32 [1])."""
        import torch
        g = z.shape[0] - 1
        if out is None:
            out = (torch.empty(g + 1, dtype=torch.int32, device=z.device),
                   torch.empty(1, dtype=torch.int32, device=z.device))
        tok, nacc = out
        n_S = 0 if subset is None else int(subset.numel())
        _check(lib().evospec_verify_chain(self._h, _ptr(z), int(z.shape[1]), g, _ptr(proposals), _ptr(subset), n_S,
                                          _ptr(draft_probs), float(inv_temp), int(bool(greedy)), _ptr(u), _ptr(w),
                                          _ptr(tok), _ptr(nacc), _stream(stream)))
        return tok, nacc

    # ---- N4: coverage of the active vocabulary
    def coverage(self, z, subset, ks, *, inv_temp: float = 1.0, out=None, stream=None):
        """Covered mass and Recall@k of `subset` (sorted int32, device) against the target rows
        z (fp32 [n_rows, V], device); ks int32 device tensor. Returns (mass fp64 [n_rows],
        recall fp64 [n_rows, len(ks)])."""
        import torch
        n_rows, V = z.shape
        if out is None:
            out = (torch.empty(n_rows, dtype=torch.float64, device=z.device),
                   torch.empty((n_rows, max(1, ks.numel())), dtype=torch.float64, device=z.device))
        mass, rec = out
        _check(lib().evospec_coverage(self._h, _ptr(z), n_rows, V, _ptr(subset), int(subset.numel()),
                                      float(inv_temp), _ptr(ks), int(ks.numel()), _ptr(mass), _ptr(rec),
                                      _stream(stream)))
        return mass, rec[:, :ks.numel()]

    # ---- N3: curriculum-weighted distillation objective
    def kd_loss(self, target_logits, draft_logits, verified, *, T_kd: float = 1.0, beta: float = 0.3,
                out=None, stream=None):
        """Eq. lora_objective with the curriculum weights (evospec_kd_loss). target_logits /
        draft_logits fp32 [B, g, K], verified int32 [B] (device). Returns (loss [B],
        grad [B, g, K], weights [B, g]), fp32."""
        import torch
        B, g, K = target_logits.shape
        if out is None:
            dev = target_logits.device
            out = (torch.empty(B, dtype=torch.float32, device=dev),
                   torch.empty((B, g, K), dtype=torch.float32, device=dev),
                   torch.empty((B, g), dtype=torch.float32, device=dev))
        loss, grad, w = out
        _check(lib().evospec_kd_loss(self._h, B, g, K, _ptr(target_logits), _ptr(draft_logits), _ptr(verified),
                                     float(T_kd), float(beta), _ptr(loss), _ptr(grad), _ptr(w), _stream(stream)))
        return loss, grad, w

    # ---- whole step
    def draft_step(self, *, E, W_local, static_ids, csr_row_ptr, csr_col, q, H, seeds, k: int,
                   n_sem: int, n_dyn: int, n_graph_sem_seeds: int = 10, per_seed: int = 8,
                   inv_temp: float = 1.0, ctx_ids=None, ctx_min_count: int = 0, n_ctx_max: int = 0,
                   out=None, stream=None):
        """One draft step. q/H/seeds/ctx and `out` may be pinned HOST tensors
        (then the call stages them through device buffers) or device tensors."""
        import torch
        host_io = not H.is_cuda
        n_h = H.shape[0]
        if out is None:
            # one contiguous block [ids | vals | lse | probs]: with host I/O the library
            # then reads the step's outputs back with a single copy
            kw = dict(pin_memory=True) if host_io else dict(device=H.device)
            hk = n_h * k
            blk = torch.empty(3 * hk + n_h, dtype=torch.int32, **kw)
            out = (blk[:hk].view(n_h, k), blk[hk:2 * hk].view(torch.float32).view(n_h, k),
                   blk[2 * hk:2 * hk + n_h].view(torch.float32),
                   blk[2 * hk + n_h:].view(torch.float32).view(n_h, k))
        io = StepIO()
        io.E, io.n_e_rows = E.data_ptr(), E.shape[0]
        io.W_local, io.n_w_rows = W_local.data_ptr(), W_local.shape[0]
        io.static_ids, io.n_static = static_ids.data_ptr(), static_ids.numel()
        io.csr_row_ptr = None if csr_row_ptr is None else csr_row_ptr.data_ptr()
        io.csr_col = None if csr_col is None else csr_col.data_ptr()
        io.build = BuildParams(n_sem, n_graph_sem_seeds, per_seed, ctx_min_count, n_ctx_max, n_dyn)
        io.n_h, io.k, io.inv_temp = n_h, k, float(inv_temp)
        io.q, io.H = q.data_ptr(), H.data_ptr()
        io.seeds = None if seeds is None else seeds.data_ptr()
        io.n_seed = 0 if seeds is None else seeds.numel()
        io.ctx_ids = None if ctx_ids is None else ctx_ids.data_ptr()
        io.n_ctx = 0 if ctx_ids is None else ctx_ids.numel()
        io.out_ids, io.out_vals, io.out_lse, io.out_probs = (t.data_ptr() for t in out)
        io.host_io = int(host_io)
        _check(lib().evospec_draft_step(self._h, C.byref(io), _stream(stream)))
        return out

    def prepare_draft_step(self, *, out=None, stream=None, **kw):
        """A reusable draft step for a serving loop: the I/O descriptor is marshalled
        once; each `run()` is one evospec_draft_step call on the same buffers (the
        caller refills q / H / seeds in place, e.g. pinned host tensors, between
        steps). Returns a DraftStep whose `.out` holds the outputs."""
        out = self.draft_step(out=out, stream=stream, **kw)   # one step: also builds / validates the I/O
        return DraftStep(self, kw, out, stream)


