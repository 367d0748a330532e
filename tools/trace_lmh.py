"""Phase trace of the tcgen05 LM-head kernel on the llama config (profiling aid).

Runs subset_logits_topk on n_S = 36,864 gathered rows, n_h = 60, with
EVOSPEC_TRACE=1 and prints per-CTA globaltimer phases (us, relative to the
earliest CTA start), (one run).
"""
import os
import statistics
import sys

os.environ["EVOSPEC_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_27390_b200 as es
import synth

V, d, k = 128256, 4096, 10
n_h = int(os.environ.get("TRACE_NH", "60"))
n_S = int(os.environ.get("TRACE_NS", "36864"))
W = synth.matrix(0, V, d, 0.02, "bf16")
H = synth.matrix(1, n_h, d, 1.0, "bf16")
Wd = torch.from_numpy(W.view(np.int16)).view(torch.bfloat16).cuda()
Hd = torch.from_numpy(H.view(np.int16)).view(torch.bfloat16).cuda()
S = np.sort(np.random.default_rng(int(os.environ.get("TRACE_SEED", "11"))).permutation(V)[:n_S]).astype(np.int32)
Sd = torch.from_numpy(S).cuda()
nd = torch.tensor([n_S], dtype=torch.int32, device="cuda")
ctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=V, max_rows=n_h, max_k=k,
                 max_sem=8192)
ctx.prepare_weights(Wd)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
names = ["start", "prod_done", "mma_done", "t0_ready", "t0_fold", "t1_ready", "t1_fold", "end"]
small = torch.from_numpy(S[:256].copy()).cuda()
nsmall = torch.tensor([256], dtype=torch.int32, device="cuda")
# modes: flushed (L2 flushed before the call), warmcode (flushed, then a 256-row call of
# the same kernels so their code is in L2 / the I-caches, then the timed call), steady
# (calls back to back, no flush)
for pf in os.environ.get("TRACE_MODES", "flushed,warmcode,steady").split(","):
    evs = []
    for it in range(8):
        if pf != "steady":
            flush.fill_(it)
        if pf == "warmcode":
            ctx.subset_logits_topk(Wd, Hd, small, nsmall, 256, k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.subset_logits_topk(Wd, Hd, Sd, nd, n_S, k)
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) * 1e3 for a, b in evs]
    full = ctx.read_trace(296 * 8).astype(np.float64).reshape(296, 8)
    tr = full[:148]
    fin = full[148:148 + n_h]
    t0 = tr[:, 0].min()
    rel = (tr - t0) / 1e3
    print(f"PF={pf}: kernel+finalize median {statistics.median(times[2:]):.1f} us")
    for j, n in enumerate(names):
        col = rel[:, j]
        col = col[tr[:, j] > 0]
        if col.size:
            print(f"   {n:10s} min {col.min():7.1f}  med {np.median(col):7.1f}  max {col.max():7.1f}")
    ovf_base = 2 * 148 * 8 + 16 + 32 + 64 + 2 * 148 + 8
    ovf = ctx.read_trace(ovf_base + 296)[ovf_base:].astype(np.int64)
    print("   rows overflowing their candidate buffer: last tile", {int(b): int(ovf[b]) for b in np.nonzero(ovf[:148])[0]},
          "middle tiles", {int(b): int(ovf[148 + b]) for b in np.nonzero(ovf[148:])[0]})
    fold = rel[:, 6] - rel[:, 5]
    slow = np.argsort(-fold)[:6]
    print("   slowest last folds (block: t1_ready -> t1_fold us):", [(int(b), round(fold[b], 1)) for b in slow])
    late = np.argsort(-rel[:, 7])[:8]
    print("   latest CTAs (block: end / prod_done us):", [(int(b), round(rel[b, 7], 1), round(rel[b, 1], 1)) for b in late])
    frel = (fin[:, :7] - t0) / 1e3
    for j, n in enumerate(["fin_start", "fin_hnorm", "fin_B1", "fin_filter", "fin_runs", "fin_rescore", "fin_end"]):
        col = frel[:, j]
        print(f"   {n:10s} min {col.min():7.1f}  med {np.median(col):7.1f}  max {col.max():7.1f}")
    nc, nn = fin[:, 7] % 10000, fin[:, 7] // 10000
    print("   ncand per row: mean", nc.mean(), "max", nc.max(), "| re-scored per row: mean", nn.mean(), "max", nn.max())
    dur = (fin[:, 6] - fin[:, 0]) / 1e3
    slow = np.argsort(-dur)[:6]
    print("   slowest rows (row: us, ncand, re-scored):", [(int(i), round(dur[i], 1), int(nc[i]), int(nn[i])) for i in slow])
    det = ctx.read_trace(296 * 8 + 16 + 32)[296 * 8 + 16:].astype(np.int64)
    if det[0] > 0:
        print("   finalize row 0 clock64 deltas (cycles from slot 0):",
              {i: int(det[i] - det[0]) for i in range(32) if det[i] > 0})
    dd = ctx.read_trace(296 * 8 + 48 + 64)[296 * 8 + 48:].astype(np.int64)
    b = dd[40]
    if b > 0:
        print("   CTA0 last tile clock64 (cycles from tfull): tmem->smem", dd[41] - b, "bar1", dd[42] - b, "bar2", dd[43] - b,
              "par1", dd[44] - b, "bar", dd[45] - b, "par2", dd[46] - b, "cands overflow/ok", dd[48], dd[49])
        print("   phase1 detail (rowstate, pass1 done, pass2 done, stores done):", [int(dd[50 + i] - b) for i in (3, 0, 1, 2)])
        print("   phase1 end per warp (cycles from tfull):", [int(dd[20 + w] - b) for w in range(13)])
        for it in range(5):
            if dd[it * 4] > 0:
                print("     row", it, [int(dd[it * 4 + j] - b) for j in range(4)])
    evs = []
    for it in range(8):
        if pf != "steady":
            flush.fill_(it)
        if pf == "warmcode":
            ctx.subset_logits_topk(Wd, Hd, small, nsmall, 256, k)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.subset_logits_topk_merged(Wd, Hd, Sd, nd, n_S, k)
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    times = [a.elapsed_time(b) * 1e3 for a, b in evs]
    print(f"   merged path: median {statistics.median(times[2:]):.1f} us")
