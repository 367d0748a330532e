"""Phase trace of the H-on-lanes LM-head kernel (lmh_hl.cu) + finalisation
(profiling aid): per-CTA globaltimer stamps, us relative to the earliest CTA start.

  TRACE_NS=36864 python tools/trace_hl.py
"""
import os
import statistics
import sys

os.environ["EVOSPEC_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_27390_b200 as es

V, d, n_h, k = 128256, int(os.environ.get("TRACE_D", "4096")), 60, 10
torch.manual_seed(0)
Wd = (torch.randn(V, d, device="cuda") * 0.02).to(torch.bfloat16)
Hd = torch.randn(n_h, d, device="cuda").to(torch.bfloat16)
ctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=V, max_rows=n_h, max_k=k)
ctx.prepare_weights(Wd)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
names = ["start", "prod_done", "mma_done", "t0_ready", "t0_folded", "tlast_ready", "stored", "end"]
for n_S in [int(x) for x in os.environ.get("TRACE_NS", "8192,36864").split(",")]:
    S = np.sort(np.random.default_rng(11).permutation(V)[:n_S]).astype(np.int32)
    Sd = torch.from_numpy(S).cuda()
    nd = torch.tensor([n_S], dtype=torch.int32, device="cuda")
    evs = []
    for it in range(8):
        if not os.environ.get("TRACE_NOFLUSH"): flush.fill_(it)
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
    t0 = tr[:, 0][tr[:, 0] > 0].min()
    rel = (tr - t0) / 1e3
    print(f"n_S={n_S}: LM head + finalize median {statistics.median(times[2:]):.1f} us (events)")
    for j, n in enumerate(names):
        col = rel[:, j][tr[:, j] > 0]
        if col.size:
            print(f"   {n:12s} min {col.min():7.1f}  med {np.median(col):7.1f}  max {col.max():7.1f}  (n={col.size})")
    frel = (fin[:, :7] - t0) / 1e3
    for j, n in enumerate(["fin_start", "fin_hnorm", "fin_B1", "fin_filter", "fin_runs", "fin_rescore", "fin_end"]):
        col = frel[:, j][fin[:, j] > 0]
        if col.size:
            print(f"   {n:12s} min {col.min():7.1f}  med {np.median(col):7.1f}  max {col.max():7.1f}")
    print("   ncand per row: mean", fin[:, 7].mean(), "max", fin[:, 7].max())
    clk = ctx.read_trace(296 * 8 + 48 + 16)[296 * 8 + 48:].astype(np.int64)
    if clk[0] > 0:
        print("   CTA0 warp0 epilogue clock64 (cycles from tfull): ",
              {i: int(clk[i] - clk[0]) for i in range(1, 16) if clk[i] > 0})
    g0 = ctx.read_trace(296 * 8 + 48 + 32)[296 * 8 + 48 + 16:].astype(np.float64)
    if g0[0] > 0:
        print("   CTA0 (us from its start):", {n: round((g0[i] - tr[0, 0]) / 1e3, 2) for i, n in enumerate(
            ["setup", "pdl_wait", "prod_kb0", "prod_kb8", "prod_kb32", "mma_kb0", "mma_kb8", "mma_kb32"]) if g0[i] > 0})
