"""Phase trace of the subset builder (union kernel) on the llama config (profiling aid)."""
import os
import statistics
import sys

os.environ["EVOSPEC_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_27390_b200 as es
import synth

c = synth.CONFIGS["llama"]
V, d = c["V"], c["d"]
W = synth.matrix(0, V, d, 0.02, "bf16")
q = synth.matrix(2, 1, d, 1.0, "bf16")[0]
static = synth.static_ids(3, V, c["n_static"])
rp, col, _ = synth.csr_graph(4, V, c["avg_deg"])
seeds = synth.seed_ids(5, V, 10)
T = lambda a: (torch.from_numpy(a.view(np.int16)).view(torch.bfloat16) if a.dtype == np.uint16 else torch.from_numpy(a)).cuda()
Wd, qd, sd, rpd, cold, seedd = T(W), T(q), T(static), T(rp), T(col), T(seeds)
ctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=V, max_rows=60, max_k=10,
                 max_sem=8192)
ctx.set_timing(True)
for it in range(6):
    ids, n, _, _ = ctx.build_subset(Wd, qd, sd, seedd, rpd, cold, n_sem=8192, n_dyn=4096)
torch.cuda.synchronize()
st = ctx.read_stats()
print({k: round(v / max(1, st["calls"][k]) * 1e3, 1) for k, v in st["ms"].items() if st["calls"][k]})
tr = ctx.read_trace()[2 * 148 * 8:2 * 148 * 8 + 7].astype(np.float64)
names = ["start", "loaded", "S_sem", "gs", "G/graph", "formation", "end"]
print("union phases (us from start):", {n: round((t - tr[0]) / 1e3, 1) for n, t in zip(names, tr)})
tr2 = ctx.read_trace(2 * 148 * 8 + 40)[2 * 148 * 8 + 17:2 * 148 * 8 + 40].astype(np.float64)   # [7] = selection start
print("multi-select: setup", round((tr2[8] - tr2[7]) / 1e3, 2) if tr2[8] > 0 else None,
      "later passes (us):", [round((tr2[8 + i] - tr2[7 + i]) / 1e3, 2) for i in range(1, 8) if tr2[8 + i] > 0 and i < 9],
      "n_cand", int(tr2[6]))
print("setup detail (us from start): count loop", round((tr2[17] - tr2[7]) / 1e3, 2), "scan+minmax", round((tr2[18] - tr2[7]) / 1e3, 2),
      "pass0 hist done", round((tr2[19] - tr2[7]) / 1e3, 2), "pass0 end", round((tr2[8] - tr2[7]) / 1e3, 2),
      "marked", round((tr2[20] - tr2[7]) / 1e3, 2), "ranked", round((tr2[21] - tr2[7]) / 1e3, 2))
