"""Timeline of one llama draft step (profiling aid): globaltimer stamps of the
scan CTAs, the candidate kernel, the union phases, the LM-head CTAs and the
finalize rows, on one clock, relative to the first scan CTA's start (us).
EVOSPEC_TRACE=1 (the stamps' own cost included)."""
import os
import sys

os.environ["EVOSPEC_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import paper_2605_27390_b200 as es

c, W, H, q, static, row_ptr, col, seeds = bench.make_workload()
bf = torch.bfloat16
T = lambda a: (torch.from_numpy(a.view(np.int16)).view(bf) if a.dtype == np.uint16 else
               torch.from_numpy(np.ascontiguousarray(a))).cuda()
Wd, Hd, qd, sd, rpd, cold, seedd = T(W), T(H), T(q), T(static), T(row_ptr), T(col), T(seeds)
del W
n_h, k = c["n_h"], c["k"]
ctx = es.Context(V=c["V"], d=c["d"], w_dtype=bf, h_dtype=bf, max_subset=c["V"], max_rows=n_h, max_k=k,
                 max_sem=c["n_sem"], max_seeds=32)
ctx.prepare_weights(Wd)
kw = dict(E=Wd, W_local=Wd, static_ids=sd, csr_row_ptr=rpd, csr_col=cold, k=k, n_sem=c["n_sem"], n_dyn=c["n_dyn"],
          n_graph_sem_seeds=c["n_graph_sem_seeds"], per_seed=c["per_seed"])
out = (torch.empty((n_h, k), dtype=torch.int32, device="cuda"), torch.empty((n_h, k), device="cuda"),
       torch.empty(n_h, device="cuda"), torch.empty((n_h, k), device="cuda"))
for it in range(int(os.environ.get("STEPS", "6"))):
    ctx.draft_step(q=qd, H=Hd, seeds=seedd, out=out, **kw)
torch.cuda.synchronize()
N = 148
tr = ctx.read_trace(2 * N * 8 + 112 + 2 * N + 2).astype(np.float64)
lmh = tr[:N * 8].reshape(N, 8)
fin = tr[N * 8:N * 8 + n_h * 8].reshape(n_h, 8)
uni = tr[2 * N * 8:2 * N * 8 + 7]
scan = tr[2 * N * 8 + 112:2 * N * 8 + 112 + 2 * N].reshape(N, 2)
cand = tr[2 * N * 8 + 112 + 2 * N:2 * N * 8 + 112 + 2 * N + 2]
t0 = scan[:, 0].min()
rel = lambda x: (x - t0) / 1e3


def dist(name, col):
    col = col[col > 0]
    if col.size:
        r = rel(col)
        print(f"  {name:22s} min {r.min():7.1f}  med {np.median(r):7.1f}  max {r.max():7.1f}")


print("draft step timeline (us from the first scan CTA start)")
dist("scan start", scan[:, 0])
dist("scan end", scan[:, 1])
dist("cand kernel start", cand[:1])
dist("cand kernel end", cand[1:])
for i, nm in enumerate(["start", "loaded", "S_sem", "gs", "G/graph", "formation", "end"]):
    dist("union " + nm, uni[i:i + 1])
dist("union after wait", tr[2 * N * 8 + 40:2 * N * 8 + 41])
dist("union sbits copied", tr[2 * N * 8 + 41:2 * N * 8 + 42])
dist("union seeds walked", tr[2 * N * 8 + 42:2 * N * 8 + 43])
dist("union cands in (t0)", tr[2 * N * 8 + 43:2 * N * 8 + 44])
print("  union n_cand", int(tr[2 * N * 8 + 23]))
sel = tr[2 * N * 8 + 24:2 * N * 8 + 40]
for i, nm in [(0, "start"), (10, "stats"), (11, "setup"), (12, "hist0"), (1, "pass0"), (2, "pass1"), (13, "marked"),
              (14, "ranked")]:
    dist("  select " + nm, sel[i:i + 1])
for i, nm in enumerate(["start", "prod_done", "mma_done", "t0_ready", "t0_fold", "t1_ready", "t1_fold", "end"]):
    dist("lmh " + nm, lmh[:, i])
for i, nm in enumerate(["start", "hnorm", "B1", "filter", "runs", "rescore", "end"]):
    dist("fin " + nm, fin[:, i])
