"""Timeline of one draft step (profiling aid): union stamps and LM-head per-CTA stamps
(globaltimer, us from the union's start) -- shows how much of the LM head overlaps the
union in the two-list mode (EVOSPEC_OVERLAP=1)."""
import os
import sys

os.environ["EVOSPEC_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_27390_b200 as es
import synth

c = synth.CONFIGS["llama"]
V, d = c["V"], c["d"]
W = torch.from_numpy(synth.matrix(0, V, d, 0.02, "bf16").view(np.int16)).view(torch.bfloat16).cuda()
H = torch.from_numpy(synth.matrix(1, 60, d, 1.0, "bf16").view(np.int16)).view(torch.bfloat16).cuda()
q = torch.from_numpy(synth.matrix(2, 1, d, 1.0, "bf16")[0].view(np.int16)).view(torch.bfloat16).cuda()
static = torch.from_numpy(synth.static_ids(3, V, c["n_static"])).cuda()
rp, col, _ = synth.csr_graph(4, V, c["avg_deg"])
seeds = torch.from_numpy(synth.seed_ids(5, V, 10)).cuda()
ctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=V, max_rows=60, max_k=10,
                 max_sem=8192)
ctx.prepare_weights(W)
kw = dict(E=W, W_local=W, static_ids=static, csr_row_ptr=torch.from_numpy(rp).cuda(),
          csr_col=torch.from_numpy(col).cuda(), k=10, n_sem=8192, n_dyn=4096)
for _ in range(4):
    ctx.draft_step(q=q, H=H, seeds=seeds, **kw)
torch.cuda.synchronize()
tr = ctx.read_trace(2 * 148 * 8 + 17).astype(np.float64)
lm = tr[:148 * 8].reshape(148, 8)
un = tr[2 * 148 * 8:2 * 148 * 8 + 7]
t0 = un[0]
rel = lambda x: round((x - t0) / 1e3, 1)
print("union: start 0, loaded", rel(un[1]), "sel", rel(un[2]), "end", rel(un[6]))
ok = lm[:, 0] > 0
for j, n in enumerate(["start", "prod_done", "mma_done", "t0_ready", "t0_fold", "t1_ready", "t1_fold", "end"]):
    col_ = lm[ok, j]
    col_ = col_[col_ > 0]
    if col_.size:
        print(f"  lmh {n:9s} min {rel(col_.min()):7.1f} med {rel(np.median(col_)):7.1f} max {rel(col_.max()):7.1f}")
fin = tr[148 * 8:148 * 8 + 60 * 8].reshape(60, 8)
print("  finalize start", rel(fin[:, 0].min()), "end", rel(fin[:, 6].max()))
