"""GEMV LM head (n_H = 1) on the llama subset: event-timed calls (profiling aid for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_27390_b200 as es
import synth

V, d, k = 128256, 4096, 10
n_h = int(os.environ.get("NH", "1"))
n_S = int(os.environ.get("NS", "36864"))
W = synth.matrix(0, V, d, 0.02, "bf16")
Wd = torch.from_numpy(W.view(np.int16)).view(torch.bfloat16).cuda()
del W
H = synth.matrix(1, n_h, d, 1.0, "bf16")
Hd = torch.from_numpy(H.view(np.int16)).view(torch.bfloat16).cuda()
S = np.sort(np.random.default_rng(11).permutation(V)[:n_S]).astype(np.int32)
Sd = torch.from_numpy(S).cuda()
nd = torch.tensor([n_S], dtype=torch.int32, device="cuda")
ctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=V, max_rows=max(n_h, 8), max_k=k)
ctx.prepare_weights(Wd)
ts = []
for it in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.subset_logits_topk_merged(Wd, Hd, Sd, nd, n_S, k)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
print("n_h", n_h, "median us", float(np.median(ts[5:])))
