"""Config Bt breakdown (profiling aid): the ragged LM head's static block and its
dynamic blocks timed apart with the context's stage timers (which serialise the
launches), L2 flushed before each call."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_27390_b200 as es
import synth

V, d, k, B, n_b = 128256, 4096, 10, 64, 10
W = synth.matrix(0, V, d, 0.02, "bf16")
Wd = torch.from_numpy(W.view(np.int16)).view(torch.bfloat16).cuda()
del W
rng = np.random.default_rng(21)
perm = rng.permutation(V)
static = np.sort(perm[:32768]).astype(np.int32)
pool = perm[32768:]
sizes = rng.integers(256, 4097, B)
dyn = np.concatenate([np.sort(rng.choice(pool, n, replace=False)) for n in sizes]).astype(np.int32)
d_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
h_off = [n_b * b for b in range(B + 1)]
H = synth.matrix(22, B * n_b, d, 1.0, "bf16")
Hd = torch.from_numpy(H.view(np.int16)).view(torch.bfloat16).cuda()
ctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=V, max_rows=B * n_b,
                 max_k=k, max_sem=1, max_seeds=1)
ctx.prepare_weights(Wd)
sd, dd, od = (torch.from_numpy(x).cuda() for x in (static, dyn, d_off))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def run(tag, n_static_use, timing):
    ctx.set_timing(timing)
    s0 = ctx.read_stats()
    out = None
    evs = []
    for it in range(8):
        flush.fill_(it & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = ctx.subset_logits_topk_ragged(Wd, Hd, h_off, sd[:n_static_use], dd, od, int(sizes.max()), k, out=out)
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
    t = statistics.median([a.elapsed_time(b) * 1e3 for a, b in evs[3:]])
    s1 = ctx.read_stats()
    calls = {kk: s1["calls"][kk] - s0["calls"][kk] for kk in s1["calls"]}
    ms = {kk: s1["ms"][kk] - s0["ms"][kk] for kk in s1["ms"]}
    print(tag, "us", round(t, 1), {kk: (calls[kk], round(ms[kk] / 8 * 1e3, 1)) for kk in ms if calls[kk]}
          if timing else "", flush=True)


run("full", 32768, False)
run("full(timed stages)", 32768, True)
run("dynamic only", 0, False)
run("dynamic only(timed)", 0, True)
