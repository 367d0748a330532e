"""Config Bt timing aid: ragged LM head (64 sequences x 10 rows, static 32768,
dyn_b ~ U[256, 4096]) and the batched build (B scans), device-timed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_27390_b200 as es
import synth

V, d, B, n_b, k = 128256, 4096, 64, 10, 10
W = synth.matrix(0, V, d, 0.02, "bf16")
Wd = torch.from_numpy(W.view(np.int16)).view(torch.bfloat16).cuda()
H = synth.matrix(1, B * n_b, d, 1.0, "bf16")
Hd = torch.from_numpy(H.view(np.int16)).view(torch.bfloat16).cuda()
rng = np.random.default_rng(2)
perm = rng.permutation(V)
static = np.sort(perm[:32768]).astype(np.int32)
pool = perm[32768:]
sizes = rng.integers(256, 4097, B)
dyn = np.concatenate([np.sort(rng.choice(pool, n, replace=False)) for n in sizes]).astype(np.int32)
d_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
h_off = [n_b * b for b in range(B + 1)]
ctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=V, max_rows=B * n_b,
                 max_k=k, max_sem=8192)
ctx.prepare_weights(Wd)
sd, dd, od = (torch.from_numpy(x).cuda() for x in (static, dyn, d_off))
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for it in range(12):
    flush.fill_(it)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.subset_logits_topk_ragged(Wd, Hd, h_off, sd, dd, od, int(sizes.max()), k)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
t = float(np.median(ts[2:]))
alg = (32768 + int(sizes.sum())) * d * 2 + H.nbytes
print(f"ragged Bt: {t:.1f} us  tokens/s {B * n_b / t * 1e6:.3e}  alg bytes {alg / 1e6:.1f} MB -> {alg / t / 1e3:.0f} GB/s")


def timed(fn, n=8):
    ts = []
    for it in range(n):
        flush.fill_(it)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts[2:]))


ctx.set_timing(True)
ctx.subset_logits_topk_ragged(Wd, Hd, h_off, sd, dd, od, int(sizes.max()), k)
torch.cuda.synchronize()
print("stage breakdown (ms, summed over launches):", ctx.read_stats())
ctx.set_timing(False)
z = torch.zeros(B + 1, dtype=torch.int32, device="cuda")
print("static only:", timed(lambda: ctx.subset_logits_topk_ragged(Wd, Hd, h_off, sd, dd, z, 0, k)))
print("dyn only:", timed(lambda: ctx.subset_logits_topk_ragged(Wd, Hd, h_off, None, dd, od, int(sizes.max()), k)))
nS = torch.tensor([32768], dtype=torch.int32, device="cuda")
print("plain 128-row call on static:", timed(lambda: ctx.subset_logits_topk(Wd, Hd[:128], sd, nS, 32768, k)))
print("plain 60-row call on static:", timed(lambda: ctx.subset_logits_topk(Wd, Hd[:60], sd, nS, 32768, k)))
# batched build, 8 sequences (each one E scan)
Bb = 8
Q = synth.matrix(3, Bb, d, 1.0, "bf16")
Qd = torch.from_numpy(Q.view(np.int16)).view(torch.bfloat16).cuda()
row_ptr, col, _ = synth.csr_graph(4, V, 32.0)
seeds = synth.seed_ids(5, V, 10 * Bb)
args = (Wd, Qd, sd, torch.from_numpy(seeds).cuda(), [10 * b for b in range(Bb + 1)],
        torch.from_numpy(row_ptr).cuda(), torch.from_numpy(col).cuda())
for it in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx.build_subset_batched(*args, n_sem=8192, n_dyn=4096)
    e1.record()
    torch.cuda.synchronize()
print(f"batched build B={Bb}: {e0.elapsed_time(e1) * 1e3:.1f} us ({e0.elapsed_time(e1) * 1e3 / Bb:.1f} us / sequence)")
