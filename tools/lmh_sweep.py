"""LM-head + top-k + merge (subset_logits_topk_merged) vs subset size, L2 flushed,
on device-generated weights (fast to set up; bench.py's sweep uses the seeded synth
weights). Prints one JSON line per n_S. Profiling aid for the LM-head kernels.

  python tools/lmh_sweep.py [--d 4096] [--n 8192,16384,36864,65536,128256] [--iters 20]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2605_27390_b200 as es
    from bench import L2Flush, load_peaks

    ap = argparse.ArgumentParser()
    ap.add_argument("--d", type=int, default=4096)
    ap.add_argument("--V", type=int, default=128256)
    ap.add_argument("--n", default="8192,16384,36864,65536,128256")
    ap.add_argument("--nh", type=int, default=60)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--steady", action="store_true")
    args = ap.parse_args()
    dev = "cuda:0"
    torch.manual_seed(0)
    V, d, nh, k = args.V, args.d, args.nh, args.k
    W = (torch.randn(V, d, device=dev) * 0.02).to(torch.bfloat16)
    H = torch.randn(nh, d, device=dev).to(torch.bfloat16)
    ctx = es.Context(V=V, d=d, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=V, max_rows=nh,
                     max_k=k, device=0)
    ctx.prepare_weights(W)
    flush = L2Flush(dev)
    rng = np.random.default_rng(11)
    peak = load_peaks()["hbm_gbs"]
    for n_S in [int(x) for x in args.n.split(",")]:
        S = torch.from_numpy(np.sort(rng.permutation(V)[:n_S]).astype(np.int32)).to(dev)
        nd = torch.tensor([n_S], dtype=torch.int32, device=dev)
        trip = None
        evs = []
        for it in range(3 + args.iters):
            flush(it)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            trip = ctx.subset_logits_topk_merged(W, H, S, nd, n_S, k, out=trip)
            e1.record()
            evs.append((e0, e1))
        torch.cuda.synchronize()
        ts = [a.elapsed_time(b) * 1e3 for a, b in evs[3:]]
        us = statistics.median(ts)
        nbytes = n_S * d * 2 + nh * d * 2 + n_S * 4
        row = dict(n_S=n_S, d=d, us=round(us, 2), us_min=round(min(ts), 2), frac=round(nbytes / us / 1e3 / peak, 4),
                   flags=ctx.get_flags(clear=True))
        if args.steady:
            for _ in range(3):
                trip = ctx.subset_logits_topk_merged(W, H, S, nd, n_S, k, out=trip)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                trip = ctx.subset_logits_topk_merged(W, H, S, nd, n_S, k, out=trip)
            e1.record()
            torch.cuda.synchronize()
            row["us_steady"] = round(e0.elapsed_time(e1) * 1e3 / 20, 2)
        # spot check of the ids against a dense fp32 recomputation of 4 rows
        ids = trip[0][:4].cpu()
        z = (H[:4].float() @ W[S.long()].float().T)
        ref = S[torch.topk(z, k, dim=1).indices].cpu()
        row["ids_match_fp32_4rows"] = bool((ids == ref).all())
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
