"""Stress test of the semantic scan's TMA ring (compute-sanitizer
racecheck reports read/write hazards between the ring's bulk-copy refills and the
slab warps' reads, which DESIGN §5 reads as the tool not modelling the mbarrier-
ordered WAR against the async proxy). Here the claim is tested instead of argued:

- every score of the production ring (3 stages) over the full Llama vocabulary and
  over a d = 256 index (one slab warp, ~100 stages per CTA: the configuration
  racecheck flagged) equals the oracle's fp64 score within 1e-12 relative, for many
  queries back to back (a refill overwriting unread data corrupts whole rows: errors
  of order 1, not 1e-16);
- a 2-stage ring (EVOSPEC_SCAN_RING2=1, test-only: every slot is refilled while the
  previous stage is still being computed -- the tightest release / refill reuse)
  produces bit-identical scores to the 3-stage ring (same summation order).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import synth, paper_2605_27390_b200 as es
V, d, nq = {V}, {d}, {nq}
bf = torch.bfloat16
W = synth.matrix(90 + d, V, d, 0.02, "bf16")
Wd = torch.from_numpy(W.view(np.int16)).view(bf).cuda()
ctx = es.Context(V=V, d=d, w_dtype=bf, h_dtype=bf, max_subset=400, max_rows=1, max_k=1, max_sem=64, max_seeds=16)
static = torch.arange(0, 300, dtype=torch.int32, device="cuda")
out = []
for i in range(nq):
    q = synth.matrix(1000 + i, 1, d, 1.0, "bf16")[0]
    qd = torch.from_numpy(q.view(np.int16)).view(bf).cuda()
    ctx.build_subset(Wd, qd, static, None, None, None, n_sem=64, n_dyn=50)
    out.append(ctx.last_scores(V).cpu().numpy())
np.save({path!r}, np.stack(out))
print("scan ok")
"""


def run_scan(tmp_path, V, d, nq, ring2):
    path = str(tmp_path / f"scores_{V}_{d}_{int(ring2)}.npy")
    env = dict(os.environ)
    if ring2:
        env["EVOSPEC_SCAN_RING2"] = "1"
    else:
        env.pop("EVOSPEC_SCAN_RING2", None)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, V=V, d=d, nq=nq, path=path)], env=env,
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0 and "scan ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    return np.load(path)


@pytest.mark.parametrize("V,d,nq", [(128256, 4096, 6), (131072, 256, 24)])
def test_scan_ring_against_oracle_and_two_stage_ring(tmp_path, V, d, nq):
    import synth
    s3 = run_scan(tmp_path, V, d, nq, ring2=False)
    s2 = run_scan(tmp_path, V, d, nq, ring2=True)
    np.testing.assert_array_equal(s2, s3)   # bit-identical: same order, no corrupted slot
    W = synth.matrix(90 + d, V, d, 0.02, "bf16")
    for i in (0, nq - 1):
        q = synth.matrix(1000 + i, 1, d, 1.0, "bf16")[0]
        ref = oracle.sem_scores(W, q)
        np.testing.assert_allclose(s3[i], ref, rtol=1e-12, atol=1e-13)
