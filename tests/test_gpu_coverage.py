"""GPU parity of N4: evospec_coverage vs oracle.coverage.

Recall@k is an integer count decided on the fp32 logits (the top-k order is
exact): bit-exact. The covered mass is an fp64 sum in a different order:
relative tolerance 1e-12. Full Llama-3 vocabulary, the llama subset size,
the paper's Recall@{10, 50, 100} (App. E) plus k = 1 and 256.
"""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_27390_b200 as es  # noqa: E402

DEV = "cuda:0"
KS = [1, 10, 50, 100, 256]


def run(z, S, ks, inv_temp=1.0):
    ctx = es.Context(V=z.shape[1], d=64, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=1,
                     max_rows=1, max_k=1, max_sem=1)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    m, r = ctx.coverage(t(z), t(S), t(np.asarray(ks, np.int32)), inv_temp=inv_temp)
    torch.cuda.synchronize()
    return m.cpu().numpy(), r.cpu().numpy()


@pytest.mark.parametrize("seed,integer", [(0, False), (1, False), (2, True)])
def test_coverage_full_vocab(seed, integer):
    rng = np.random.default_rng(seed)
    V, n = 128256, 8
    z = (rng.integers(-3, 4, size=(n, V)) if integer else rng.normal(size=(n, V)) * 1.28).astype(np.float32)
    S = np.sort(rng.choice(V, 36864, replace=False)).astype(np.int32)
    it = float(np.float32(1.0 if seed != 1 else 1 / 0.7))   # the ABI's inv_temp is fp32: same value both sides
    m, r = run(z, S, KS, it)
    mo, ro = oracle.coverage(z, S, KS, inv_temp=it)
    np.testing.assert_allclose(m, mo, rtol=1e-12, atol=0)
    np.testing.assert_array_equal(r, ro)


def test_coverage_edges():
    rng = np.random.default_rng(3)
    V = 5000
    z = rng.normal(size=(3, V)).astype(np.float32)
    z[1, :] = 0.5                                # all tied: top-k = the k smallest ids
    full = np.arange(V, dtype=np.int32)
    m, r = run(z, full, [1, 7, 1024])               # (k <= 1024, the header bound)
    assert np.all(np.abs(m - 1.0) < 1e-12) and np.all(r == 1.0)
    S = np.arange(3, 40, dtype=np.int32)
    m, r = run(z, S, [1, 3, 5, 40])
    mo, ro = oracle.coverage(z, S, [1, 3, 5, 40])
    np.testing.assert_allclose(m, mo, rtol=1e-12)
    np.testing.assert_array_equal(r, ro)
    assert r[1, 0] == 0.0 and r[1, 3] == (40 - 3) / 40


def test_coverage_bad_k_entries():
    """Every k outside [1, min(V, 1024)] gives NaN for that k (the others stay exact)
    and raises FLAG_BAD_IDS -- including a non-positive k next to a valid maximum."""
    rng = np.random.default_rng(4)
    V = 5000
    z = rng.normal(size=(2, V)).astype(np.float32)
    S = np.sort(rng.choice(V, 900, replace=False)).astype(np.int32)
    ctx = es.Context(V=V, d=64, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=1, max_rows=1,
                     max_k=1, max_sem=1)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    m, r = ctx.coverage(t(z), t(S), t(np.asarray([10, 0, -3, 50], np.int32)))
    torch.cuda.synchronize()
    r = r.cpu().numpy()
    _, ro = oracle.coverage(z, S, [10, 50])
    assert np.all(np.isnan(r[:, 1:3]))
    np.testing.assert_array_equal(r[:, [0, 3]], ro)
    assert ctx.get_flags() & es.FLAG_BAD_IDS
