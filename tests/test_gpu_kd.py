"""GPU parity of N3: evospec_kd_loss vs oracle.kd_loss.

The kernel computes in fp32, the oracle in fp64: loss |d| <= 1e-5 (1 + |J|),
gradient |d| <= 1e-5, weights relative 1e-5. Shapes: the paper's horizon
gamma = 6 and buffer size B = 32, supports of 64 and 1000
logits (K_logit is not given: reading K2), T_kd in {1, 2}, beta in {0, 0.3}.
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


@pytest.mark.parametrize("B,g,K,T,beta", [(32, 6, 64, 1.0, 0.3), (32, 6, 1000, 2.0, 0.3), (5, 1, 7, 1.0, 0.0),
                                          (3, 32, 100, 1.0, 0.7)])
def test_kd_loss(B, g, K, T, beta):
    rng = np.random.default_rng(B * 1000 + K)
    zp = (rng.normal(size=(B, g, K)) * 2.0).astype(np.float32)
    zq = (zp + rng.normal(size=(B, g, K)) * 0.7).astype(np.float32)
    v = rng.integers(0, K, size=B).astype(np.int32)
    v[0] = int(np.argmax(zp[0, 0]))
    ctx = es.Context(V=1024, d=64, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=1, max_rows=1,
                     max_k=1, max_sem=1)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    J, grad, w = ctx.kd_loss(t(zp), t(zq), t(v), T_kd=T, beta=beta)
    torch.cuda.synchronize()
    Jo, go, wo = oracle.kd_loss(zp, zq, v, T=T, beta=beta)
    J, grad, w = J.cpu().numpy(), grad.cpu().numpy(), w.cpu().numpy()
    assert np.all(np.abs(J - Jo) <= 1e-5 * (1 + np.abs(Jo))), np.abs(J - Jo).max()
    assert np.abs(grad - go).max() <= 1e-5
    np.testing.assert_allclose(w, wo, rtol=1e-5, atol=1e-30)


def test_kd_loss_bad_verified_index_and_minus_inf_target():
    """A verified index outside [0, K) gives that trajectory NaN outputs and raises
    FLAG_BAD_IDS (the others are unaffected); a -inf target logit (p_hat = 0) adds 0 to
    the KL instead of 0 * -inf."""
    rng = np.random.default_rng(77)
    B, g, K = 4, 3, 50
    zp = (rng.normal(size=(B, g, K)) * 2.0).astype(np.float32)
    zq = (zp + rng.normal(size=(B, g, K)) * 0.7).astype(np.float32)
    zp[2, 1, 5] = -np.inf
    v = rng.integers(0, K, size=B).astype(np.int32)
    ctx = es.Context(V=1024, d=64, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=1, max_rows=1,
                     max_k=1, max_sem=1)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    J, _, _ = ctx.kd_loss(t(zp), t(zq), t(v), T_kd=1.0, beta=0.3)
    torch.cuda.synchronize()
    assert ctx.get_flags() == 0
    assert np.all(np.isfinite(J.cpu().numpy()))
    zp2 = zp.copy()
    zp2[2, 1, 5] = -1e30   # (the oracle's stand-in for the -inf target logit: p_hat underflows to 0)
    Jo, _, _ = oracle.kd_loss(zp2, zq, v, T=1.0, beta=0.3)
    assert np.all(np.abs(J.cpu().numpy() - Jo) <= 1e-5 * (1 + np.abs(Jo)))
    v_bad = v.copy()
    v_bad[1] = K
    J, _, _ = ctx.kd_loss(t(zp), t(zq), t(v_bad), T_kd=1.0, beta=0.3)
    torch.cuda.synchronize()
    J = J.cpu().numpy()
    assert np.isnan(J[1]) and np.all(np.isfinite(J[[0, 2, 3]]))
    assert ctx.get_flags() & es.FLAG_BAD_IDS
