"""GPU parity of N2: evospec_verify_chain vs oracle.verify_chain.

Integer results (accepted count, emitted tokens) must match bit-exactly on the
same inputs and the same uniforms; both sides decide in fp64 (the sums run in a
different order, so a mismatch needs a uniform within ~1e-15 relative of a
decision boundary -- never hit by these seeded cases). Full Llama-3 vocabulary
(V = 128,256), the paper's horizon g = 6, a 36,864-id restricted draft
distribution, both greedy (T = 0) and sampling modes.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_27390_b200 as es  # noqa: E402

DEV = "cuda:0"


def problem(seed, V=128256, g=6, n_S=36864, inv_temp=1.0, s_range=0):
    """Seeded verification inputs (synth.verify_problem: target logits, subset, draft
    distribution on it, proposals drawn from the draft, uniforms)."""
    # the ABI's inv_temp is fp32: both sides take that value
    return synth.verify_problem(seed, V=V, g=g, n_S=n_S, inv_temp=float(np.float32(inv_temp)), s_range=s_range)


def run_gpu(P, greedy, ctx=None):
    ctx = ctx or es.Context(V=P["V"], d=64, w_dtype=torch.bfloat16, h_dtype=torch.bfloat16, max_subset=1, max_rows=1,
                            max_k=1, max_sem=1)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(DEV)
    tok, n = ctx.verify_chain(t(P["z"]), t(P["x"]), subset=t(P["S"]), draft_probs=t(P["q"]),
                              inv_temp=P["inv_temp"], greedy=greedy, u=t(P["u"]), w=t(P["w"]))
    torch.cuda.synchronize()
    return tok.cpu().numpy(), int(n.item()), ctx.get_flags()


def check(P, greedy):
    ref_tok, ref_n = oracle.verify_chain(P["z"], P["x"], P["S"], P["q"], inv_temp=P["inv_temp"], greedy=greedy,
                                         u=P["u"], w=P["w"])
    tok, n, flags = run_gpu(P, greedy)
    assert flags == 0
    assert n == ref_n
    np.testing.assert_array_equal(tok[:n + 1], ref_tok)
    assert np.all(tok[n + 1:] == -1)
    return n


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("greedy", [False, True])
def test_verify_full_vocab(seed, greedy):
    check(problem(seed, inv_temp=1.0 if seed % 2 == 0 else 1 / 0.7), greedy)


def test_verify_all_accepted_and_first_rejected():
    P = problem(11)
    P["u"][:] = 0.0                       # every proposal accepted -> the bonus draw from p_g
    assert check(P, False) == P["x"].size
    P = problem(12)
    P["u"][:] = np.nextafter(1.0, 0.0)    # rejected wherever p < q (draws from the residual)
    check(P, False)


def test_verify_greedy_argmax_chain():
    P = problem(13)
    am = np.argmax(P["z"], axis=1).astype(np.int32)
    P["x"] = am[:-1].copy()
    assert check(P, True) == P["x"].size
    P["x"][2] = (P["x"][2] + 1) % P["V"]
    assert check(P, True) == 2


@pytest.mark.parametrize("V,g,n_S", [(1000, 1, 10), (4099, 3, 4099), (77, 0, 5), (50000, 9, 333)])
def test_verify_odd_shapes(V, g, n_S):
    P = problem(20 + V % 7, V=V, g=g, n_S=n_S)
    check(P, False)
    check(P, True)


def test_verify_proposal_outside_support_flags():
    P = problem(30, V=2000, g=2, n_S=100)
    P["x"][0] = np.setdiff1d(np.arange(P["V"]), P["S"])[0]
    tok, n, flags = run_gpu(P, False)
    assert n == 0 and tok[0] == -1 and flags & 0x1


@pytest.mark.parametrize("greedy", [False, True])
def test_verify_subset_slice_beyond_smem(greedy):
    """A subset concentrated in the first eighth of the vocabulary: the first CTA of
    each 8-CTA cluster holds 12,000 > 8,192 subset entries, more than its shared-memory
    slice (kVerSCap), so the residual walk takes the global binary-search path."""
    for seed in (40, 41):
        check(problem(seed, n_S=12000, s_range=128256 // 8), greedy)
