"""GPU parity of N1's incremental subset update (evospec_subset_update) against
oracle.subset_update: bit-exact ids, the llama subset size, an ARC-driven sequence
of OOV events (max 32 insertions per event) applied incrementally equals the
oracle's result event by event."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2605_27390_b200 as es  # noqa: E402

DEV = "cuda:0"
t = lambda a: torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.int32))).to(DEV)


def gpu_update(S, rem, add):
    out, n = es.subset_update(t(S), t(rem), t(add))
    torch.cuda.synchronize()
    return out.cpu().numpy(), int(n.item())


@pytest.mark.parametrize("case", ["random", "empty_delta", "remove_all", "extremes"])
def test_subset_update(case):
    rng = np.random.default_rng(5)
    V = 128256
    S = np.sort(rng.choice(V, 36864, replace=False)).astype(np.int32)
    free = np.setdiff1d(np.arange(V), S)
    if case == "random":
        rem, add = np.sort(rng.choice(S, 32, replace=False)), np.sort(rng.choice(free, 32, replace=False))
    elif case == "empty_delta":
        rem, add = S[:0], S[:0]
    elif case == "remove_all":
        S = S[:100]
        rem, add = S.copy(), np.sort(rng.choice(free, 7, replace=False))
    else:
        S = S[(S > 0) & (S < V - 1)]
        rem, add = S[[0, -1]], np.array([0, V - 1], np.int32)
    out, n = gpu_update(S, rem, add)
    ref = oracle.subset_update(S, rem, add)
    assert n == ref.size
    np.testing.assert_array_equal(out, ref)


def test_arc_driven_incremental_updates():
    """Static core + an ARC dynamic buffer (capacity 256, paper defaults): each OOV event's
    admissions / evictions applied to the device subset incrementally equal the sorted
    static u members after every event."""
    rng = np.random.default_rng(9)
    V = 128256
    static = np.sort(rng.choice(V, 32768, replace=False)).astype(np.int32)
    pool = np.setdiff1d(np.arange(V), static)
    arc = es.Arc(256)
    S = static.copy()
    for step in range(120):
        toks = [int(x) for x in rng.choice(pool[:2000], int(rng.integers(1, 33)), replace=False)]
        before = set(arc.members())
        ev = arc.admit(toks, step)
        after = set(arc.members())
        add = np.array(sorted(after - before), np.int32)
        rem = np.array(sorted(before - after), np.int32)
        # evicted = the members that left, plus tokens of this event admitted and evicted again
        assert set(rem.tolist()) <= set(ev) and set(ev) - set(rem.tolist()) <= set(toks)
        S, n = gpu_update(S, rem, add)
        np.testing.assert_array_equal(S, np.union1d(static, np.array(sorted(after), np.int32)))


def test_contract_violation_is_flagged_not_corrupting():
    """A removed id that is not in the subset, or an added id that is already kept,
    violates the header's contract: the kernel raises FLAG_BAD_IDS and never writes
    outside out[] (a guard buffer past it stays intact)."""
    rng = np.random.default_rng(11)
    V = 50000
    S = np.sort(rng.choice(V, 4000, replace=False)).astype(np.int32)
    free = np.setdiff1d(np.arange(V), S)
    for rem, add in ((np.sort(rng.choice(free, 5, replace=False)), free[:0]),          # removed not in S
                     (S[:0], np.sort(np.concatenate([S[:3], free[:2]])))):            # added already kept
        n_new = S.size - rem.size + add.size
        buf = torch.full((n_new + 64,), -7, dtype=torch.int32, device=DEV)
        n = torch.zeros(1, dtype=torch.int32, device=DEV)
        flags = torch.zeros(1, dtype=torch.int32, device=DEV)
        es.subset_update(t(S), t(rem), t(add), out=(buf[:max(1, n_new)], n), flags=flags)
        torch.cuda.synchronize()
        assert int(flags.item()) & es.FLAG_BAD_IDS
        assert np.all(buf[n_new:].cpu().numpy() == -7)
    # a conforming call leaves the flag clear
    flags = torch.zeros(1, dtype=torch.int32, device=DEV)
    es.subset_update(t(S), t(S[:4]), t(free[:4]), flags=flags)
    torch.cuda.synchronize()
    assert int(flags.item()) == 0
