"""N1 product ARC (libevospec.so evospec_arc_*, host code -- no GPU needed) against the
oracle ARC (oracle.Arc), state for state after every operation, on random traces with
the paper's safeguards (min residency, warm-up) and small capacities that
force evictions, ghost hits and p adaptation."""
import numpy as np
import pytest

import oracle


@pytest.mark.parametrize("seed,c,p0,b1,b2,mr,wu", [(0, 16, 8, 10, 7, 0, 0), (1, 16, 8, 10, 7, 3, 5),
                                                    (2, 256, 128, 256, 256, 8, 50), (3, 5, 0, 2, 9, 2, 1)])
def test_arc_product_equals_oracle(seed, c, p0, b1, b2, mr, wu):
    import paper_2605_27390_b200 as es
    rng = np.random.default_rng(seed)
    V = 4 * c
    a = es.Arc(c, p0=p0, b1_cap=b1, b2_cap=b2, min_residency=mr, warmup_events=wu)
    o = oracle.Arc(c, p0=p0, b1cap=b1, b2cap=b2, min_res=mr, warmup=wu)
    for step in range(600):
        if rng.random() < 0.4:
            t = int(rng.integers(V))
            assert a.touch(t, step) == o.touch(t, step)
        else:
            toks = [int(t) for t in rng.choice(V, int(rng.integers(1, min(33, V))), replace=False)]
            assert a.admit(toks, step) == o.admit(toks, step)
        assert a.state() == o.state()
    a.close()


def test_arc_bad_arguments():
    import paper_2605_27390_b200 as es
    with pytest.raises(es.EvospecError):
        es.Arc(0)


@pytest.mark.parametrize("seed,c", [(4, 16), (5, 256)])
def test_arc_admit_delta_is_the_net_membership_change(seed, c):
    """evospec_arc_admit_delta (the N1 OOV event's ARC step): the returned (added,
    removed) equal the oracle ARC's member sets after minus before / before minus after
    for the same event -- including tokens admitted and evicted within one event (in
    neither list) -- and the two ARCs stay state-identical."""
    import paper_2605_27390_b200 as es
    rng = np.random.default_rng(seed)
    V = 4 * c
    a = es.Arc(c, p0=c // 2, b1_cap=c, b2_cap=c, min_residency=2, warmup_events=3)
    o = oracle.Arc(c, p0=c // 2, b1cap=c, b2cap=c, min_res=2, warmup=3)
    members = lambda st: set(st["T1"]) | set(st["T2"])
    seen_both = False
    for step in range(300):
        toks = sorted(int(t) for t in rng.choice(V, int(rng.integers(1, min(33, V))), replace=False))
        before = members(o.state())
        add, rem = a.admit_delta(toks, step)
        o.admit(toks, step)
        after = members(o.state())
        assert add == sorted(after - before)
        assert rem == sorted(before - after)
        seen_both |= any(t not in after and t not in before for t in toks)
        assert a.state() == o.state()
    if c <= 16:
        assert seen_both   # the small cache exercised admitted-and-evicted-within-an-event
    a.close()
