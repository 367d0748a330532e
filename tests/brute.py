"""Pure-Python brute force for tiny vocabularies (V <= 64).

An independent restatement of the plain definitions, used to pin the C
oracle: exact rational arithmetic (fractions.Fraction) for dot products of
exactly-representable inputs, math.fsum for sums of exponentials, Python's
stable sort for every "(-value, id)" ordering. No numpy, no code shared with
oracle/ or the CUDA path.
"""
from __future__ import annotations

import math
from fractions import Fraction


def dot(a, b):
    return sum((Fraction(float(x)) * Fraction(float(y)) for x, y in zip(a, b)), Fraction(0))


def order_desc(values, ids):
    """ids ordered by (-value, id)."""
    return [i for _, i in sorted(zip(values, ids), key=lambda t: (-t[0], t[1]))]


def restricted_softmax(logits, support, inv_temp=1.0):
    """dict id -> prob over the support only (zero mass outside)."""
    z = [float(l) * inv_temp for l in logits]
    m = max(z)
    tot = math.fsum(math.exp(x - m) for x in z)
    return {sid: math.exp(x - m) / tot for sid, x in zip(support, z)}


def full_softmax_conditioned(all_logits, support, inv_temp=1.0):
    """Full-vocab softmax, then conditioned on the support."""
    z = [float(l) * inv_temp for l in all_logits]
    m = max(z)
    e = [math.exp(x - m) for x in z]
    tot_s = math.fsum(e[v] for v in support)
    return {v: e[v] / tot_s for v in support}


def build_subset(E, q, static, seeds, rows, n_sem, n_graph_sem_seeds, per_seed, n_dyn):
    """Formation per Eq. vocab_union + App A.3 + cap.

    rows: dict src -> ordered successor list (already (p desc, id asc)).
    """
    V = len(E)
    scores = [dot(q, E[v]) for v in range(V)]
    sem = order_desc(scores, list(range(V)))[:n_sem]
    G = []
    for g in list(seeds) + sem[:n_graph_sem_seeds]:
        if g not in G:
            G.append(g)
    graph = []
    for g in G:
        graph.extend(rows.get(g, [])[:per_seed])
    dyn = []
    st = set(static)
    for c in list(seeds) + sem + graph:
        if len(dyn) == n_dyn:
            break
        if c in st or c in dyn:
            continue
        dyn.append(c)
    return sorted(st | set(dyn)), sem, dyn


class ArcSim:
    """An independently written simulator of the dynamic buffer's ARC rules (SPEC
    S:288-348 as read in DESIGN.md A1/A2), OrderedDict-based -- used only to
    cross-check the C oracle's list bookkeeping operation for operation."""

    def __init__(self, c, p0, b1cap, b2cap, min_res, warmup):
        from collections import OrderedDict
        self.c, self.p, self.caps, self.min_res, self.warmup = c, max(0, min(c, p0)), (b1cap, b2cap), min_res, warmup
        self.T = [OrderedDict(), OrderedDict()]   # token -> admission step, LRU first
        self.B = [OrderedDict(), OrderedDict()]   # ghosts
        self.events = 0

    def touch(self, t):
        for T in self.T:
            if t in T:
                adm = T.pop(t)
                self.T[1][t] = adm
                return True
        return False

    def _evict(self, step):
        l = 0 if (self.T[0] and (len(self.T[0]) > self.p or not self.T[1])) else 1
        pick = next((t for t, a in self.T[l].items() if step - a >= self.min_res), None)
        if pick is None:
            other = next((t for t, a in self.T[1 - l].items() if step - a >= self.min_res), None)
            if other is not None:
                l, pick = 1 - l, other
            else:
                pick = next(iter(self.T[l]))
        del self.T[l][pick]
        self.B[l][pick] = 0
        while len(self.B[l]) > self.caps[l]:
            self.B[l].popitem(last=False)
        return pick

    def admit(self, tokens, step):
        self.events += 1
        adapt = self.events > self.warmup
        ev = []
        for t in tokens:
            if self.touch(t):
                continue
            to2 = False
            if t in self.B[0]:
                if adapt:
                    self.p = min(self.c, self.p + max(1, len(self.B[1]) // len(self.B[0])))
                del self.B[0][t]
                to2 = True
            elif t in self.B[1]:
                if adapt:
                    self.p = max(0, self.p - max(1, len(self.B[0]) // len(self.B[1])))
                del self.B[1][t]
                to2 = True
            if len(self.T[0]) + len(self.T[1]) >= self.c:
                ev.append(self._evict(step))
            self.T[1 if to2 else 0][t] = step
        return ev

    def state(self):
        return dict(T1=list(self.T[0]), T2=list(self.T[1]), B1=list(self.B[0]), B2=list(self.B[1]), p=self.p)
