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
