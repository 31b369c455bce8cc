"""TEST INFRASTRUCTURE — pure-Python restatement of the planner's scoring.

Never imported by the product.  Independent checker for Eq. 1 (paper §4,
"sum of the memory cost over all the stored tensors" + the largest re-forward
unit) and for the exhaustive-subset oracle:

* ``segments`` / ``score``   — reference objective.hpp:33-65 (segments are the
  weakly-connected components of non-stored interior vertices), restated by
  recursive flooding like tests/support/independent_scorer.hpp:18-39.
* ``oracle_min``              — reference oracle.hpp:13-33 (all 2^n subsets of
  the interior, ties: fewer stored, then lexicographically smaller id list —
  objective.hpp:69-74).
* ``simulate_peak``           — reference simulate.hpp:38-94 (stored set
  resident, one segment re-forwarded at a time).

Graphs are given as (n, costs, edges, source, sink) with dense integer ids.
"""
from __future__ import annotations

from itertools import combinations
from typing import Dict, Iterable, List, Sequence, Set, Tuple


def _adjacency(n: int, edges: Iterable[Tuple[int, int]]) -> List[Set[int]]:
    adj: List[Set[int]] = [set() for _ in range(n)]
    for u, v in edges:
        adj[u].add(v)
        adj[v].add(u)
    return adj


def segments(n, costs, edges, source, sink, stored: Set[int]) -> List[Tuple[List[int], int]]:
    adj = _adjacency(n, edges)
    live = {v for v in range(n) if v not in (source, sink) and v not in stored}
    seen: Set[int] = set()
    out = []
    for v in sorted(live):
        if v in seen:
            continue
        comp, stack = [], [v]
        seen.add(v)
        while stack:
            x = stack.pop()
            comp.append(x)
            for y in adj[x]:
                if y in live and y not in seen:
                    seen.add(y)
                    stack.append(y)
        out.append((sorted(comp), sum(costs[x] for x in comp)))
    return out


def score(n, costs, edges, source, sink, stored: Set[int]) -> int:
    segs = segments(n, costs, edges, source, sink, stored)
    return sum(costs[v] for v in stored) + max([c for _, c in segs], default=0)


def oracle_min(n, costs, edges, source, sink) -> Tuple[int, List[int]]:
    interior = [v for v in range(n) if v not in (source, sink)]
    best = None
    for k in range(len(interior) + 1):
        for sub in combinations(interior, k):  # ascending k, then lexicographic
            t = score(n, costs, edges, source, sink, set(sub))
            if best is None or t < best[0]:
                best = (t, list(sub))
    return best


def simulate_peak(n, costs, edges, source, sink, stored: Set[int]) -> int:
    base = sum(costs[v] for v in stored)
    segs = segments(n, costs, edges, source, sink, stored)
    peak = base
    for _, c in segs:
        peak = max(peak, base + c)
    return peak


def graph_tuple(g) -> Tuple[int, Sequence[int], Sequence[Tuple[int, int]], int, int]:
    """Adapter for a paper_1808_00079_b200.planner.CompGraph."""
    return g.n_vertices(), g.costs(), g.edges(), g.source, g.sink


def summary(d: Dict) -> str:
    return ", ".join(f"{k}={v}" for k, v in sorted(d.items()))
