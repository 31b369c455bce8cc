"""Generate tests/golden/planner_golden.json from the REFERENCE planner.

Runs only where /root/reference exists: it loads oracle/_ref/libreforward_ref.so
(the reference headers compiled in place by oracle/Makefile) and records, for a
fixed list of graphs, every planner output the product must reproduce
bit-exactly.  The JSON travels with the repo so the product can be checked
anywhere (CPU CI, GPU box) without the reference.

    make -C oracle && python tests/golden/make_planner_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_1808_00079_b200.planner import reference_planner  # noqa: E402


def fixture_graphs(P):
    """Canonical fixtures of the reference test suite (tests/support/fixtures.hpp)."""
    g = {}
    g["F1_chain4"] = P.gen_chain(4)
    g["F2_diamond"] = P.from_named_edges([("s", 1), ("a", 1), ("b", 1), ("t", 1)],
                                         [("s", "a"), ("s", "b"), ("a", "t"), ("b", "t")])
    g["F3_residual"] = P.from_named_edges([("s", 1), ("v1", 1), ("v2", 1), ("t", 1)],
                                          [("s", "v1"), ("v1", "v2"), ("v2", "t"), ("s", "v2")])
    g["F4_fig3a"] = P.from_named_edges([("v1", 1), ("v2", 1), ("v3", 1), ("v4", 1)],
                                       [("v1", "v2"), ("v2", "v3"), ("v3", "v4"), ("v1", "v3")])
    g["fig4c_type3"] = P.from_named_edges([("v1", 1), ("v2", 1), ("v3", 1), ("v4", 1)],
                                          [("v1", "v2"), ("v2", "v3"), ("v3", "v4"), ("v1", "v3"), ("v2", "v4")])
    g["fig3b_splittable"] = P.from_named_edges(
        [("v1", 1), ("a", 1), ("b", 1), ("v2", 1), ("v3", 1)],
        [("v1", "a"), ("v1", "b"), ("a", "v2"), ("b", "v2"), ("v2", "v3")])
    g["fig4b_three_branches"] = P.from_named_edges(
        [("s", 1), ("p1", 1), ("p2", 1), ("p3", 1), ("t", 1)],
        [("s", "p1"), ("p1", "t"), ("s", "p2"), ("p2", "t"), ("s", "p3"), ("p3", "t")])
    # test_acg.cpp "structures a greedy expansion mishandles"
    g["asym_diamond"] = P.from_named_edges(
        [("s", 1), ("u", 5), ("a", 3), ("b", 3), ("v", 5), ("t", 1)],
        [("s", "u"), ("u", "a"), ("u", "b"), ("a", "v"), ("b", "v"), ("v", "t")])
    names = ["n1", "a", "n2", "b", "n3", "c", "d", "e", "n4"]
    pairs = [(0, 1), (1, 2), (2, 3), (3, 4), (0, 5), (5, 4), (2, 6), (6, 8), (4, 7), (7, 8)]
    g["double_chord"] = P.from_named_edges([(n, 1) for n in names], [(names[a], names[b]) for a, b in pairs])
    g["spike_chain9"] = P.gen_chain(9, [1, 1, 1, 1, 9, 1, 1, 1, 1])
    for n in (1, 4, 16, 25, 100):
        g[f"chain{n}"] = P.gen_chain(n)
    for b in (1, 2, 5, 16):
        g[f"residual{b}x4"] = P.gen_residual(b, 4)
    g["residual1x2"] = P.gen_residual(1, 2)
    for b, w in ((1, 3), (3, 2), (4, 4)):
        g[f"inception{b}x{w}"] = P.gen_inception(b, w)
    for k in (1, 2, 3, 5, 7):
        g[f"dense{k}"] = P.gen_dense(k)
    # multi-root / multi-leaf normalisation and a lone vertex
    g["two_roots"] = P.from_named_edges([("a", 2), ("b", 3), ("c", 1)], [("a", "c"), ("b", "c")])
    g["lone"] = P.from_named_edges([("x", 5)], [])
    return g


def random_graphs(P):
    g = {}
    # acceptance.cpp criterion 2 seeds (first 120) and fuzz-style mixes
    for i in range(120):
        seed = 900000 + i
        n = 3 + seed % 10
        g[f"acc2_seed{seed}"] = P.gen_random(n, 0.3, seed, 1, 8)
    rng = random.Random(1808)
    for i in range(120):
        n = rng.randint(3, 16)
        p = rng.choice([0.2, 0.3, 0.4, 0.5])
        seed = rng.randint(0, 2 ** 40)
        g[f"rand{i}_n{n}_p{p}"] = P.gen_random(n, p, seed, 1, rng.choice([1, 8, 100]))
    rng2 = random.Random(77)
    for i in range(20):
        n = rng2.randint(1, 30)
        costs = [rng2.randint(1, 8) for _ in range(n)]
        g[f"chain_rand{i}"] = P.gen_chain(n, costs)
    return g


def closed_sets_digest(cs) -> str:
    return hashlib.sha256(json.dumps(cs, separators=(",", ":")).encode()).hexdigest()


def record(name, g):
    rec = {"name": name, "graph": g.to_dict(), "source": g.name(g.source), "sink": g.name(g.sink),
           "topo": [g.name(v) for v in g.topo_order()]}
    s = g.solve_acg()
    rec["acg"] = {"stored": s.stored_names(g), "stored_cost": s.stored_cost, "realized_max": s.realized_max,
                  "total": s.total, "candidate_max_term": s.candidate_max_term,
                  "segments": [[g.name(v) for v in seg] for seg in s.segments]}
    rec["max_terms"] = g.max_term_list()
    rec["tree_text"] = g.division_tree_text()
    rec["tree_canonical"] = g.division_tree_canonical()
    rec["tree_nodes"] = g.division_tree_count()
    cs = [[g.name(c.entry), g.name(c.exit), c.includes_direct_edge, c.cost, [g.name(v) for v in c.members]]
          for c in g.enumerate_closed_sets()]
    rec["closed_sets_sha256"] = closed_sets_digest(cs)
    rec["closed_sets_count"] = len(cs)
    if g.n_vertices() <= 24:
        rec["closed_sets"] = cs
    if len(g.interior()) > 0:
        t, parts = g.divide_whole()
        rec["divide"] = {"type": t, "parts": [[g.name(c.entry), g.name(c.exit), c.includes_direct_edge,
                                               [g.name(v) for v in c.members]] for c in parts]}
    peak, nev, rec_counts = g.simulate(s.stored)
    rec["simulate"] = {"peak": peak, "events": nev, "recompute": {g.name(v): rec_counts[v] for v in g.interior()}}
    sa = g.store_all()
    rec["store_all_total"] = sa.total
    if len(g.interior()) <= 16:
        o = g.oracle_min()
        rec["oracle"] = {"stored": o.stored_names(g), "total": o.total}
    if g.is_linear_chain():
        st, sc, mt, tot = g.solve_lcg()
        rec["lcg"] = {"stored": [g.name(v) for v in st], "stored_cost": sc, "max_term": mt, "total": tot}
        h = g.sqrt_heuristic_chain()
        rec["sqrt_heuristic"] = {"stored": h.stored_names(g), "total": h.total}
    mts = rec["max_terms"]
    rec["with_max_term"] = {}
    for c in mts[: min(len(mts), 6)]:
        w = g.solve_with_max_term(c)
        rec["with_max_term"][str(c)] = {"stored": w.stored_names(g), "total": w.total}
    return rec


def network_graphs(P):
    """Tensor graphs of the executor's networks (byte costs), if available."""
    from paper_1808_00079_b200.executor import ReforwardNet
    out = {}
    for arch, batch, hw, classes in NETWORKS:
        net = ReforwardNet.named(arch, batch, hw, hw, classes)
        vs, es = net.graph()
        out[f"net_{arch}_b{batch}_{hw}"] = P.from_named_edges(vs, es)
    return out


# the executor's tensor graphs (vertex = tensor, cost = arena bytes)
NETWORKS = [("chain8", 4, 32, 10), ("resnet18", 32, 224, 1000), ("resnet34", 32, 224, 1000),
            ("resnet50", 32, 224, 1000), ("resnet101", 32, 224, 1000), ("resnet50", 2, 64, 16)]


def main():
    P = reference_planner()
    assert P.abi_name().startswith("reforward_ref"), P.abi_name()
    cases = {}
    cases.update(fixture_graphs(P))
    cases.update(random_graphs(P))
    cases.update(network_graphs(P))
    recs = [record(k, g) for k, g in cases.items()]
    out = {"generator": "tests/golden/make_planner_golden.py", "oracle": P.abi_name(),
           "reference": "/root/reference/proj/include/reforward (header-only, compiled by oracle/Makefile)",
           "cases": recs}
    path = os.path.join(HERE, "planner_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print(f"wrote {len(recs)} cases to {path}")


if __name__ == "__main__":
    main()
