"""Product planner vs the reference planner's recorded outputs (bit-exact).

tests/golden/planner_golden.json was produced by tests/golden/make_planner_golden.py
from the reference headers compiled in place (oracle/_ref).  Every field the
reference computed — the chosen checkpoint set, Eq. 1 totals, segments, the
max-term list, the division tree, closed sets, the simulator peak, the LCG
solution and the exhaustive oracle — must match exactly.
"""
import hashlib
import json
import os

import pytest

from paper_1808_00079_b200.planner import default_planner

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "planner_golden.json")))
CASES = GOLDEN["cases"]


def _build(P, rec):
    gd = rec["graph"]
    return P.from_named_edges([(v["name"], v["cost"]) for v in gd["vertices"]], [tuple(e) for e in gd["edges"]])


@pytest.mark.parametrize("rec", CASES, ids=[c["name"] for c in CASES])
def test_matches_reference(rec):
    P = default_planner()
    g = _build(P, rec)
    assert g.to_dict() == rec["graph"]
    assert g.name(g.source) == rec["source"] and g.name(g.sink) == rec["sink"]
    assert [g.name(v) for v in g.topo_order()] == rec["topo"]

    s = g.solve_acg()
    got = {"stored": s.stored_names(g), "stored_cost": s.stored_cost, "realized_max": s.realized_max,
           "total": s.total, "candidate_max_term": s.candidate_max_term,
           "segments": [[g.name(v) for v in seg] for seg in s.segments]}
    assert got == rec["acg"]
    assert g.max_term_list() == rec["max_terms"]
    assert g.division_tree_text() == rec["tree_text"]
    assert g.division_tree_canonical() == rec["tree_canonical"]
    assert g.division_tree_count() == rec["tree_nodes"]

    cs = [[g.name(c.entry), g.name(c.exit), c.includes_direct_edge, c.cost, [g.name(v) for v in c.members]]
          for c in g.enumerate_closed_sets()]
    assert len(cs) == rec["closed_sets_count"]
    assert hashlib.sha256(json.dumps(cs, separators=(",", ":")).encode()).hexdigest() == rec["closed_sets_sha256"]
    if "closed_sets" in rec:
        assert cs == rec["closed_sets"]
    if "divide" in rec:
        t, parts = g.divide_whole()
        assert t == rec["divide"]["type"]
        assert [[g.name(c.entry), g.name(c.exit), c.includes_direct_edge, [g.name(v) for v in c.members]]
                for c in parts] == rec["divide"]["parts"]

    peak, nev, counts = g.simulate(s.stored)
    assert {"peak": peak, "events": nev,
            "recompute": {g.name(v): counts[v] for v in g.interior()}} == rec["simulate"]
    assert peak == s.total
    assert g.store_all().total == rec["store_all_total"]
    if "oracle" in rec:
        o = g.oracle_min()
        assert {"stored": o.stored_names(g), "total": o.total} == rec["oracle"]
        assert o.total == s.total
    if "lcg" in rec:
        st, sc, mt, tot = g.solve_lcg()
        assert {"stored": [g.name(v) for v in st], "stored_cost": sc, "max_term": mt, "total": tot} == rec["lcg"]
        h = g.sqrt_heuristic_chain()
        assert {"stored": h.stored_names(g), "total": h.total} == rec["sqrt_heuristic"]
    for c, want in rec["with_max_term"].items():
        w = g.solve_with_max_term(int(c))
        assert {"stored": w.stored_names(g), "total": w.total} == want


def test_golden_covers_network_graphs_when_generated():
    names = [c["name"] for c in CASES]
    assert any(n.startswith("F1") for n in names)
    assert sum(n.startswith("acc2_seed") for n in names) >= 100
