"""The reference's acceptance criteria (SPEC.md ACCEPTANCE CRITERIA 1-8,
proj/tests/acceptance.cpp) run against the product planner, with the
independent Python scorer in oracle/planner_oracle.py as a second checker,
plus a live differential against the reference library when it is built
(oracle/_ref, this container only)."""
import math
import os
import random
import time

import pytest

from oracle import planner_oracle as O
from paper_1808_00079_b200.planner import (DecompositionError, SizeLimitError, ValidationError,
                                           default_planner, reference_planner)

P = default_planner()


def test_c1_uniform_chain_bounds():
    t0 = time.time()
    for n in (4, 16, 25, 100):
        g = P.gen_chain(n)
        s = g.solve_acg()
        assert s.total <= 2 * math.ceil(math.sqrt(n))
        if n <= 20:
            assert s.total == g.oracle_min().total
        if n == 100:
            assert s.total <= int(0.20 * 100) + 1
        k, (num, den) = P.analytic_uniform(n)
    assert P.analytic_uniform(100) == (10, (1, 5))
    assert P.analytic_uniform(1) == (1, (2, 1))
    assert P.analytic_uniform(16) == (4, (1, 2))
    assert time.time() - t0 < 10


@pytest.mark.parametrize("block", range(5))
def test_c2_c3_oracle_equivalence_and_simulator(block):
    # criterion 2 seeds 900000.. (100 per block -> 500 total), criterion 3 on each
    for i in range(block * 100, block * 100 + 100):
        seed = 900000 + i
        n = 3 + seed % 10
        g = P.gen_random(n, 0.3, seed, 1, 8)
        s = g.solve_acg()
        o = g.oracle_min()
        assert s.total == o.total, seed
        peak, _, rec = g.simulate(s.stored)
        assert peak == s.total
        gt = O.graph_tuple(g)
        assert O.score(*gt, set(s.stored)) == s.total
        assert O.simulate_peak(*gt, set(s.stored)) == s.total
        if n <= 8:
            assert O.oracle_min(*gt)[0] == o.total
        assert all(rec[v] == 1 for v in g.interior() if v not in s.stored)


def test_c4_lcg_acg_agreement():
    rng = random.Random(777001)
    for _ in range(50):
        n = rng.randint(1, 30)
        g = P.gen_chain(n, [rng.randint(1, 8) for _ in range(n)])
        assert g.solve_lcg()[3] == g.solve_acg().total


def test_c5_paper_figures():
    f4 = P.from_named_edges([("v1", 1), ("v2", 1), ("v3", 1), ("v4", 1)],
                            [("v1", "v2"), ("v2", "v3"), ("v3", "v4"), ("v1", "v3")])
    sets = {(f4.name(c.entry), f4.name(c.exit)): [f4.name(v) for v in c.members] for c in f4.enumerate_closed_sets()}
    assert ("v2", "v4") not in sets
    assert sets[("v1", "v3")] == ["v2"]
    fig3b = P.from_named_edges([("v1", 1), ("a", 1), ("b", 1), ("v2", 1), ("v3", 1)],
                               [("v1", "a"), ("v1", "b"), ("a", "v2"), ("b", "v2"), ("v2", "v3")])
    t, parts = fig3b.divide_whole()
    assert t == "splittable"
    assert [(fig3b.name(p.entry), fig3b.name(p.exit)) for p in parts] == [("v1", "v2"), ("v2", "v3")]
    fig4b = P.from_named_edges([("s", 1), ("p1", 1), ("p2", 1), ("p3", 1), ("t", 1)],
                               [("s", "p1"), ("p1", "t"), ("s", "p2"), ("p2", "t"), ("s", "p3"), ("p3", "t")])
    t, parts = fig4b.divide_whole()
    assert t == "branched" and len(parts) == 3
    fig4c = P.from_named_edges([("v1", 1), ("v2", 1), ("v3", 1), ("v4", 1)],
                               [("v1", "v2"), ("v2", "v3"), ("v3", "v4"), ("v1", "v3"), ("v2", "v4")])
    split = fig4c.maximal_split_whole()
    assert [(fig4c.name(p.entry), fig4c.name(p.exit)) for p in split] == [
        ("v1", "v2"), ("v1", "v3"), ("v2", "v3"), ("v2", "v4"), ("v3", "v4")]


def test_c6_dominance_and_scaling():
    rng = random.Random(31415)
    suite = [P.gen_chain(4), P.gen_residual(1, 2), P.gen_inception(1, 2)]
    suite += [P.gen_random(3 + i % 10, 0.3, rng.randrange(2 ** 62), 1, 8) for i in range(60)]
    for g in suite:
        s = g.solve_acg()
        assert s.total <= g.interior_total()
        assert s.total <= g.objective_of([]).total
        for lam in (2, 7):
            h = P.build(g.names(), [c * lam for c in g.costs()], g.edges())
            sl = h.solve_acg()
            assert sl.total == s.total * lam
            assert sl.stored == s.stored


def test_c7_complexity_smoke():
    t0 = time.time()
    g64 = P.gen_residual(16, 4)
    a = time.time()
    s64 = g64.solve_acg()
    t64 = time.time() - a
    g128 = P.gen_residual(32, 4)
    a = time.time()
    s128 = g128.solve_acg()
    t128 = time.time() - a
    assert s64.total > 0 and s128.total > 0
    assert t128 / max(t64, 0.02) <= 20.0
    assert time.time() - t0 < 120


def test_c8_heuristic_dominance():
    rng = random.Random(555777)
    for _ in range(20):
        n = rng.randint(4, 24)
        g = P.gen_chain(n, [rng.randint(1, 8) for _ in range(n)])
        assert g.solve_acg().total <= g.sqrt_heuristic_chain().total
    spike = P.gen_chain(9, [1, 1, 1, 1, 9, 1, 1, 1, 1])
    assert spike.solve_acg().total < spike.sqrt_heuristic_chain().total


def test_error_behaviour():
    with pytest.raises(ValidationError, match="self-loop"):
        P.build(["a", "b"], [1, 1], [(0, 0)])
    with pytest.raises(ValidationError, match="cycle"):
        P.build(["a", "b", "c"], [1, 1, 1], [(0, 1), (1, 2), (2, 0)])
    with pytest.raises(ValidationError, match="negative cost"):
        P.build(["a", "b"], [1, -1], [(0, 1)])
    with pytest.raises(ValidationError, match="duplicate edge"):
        P.build(["a", "b"], [1, 1], [(0, 1), (0, 1)], strict=True)
    g = P.build(["a", "b"], [1, 1], [(0, 1), (0, 1)])
    assert g.warnings == ["duplicate edges removed"]
    with pytest.raises(ValidationError, match="lies on no source-sink path"):
        P.build(["a", "b", "c"], [1, 1, 1], [(0, 1)], strict=True)
    g = P.build(["a", "b", "c"], [1, 1, 1], [(0, 1)])
    assert g.n_vertices() == 2 and "pruned isolated vertex 'c'" in g.warnings
    with pytest.raises(SizeLimitError, match="oracle limited to 20"):
        P.gen_chain(21).oracle_min()
    with pytest.raises(ValidationError, match="linear chains only"):
        P.gen_residual(1, 2).sqrt_heuristic_chain()
    assert DecompositionError.__mro__[1].__name__ == "Error"


def test_normalisation():
    g = P.from_named_edges([("a", 2), ("b", 3), ("c", 1)], [("a", "c"), ("b", "c")])
    assert g.name(g.source) == "_s" and g.cost(g.source) == 0
    assert g.normalize().to_dict() == g.to_dict()
    g2 = P.from_named_edges([("_s", 1), ("b", 3), ("c", 1)], [("_s", "c"), ("b", "c")])
    assert g2.name(g2.source) == "__s"
    lone = P.from_named_edges([("x", 4)], [])
    assert lone.source == lone.sink == 0 and lone.solve_acg().total == 0


REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                   "libreforward_ref.so")


@pytest.mark.skipif(not os.path.exists(REF), reason="reference oracle not built (oracle/Makefile)")
def test_live_differential_vs_reference():
    R = reference_planner(REF)
    rng = random.Random(4242)
    for i in range(300):
        n = rng.randint(3, 15)
        p = rng.choice([0.2, 0.3, 0.45])
        seed = rng.randrange(2 ** 63)
        a, b = P.gen_random(n, p, seed, 1, 9), R.gen_random(n, p, seed, 1, 9)
        assert a.to_dict() == b.to_dict()
        sa, sb = a.solve_acg(), b.solve_acg()
        assert (sa.stored, sa.total, sa.candidate_max_term) == (sb.stored, sb.total, sb.candidate_max_term)
        assert a.division_tree_text() == b.division_tree_text()
