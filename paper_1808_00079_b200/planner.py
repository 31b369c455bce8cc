"""Python face of the host planner, over the rf_* C-ABI (include/reforward_b200.h).

Mirrors the reference's C++ interface (proj/include/reforward/*.hpp): a
``CompGraph`` built from names/costs/edges (graph.hpp:23-51), ``solve_acg``
(acg.hpp:579), ``solve_lcg`` (lcg.hpp:158), ``oracle_min`` (oracle.hpp:13),
``objective_of`` (objective.hpp:33), ``simulate`` (simulate.hpp:38), the
division tree dumps (division_tree.hpp:162,183) and the generators
(generators.hpp).  Errors surface as the reference's exception classes.

``Planner(lib)`` binds any library exporting the ABI: the product library
(default) or the reference oracle ``oracle/_ref/libreforward_ref.so`` — the
latter only from tests.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

from ._lib import load_library

# ---------------------------------------------------------------- errors (errors.hpp:8-37)


class Error(RuntimeError):
    pass


class ParseError(Error):
    pass


class ValidationError(Error):
    pass


class SizeLimitError(Error):
    pass


class DecompositionError(Error):
    pass


class InternalError(Error):
    pass


_ERRORS = {1: ParseError, 2: ValidationError, 3: SizeLimitError, 4: DecompositionError,
           5: InternalError, 6: ValueError, 7: RuntimeError, 9: Error}


class _Info(C.Structure):
    _fields_ = [("stored_cost", C.c_int64), ("realized_max", C.c_int64), ("total", C.c_int64),
                ("candidate_max_term", C.c_int64), ("n_stored", C.c_int32), ("n_segments", C.c_int32)]


_SIGS = {
    "rf_last_error": (C.c_char_p, []),
    "rf_abi_name": (C.c_char_p, []),
    "rf_graph_build": (C.c_int, [C.c_int32, C.POINTER(C.c_char_p), C.POINTER(C.c_int64), C.c_int32,
                                 C.POINTER(C.c_uint32), C.c_int32, C.POINTER(C.c_void_p), C.c_char_p,
                                 C.c_size_t]),
    "rf_graph_free": (None, [C.c_void_p]),
    "rf_graph_num_vertices": (C.c_int32, [C.c_void_p]),
    "rf_graph_num_edges": (C.c_int32, [C.c_void_p]),
    "rf_graph_edges": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32)]),
    "rf_graph_cost": (C.c_int64, [C.c_void_p, C.c_uint32]),
    "rf_graph_name": (C.c_char_p, [C.c_void_p, C.c_uint32]),
    "rf_graph_source": (C.c_uint32, [C.c_void_p]),
    "rf_graph_sink": (C.c_uint32, [C.c_void_p]),
    "rf_graph_topo_order": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint32)]),
    "rf_graph_reaches": (C.c_int32, [C.c_void_p, C.c_uint32, C.c_uint32]),
    "rf_graph_is_linear_chain": (C.c_int32, [C.c_void_p]),
    "rf_graph_interior_total": (C.c_int64, [C.c_void_p]),
    "rf_graph_normalize": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "rf_objective_of": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(_Info), C.POINTER(C.c_int32)]),
    "rf_solve_acg": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(_Info), C.POINTER(C.c_int32)]),
    "rf_solve_with_max_term": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_uint8), C.POINTER(_Info),
                                         C.POINTER(C.c_int32)]),
    "rf_solve_lcg": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                               C.POINTER(C.c_int64)]),
    "rf_oracle_min": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_uint8), C.POINTER(_Info),
                                C.POINTER(C.c_int32)]),
    "rf_store_all": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(_Info)]),
    "rf_sqrt_heuristic_chain": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(_Info)]),
    "rf_analytic_uniform": (C.c_int, [C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64)]),
    "rf_simulate": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.c_int32, C.POINTER(C.c_int64),
                              C.POINTER(C.c_int32), C.POINTER(C.c_uint32)]),
    "rf_enumerate_closed_sets": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "rf_divide_whole": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_char_p, C.c_size_t,
                                  C.POINTER(C.c_size_t)]),
    "rf_maximal_split_whole": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "rf_division_tree_text": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "rf_division_tree_canonical": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "rf_division_tree_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "rf_max_term_list": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int32)]),
    "rf_gen_chain": (C.c_int, [C.c_int32, C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_void_p)]),
    "rf_gen_residual": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "rf_gen_inception": (C.c_int, [C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "rf_gen_dense": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "rf_gen_random": (C.c_int, [C.c_int32, C.c_double, C.c_uint64, C.c_int64, C.c_int64,
                                C.POINTER(C.c_void_p)]),
}

SPLITTABLE, BRANCHED, NON_BRANCHED = 0, 1, 2
TYPE_NAMES = {0: "splittable", 1: "branched", 2: "non-branched"}


@dataclass
class Solution:
    """objective.hpp:21-28: stored set V^R (vertex ids), Eq. 1 terms, segments."""
    stored: List[int]
    stored_cost: int
    realized_max: int
    total: int
    candidate_max_term: int
    segments: List[List[int]] = field(default_factory=list)

    def stored_names(self, g: "CompGraph") -> List[str]:
        return [g.name(v) for v in self.stored]


@dataclass
class ClosedSetRec:
    entry: int
    exit: int
    includes_direct_edge: bool
    cost: int
    members: List[int]


def _parse_sets(text: str) -> List[ClosedSetRec]:
    out = []
    for line in text.splitlines():
        if not line.strip():
            continue
        parts = line.split(" ")
        mem = [int(x) for x in parts[4].split(",")] if len(parts) > 4 and parts[4] else []
        out.append(ClosedSetRec(int(parts[0]), int(parts[1]), parts[2] == "1", int(parts[3]), mem))
    return out


class Planner:
    """Binding of one rf_* library.  Default: the product library."""

    def __init__(self, lib: Optional[C.CDLL] = None):
        self.lib = lib if lib is not None else load_library()
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.lib, name)
            fn.restype = res
            fn.argtypes = args

    # ------------------------------------------------------------ plumbing
    def abi_name(self) -> str:
        return self.lib.rf_abi_name().decode()

    def check(self, rc: int) -> None:
        if rc != 0:
            msg = self.lib.rf_last_error().decode()
            raise _ERRORS.get(rc, Error)(msg)

    def _text(self, fn, *args) -> str:
        need = C.c_size_t(0)
        self.check(fn(*args, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        self.check(fn(*args, buf, need.value, C.byref(need)))
        return buf.value.decode()

    # ------------------------------------------------------------ graphs
    def build(self, names: Sequence[str], costs: Sequence[int], edges: Sequence[Tuple[int, int]],
              strict: bool = False) -> "CompGraph":
        n = len(names)
        arr_n = (C.c_char_p * max(n, 1))(*[s.encode() for s in names])
        arr_c = (C.c_int64 * max(n, 1))(*costs)
        flat = [x for e in edges for x in e]
        arr_e = (C.c_uint32 * max(len(flat), 1))(*flat)
        h = C.c_void_p()
        warn = C.create_string_buffer(4096)
        self.check(self.lib.rf_graph_build(n, arr_n, arr_c, len(edges), arr_e, int(strict), C.byref(h), warn,
                                           4096))
        g = CompGraph(self, h)
        g.warnings = [w for w in warn.value.decode().splitlines() if w]
        return g

    def from_named_edges(self, vertices: Sequence[Tuple[str, int]], edges: Sequence[Tuple[str, str]],
                         strict: bool = False) -> "CompGraph":
        ids = {}
        for i, (nm, _) in enumerate(vertices):
            if nm in ids:
                raise ParseError(f"duplicate vertex '{nm}'")
            ids[nm] = i
        try:
            e = [(ids[a], ids[b]) for a, b in edges]
        except KeyError:
            raise ParseError("edge references undeclared vertex")
        return self.build([v[0] for v in vertices], [v[1] for v in vertices], e, strict)

    def _wrap(self, rc, h) -> "CompGraph":
        self.check(rc)
        return CompGraph(self, h)

    def gen_chain(self, n: int, costs: Sequence[int] = ()) -> "CompGraph":
        h = C.c_void_p()
        arr = (C.c_int64 * max(len(costs), 1))(*costs)
        return self._wrap(self.lib.rf_gen_chain(n, arr if costs else None, len(costs), C.byref(h)), h)

    def gen_residual(self, blocks: int, length: int) -> "CompGraph":
        h = C.c_void_p()
        return self._wrap(self.lib.rf_gen_residual(blocks, length, C.byref(h)), h)

    def gen_inception(self, blocks: int, width: int) -> "CompGraph":
        h = C.c_void_p()
        return self._wrap(self.lib.rf_gen_inception(blocks, width, C.byref(h)), h)

    def gen_dense(self, k: int) -> "CompGraph":
        h = C.c_void_p()
        return self._wrap(self.lib.rf_gen_dense(k, C.byref(h)), h)

    def gen_random(self, n: int, p: float, seed: int, cost_min: int = 1, cost_max: int = 1) -> "CompGraph":
        h = C.c_void_p()
        return self._wrap(self.lib.rf_gen_random(n, p, seed, cost_min, cost_max, C.byref(h)), h)

    def analytic_uniform(self, n: int) -> Tuple[int, Tuple[int, int]]:
        k, num, den = C.c_int64(), C.c_int64(), C.c_int64()
        self.check(self.lib.rf_analytic_uniform(n, C.byref(k), C.byref(num), C.byref(den)))
        return k.value, (num.value, den.value)


class CompGraph:
    """Handle on an immutable normalized graph (graph.hpp:19-95)."""

    def __init__(self, planner: Planner, handle: C.c_void_p):
        self.p = planner
        self.h = handle
        self.warnings: List[str] = []
        lib = planner.lib
        self.n = lib.rf_graph_num_vertices(handle)
        ne = lib.rf_graph_num_edges(handle)
        buf = (C.c_uint32 * max(2 * ne, 1))()
        planner.check(lib.rf_graph_edges(handle, buf))
        self._edges = [(buf[2 * i], buf[2 * i + 1]) for i in range(ne)]
        order = (C.c_uint32 * max(self.n, 1))()
        planner.check(lib.rf_graph_topo_order(handle, order))
        self._topo = list(order[: self.n])
        self._names = [lib.rf_graph_name(handle, v).decode() for v in range(self.n)]
        self._costs = [lib.rf_graph_cost(handle, v) for v in range(self.n)]
        self.source = lib.rf_graph_source(handle)
        self.sink = lib.rf_graph_sink(handle)

    def __del__(self):
        try:
            if self.h:
                self.p.lib.rf_graph_free(self.h)
                self.h = None
        except Exception:
            pass

    # accessors
    def n_vertices(self) -> int:
        return self.n

    def edges(self) -> List[Tuple[int, int]]:
        return list(self._edges)

    def name(self, v: int) -> str:
        return self._names[v]

    def names(self) -> List[str]:
        return list(self._names)

    def cost(self, v: int) -> int:
        return self._costs[v]

    def costs(self) -> List[int]:
        return list(self._costs)

    def topo_order(self) -> List[int]:
        return list(self._topo)

    def find_vertex(self, name: str) -> Optional[int]:
        try:
            return self._names.index(name)
        except ValueError:
            return None

    def reaches(self, u: int, v: int) -> bool:
        return bool(self.p.lib.rf_graph_reaches(self.h, u, v))

    def is_linear_chain(self) -> bool:
        return bool(self.p.lib.rf_graph_is_linear_chain(self.h))

    def interior_total(self) -> int:
        return self.p.lib.rf_graph_interior_total(self.h)

    def interior(self) -> List[int]:
        return [v for v in range(self.n) if v != self.source and v != self.sink]

    def normalize(self) -> "CompGraph":
        h = C.c_void_p()
        return self.p._wrap(self.p.lib.rf_graph_normalize(self.h, C.byref(h)), h)

    # solvers
    def _mask(self, stored: Sequence[int]):
        m = (C.c_uint8 * max(self.n, 1))()
        for v in stored:
            m[v] = 1
        return m

    def _solution(self, mask, info: _Info, seg) -> Solution:
        stored = [v for v in range(self.n) if mask[v]]
        segs: Dict[int, List[int]] = {}
        if seg is not None:
            for v in range(self.n):
                if seg[v] >= 0:
                    segs.setdefault(seg[v], []).append(v)
        return Solution(stored, info.stored_cost, info.realized_max, info.total, info.candidate_max_term,
                        [segs[k] for k in sorted(segs)])

    def _solve(self, fn, *args) -> Solution:
        mask = (C.c_uint8 * max(self.n, 1))()
        seg = (C.c_int32 * max(self.n, 1))()
        info = _Info()
        self.p.check(fn(self.h, *args, mask, C.byref(info), seg))
        return self._solution(mask, info, seg)

    def solve_acg(self) -> Solution:
        return self._solve(self.p.lib.rf_solve_acg)

    def solve_with_max_term(self, c: int) -> Solution:
        return self._solve(self.p.lib.rf_solve_with_max_term, C.c_int64(c))

    def oracle_min(self, max_interior: int = 20) -> Solution:
        return self._solve(self.p.lib.rf_oracle_min, max_interior)

    def objective_of(self, stored: Sequence[int]) -> Solution:
        mask = self._mask(stored)
        seg = (C.c_int32 * max(self.n, 1))()
        info = _Info()
        self.p.check(self.p.lib.rf_objective_of(self.h, mask, C.byref(info), seg))
        return self._solution(mask, info, seg)

    def store_all(self) -> Solution:
        mask = (C.c_uint8 * max(self.n, 1))()
        info = _Info()
        self.p.check(self.p.lib.rf_store_all(self.h, mask, C.byref(info)))
        return self._solution(mask, info, None)

    def sqrt_heuristic_chain(self) -> Solution:
        mask = (C.c_uint8 * max(self.n, 1))()
        info = _Info()
        self.p.check(self.p.lib.rf_sqrt_heuristic_chain(self.h, mask, C.byref(info)))
        return self._solution(mask, info, None)

    def solve_lcg(self) -> Tuple[List[int], int, int, int]:
        mask = (C.c_uint8 * max(self.n, 1))()
        sc, mt, tot = C.c_int64(), C.c_int64(), C.c_int64()
        self.p.check(self.p.lib.rf_solve_lcg(self.h, mask, C.byref(sc), C.byref(mt), C.byref(tot)))
        return [v for v in range(self.n) if mask[v]], sc.value, mt.value, tot.value

    def simulate(self, stored: Sequence[int], order: int = 0) -> Tuple[int, int, List[int]]:
        peak, nev = C.c_int64(), C.c_int32()
        rec = (C.c_uint32 * max(self.n, 1))()
        self.p.check(self.p.lib.rf_simulate(self.h, self._mask(stored), order, C.byref(peak), C.byref(nev), rec))
        return peak.value, nev.value, list(rec[: self.n])

    # decomposition
    def enumerate_closed_sets(self) -> List[ClosedSetRec]:
        return _parse_sets(self.p._text(self.p.lib.rf_enumerate_closed_sets, self.h))

    def divide_whole(self) -> Tuple[str, List[ClosedSetRec]]:
        t = C.c_int32()
        text = self.p._text(self.p.lib.rf_divide_whole, self.h, C.byref(t))
        return TYPE_NAMES[t.value], _parse_sets(text)

    def maximal_split_whole(self) -> List[ClosedSetRec]:
        return _parse_sets(self.p._text(self.p.lib.rf_maximal_split_whole, self.h))

    def division_tree_text(self) -> str:
        return self.p._text(self.p.lib.rf_division_tree_text, self.h)

    def division_tree_canonical(self) -> str:
        return self.p._text(self.p.lib.rf_division_tree_canonical, self.h)

    def division_tree_count(self) -> int:
        c = C.c_int64()
        self.p.check(self.p.lib.rf_division_tree_count(self.h, C.byref(c)))
        return c.value

    def max_term_list(self) -> List[int]:
        n = C.c_int32()
        self.p.check(self.p.lib.rf_max_term_list(self.h, None, 0, C.byref(n)))
        arr = (C.c_int64 * max(n.value, 1))()
        self.p.check(self.p.lib.rf_max_term_list(self.h, arr, n.value, C.byref(n)))
        return list(arr[: n.value])

    def to_dict(self) -> dict:
        """JSON schema of the reference (SPEC graph-core External Interfaces)."""
        return {"vertices": [{"name": self._names[v], "cost": self._costs[v]} for v in range(self.n)],
                "edges": [[self._names[u], self._names[v]] for u, v in self._edges]}


_default: Optional[Planner] = None


def default_planner() -> Planner:
    global _default
    if _default is None:
        _default = Planner()
    return _default


def reference_planner(path: Optional[str] = None) -> Planner:
    """TEST-ONLY: bind the reference oracle library (oracle/_ref)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = path or os.path.join(root, "oracle", "_ref", "libreforward_ref.so")
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    return Planner(C.CDLL(path))
