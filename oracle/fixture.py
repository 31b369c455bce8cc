"""TEST INFRASTRUCTURE — a network + plan + schedule fixture for the CPU oracle.

The CPU reference arm of bench.py (``--impl reference``) must not load the
product library.  ``FixtureNet`` gives ``OracleNet`` (oracle/train_oracle.py)
the same read-only interface a ``ReforwardNet`` does -- tensors(), ops(),
params(), op_attrs(), schedule(), plan_sets() -- from a JSON file exported
once by ``oracle/make_fixture.py``:

* the tensor graph (names, NCHW shapes, dtypes, Eq. 1 costs, producers), ops
  with their attributes, and parameters in PyTorch layout;
* the stored set chosen by the REFERENCE planner (oracle/_ref, the reference
  ``solve_acg`` of /root/reference/proj/include/reforward/acg.hpp:579-600)
  and its segments;
* the executor's re-forward schedule for that set (forward / re-forward /
  backward / release instructions; the reference has no training code, its
  simulator simulate.hpp:39-94 defines the same order of segment visits).
"""
from __future__ import annotations

import gzip
import json
import os
from dataclasses import dataclass
from typing import Dict, List, Tuple

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURE_DIR = os.path.join(HERE, "fixtures")


@dataclass
class TensorInfo:
    id: int
    name: str
    shape: Tuple[int, int, int, int]
    dtype: str
    cost: int
    producer: int


@dataclass
class OpInfo:
    id: int
    name: str
    kind: str
    inputs: List[int]
    out: int


@dataclass
class ParamInfo:
    index: int
    name: str
    shape: Tuple[int, ...]
    kind: int
    count: int


def fixture_path(arch: str, batch: int, hw: int) -> str:
    return os.path.join(FIXTURE_DIR, f"{arch}_b{batch}_{hw}.json.gz")


class FixtureNet:
    def __init__(self, path: str):
        with gzip.open(path, "rt") as f:
            d = json.load(f)
        self.meta = d["meta"]
        self._tensors = [TensorInfo(t[0], t[1], tuple(t[2]), t[3], t[4], t[5]) for t in d["tensors"]]
        self._ops = [OpInfo(o[0], o[1], o[2], list(o[3]), o[4]) for o in d["ops"]]
        self._params = [ParamInfo(p[0], p[1], tuple(p[2]), p[3], p[4]) for p in d["params"]]
        self._attrs: Dict[int, Dict[str, int]] = {int(k): v for k, v in d["attrs"].items()}
        self._schedule = [(s[0], s[1], s[2], bool(s[3]), s[4]) for s in d["schedule"]]
        self._stored = list(d["stored"])
        self._seg_of = list(d["seg_of"])
        self.batch = self.meta["batch"]

    @classmethod
    def named(cls, arch: str, batch: int, hw: int) -> "FixtureNet":
        return cls(fixture_path(arch, batch, hw))

    def tensors(self) -> List[TensorInfo]:
        return list(self._tensors)

    def ops(self) -> List[OpInfo]:
        return list(self._ops)

    def params(self) -> List[ParamInfo]:
        return list(self._params)

    def op_attrs(self, op: int) -> Dict[str, int]:
        return dict(self._attrs[op])

    def schedule(self):
        return list(self._schedule)

    def plan_sets(self):
        return list(self._stored), list(self._seg_of)


def export(net, path: str, meta: dict) -> None:
    """Write a fixture from any object with the ReforwardNet read interface
    (called by oracle/make_fixture.py on a planned network)."""
    stored, seg = net.plan_sets()
    d = {
        "meta": meta,
        "tensors": [[t.id, t.name, list(t.shape), t.dtype, t.cost, t.producer] for t in net.tensors()],
        "ops": [[o.id, o.name, o.kind, list(o.inputs), o.out] for o in net.ops()],
        "params": [[p.index, p.name, list(p.shape), p.kind, p.count] for p in net.params()],
        "attrs": {str(o.id): net.op_attrs(o.id) for o in net.ops()},
        "schedule": [list(s) for s in net.schedule()],
        "stored": list(stored),
        "seg_of": list(seg),
    }
    os.makedirs(os.path.dirname(path), exist_ok=True)
    with gzip.open(path, "wt") as f:
        json.dump(d, f, separators=(",", ":"))
