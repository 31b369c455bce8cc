"""Python face of the re-forward training executor (rfx_net_* C-ABI).

    net = ReforwardNet.named("resnet50", batch=32)
    net.plan("reforward")          # host planner on the tensor graph
    net.setup(seed=0)              # device arenas + parameters
    net.load_batch(images, labels) # NCHW fp32 + int32 (host or device tensors)
    net.step(lr=0.1)               # forward (stored tensors only) + backward
                                   # (per-segment re-forward) + SGD, on sm_100a

The executor owns its device memory (activation arena sized to the planner's
Eq. 1 total); torch is only used to hand in host/device buffers and streams.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

from ._lib import load_library

OP_KINDS = ["input", "conv", "bn", "bn_add_relu", "relu", "maxpool", "avgpool", "fc", "concat", "loss", "avgpool2d",
            "linear"]
POLICIES = ("reforward", "store_all", "lcg", "sqrt")


class MemoryReport(C.Structure):
    _fields_ = [(n, C.c_int64) for n in (
        "planned_total", "stored_cost", "max_segment", "store_all_total", "tracked_peak", "arena_bytes",
        "grad_arena_bytes", "workspace_bytes", "param_bytes", "state_bytes", "reforward_ops", "segment_loads",
        "forward_ops", "backward_ops", "launches_per_step", "candidate_max_term")] + [
        ("n_segments", C.c_int32), ("n_stored", C.c_int32), ("device_bytes", C.c_int64)]

    def as_dict(self) -> Dict[str, int]:
        return {k: getattr(self, k) for k, _ in self._fields_}


_SIGS = {
    "rfx_net_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "rfx_net_create_named": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                       C.POINTER(C.c_void_p)]),
    "rfx_net_free": (None, [C.c_void_p]),
    "rfx_net_input": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]),
    "rfx_net_conv": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                               C.c_char_p, C.POINTER(C.c_int32)]),
    "rfx_net_conv2": (C.c_int, [C.c_void_p] + [C.c_int32] * 7 + [C.c_char_p, C.POINTER(C.c_int32)]),
    "rfx_net_bn": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, C.POINTER(C.c_int32)]),
    "rfx_net_bn_add_relu": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, C.POINTER(C.c_int32)]),
    "rfx_net_relu": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.POINTER(C.c_int32)]),
    "rfx_net_maxpool": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_char_p,
                                  C.POINTER(C.c_int32)]),
    "rfx_net_avgpool": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.POINTER(C.c_int32)]),
    "rfx_net_avgpool2d": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_char_p,
                                    C.POINTER(C.c_int32)]),
    "rfx_net_linear": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, C.POINTER(C.c_int32)]),
    "rfx_net_fc": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, C.POINTER(C.c_int32)]),
    "rfx_net_concat": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, C.POINTER(C.c_int32)]),
    "rfx_net_loss": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.POINTER(C.c_int32)]),
    "rfx_net_num_tensors": (C.c_int32, [C.c_void_p]),
    "rfx_net_tensor_info": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.c_size_t, C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "rfx_net_num_ops": (C.c_int32, [C.c_void_p]),
    "rfx_net_op_info": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.c_size_t, C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "rfx_net_flops_per_step": (C.c_int64, [C.c_void_p]),
    "rfx_net_op_attrs": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32)]),
    "rfx_net_plan": (C.c_int, [C.c_void_p, C.c_char_p]),
    "rfx_net_plan_with_stored": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.c_char_p]),
    "rfx_net_plan_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint8), C.POINTER(C.c_int32),
                                    C.POINTER(MemoryReport)]),
    "rfx_net_schedule": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                   C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_int32)]),
    "rfx_net_setup": (C.c_int, [C.c_void_p, C.c_uint64]),
    "rfx_net_stage_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "rfx_net_use_batch": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "rfx_net_load_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "rfx_net_forward_backward": (C.c_int, [C.c_void_p, C.c_void_p]),
    "rfx_net_update": (C.c_int, [C.c_void_p, C.c_float, C.c_float, C.c_float, C.c_void_p]),
    "rfx_net_step": (C.c_int, [C.c_void_p, C.c_float, C.c_float, C.c_float, C.c_int32, C.c_void_p]),
    "rfx_net_read_loss": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.c_void_p]),
    "rfx_net_copy_loss": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.c_void_p]),
    "rfx_net_instr_profile": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_double), C.c_int32,
                                        C.POINTER(C.c_int32)]),
    "rfx_net_arena_guard": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "rfx_net_gemm_try": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p,
                                   C.POINTER(C.c_double)]),
    "rfx_net_gemm_profile_detail": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_double), C.c_int32,
                                              C.POINTER(C.c_int32)]),
    "rfx_net_run_phase": (C.c_int, [C.c_void_p, C.c_int32, C.c_float, C.c_float, C.c_float, C.c_int32,
                                    C.c_void_p]),
    "rfx_net_gemm_profile": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_double),
                                       C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "rfx_net_num_params": (C.c_int32, [C.c_void_p]),
    "rfx_net_param_info": (C.c_int, [C.c_void_p, C.c_int32, C.c_char_p, C.c_size_t, C.POINTER(C.c_int32),
                                     C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "rfx_net_read_param": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "rfx_net_param_slot": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "rfx_net_pack_param": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "rfx_net_unpack_param": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "rfx_net_write_param": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "rfx_net_read_tensor": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "rfx_net_read_bn_running": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "rfx_net_grad_buffer": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64)]),
    "rfx_net_set_keep_grads": (C.c_int, [C.c_void_p, C.c_int32]),
    "rfx_comm_unique_id": (C.c_int, [C.c_char_p]),
    "rfx_net_set_comm": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_char_p, C.c_int64]),
    "rfx_net_comm_buckets": (C.c_int32, [C.c_void_p]),
    "rfx_net_bucket_plan": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64), C.c_int32, C.POINTER(C.c_int32)]),
    "rfx_net_read_grad_tensor": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "rf_last_error": (C.c_char_p, []),
}

_bound = None


def torch_float32():
    import torch
    return torch.float32


def torch_int32():
    import torch
    return torch.int32


def _lib():
    global _bound
    if _bound is None:
        L = load_library()
        for n, (r, a) in _SIGS.items():
            f = getattr(L, n)
            f.restype = r
            f.argtypes = a
        _bound = L
    return _bound


def _check(rc: int) -> None:
    if rc != 0:
        raise RuntimeError(f"rfx error {rc}: {_lib().rf_last_error().decode()}")


def _stream(stream) -> Optional[int]:
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    return stream if isinstance(stream, int) else stream.cuda_stream


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


class ReforwardNet:
    """Handle on one rfx_net (network + plan + device state)."""

    def __init__(self, batch: int, handle: Optional[C.c_void_p] = None):
        self.L = _lib()
        self.batch = batch
        if handle is None:
            handle = C.c_void_p()
            _check(self.L.rfx_net_create(batch, C.byref(handle)))
        self.h = handle

    @classmethod
    def named(cls, arch: str, batch: int, H: int = 224, W: int = 224, classes: int = 1000) -> "ReforwardNet":
        h = C.c_void_p()
        _check(_lib().rfx_net_create_named(arch.encode(), batch, H, W, classes, C.byref(h)))
        return cls(batch, h)

    def __del__(self):
        try:
            if self.h:
                self.L.rfx_net_free(self.h)
                self.h = None
        except Exception:
            pass

    # ------------------------------------------------------------ building
    def _op(self, fn, *args) -> int:
        out = C.c_int32()
        _check(fn(self.h, *args, C.byref(out)))
        return out.value

    def input(self, H, W, Cin):
        return self._op(self.L.rfx_net_input, H, W, Cin)

    def conv(self, x, cout, k, stride=1, pad=0, name="conv", R=None, S=None):
        return self._op(self.L.rfx_net_conv, x, cout, R or k, S or k, stride, pad, name.encode())

    def conv2(self, x, cout, R, S, stride=1, pad_h=0, pad_w=0, name="conv"):
        """Convolution with rectangular filter and padding (Inception 1x7 / 7x1 / 1x3 / 3x1)."""
        return self._op(self.L.rfx_net_conv2, x, cout, R, S, stride, pad_h, pad_w, name.encode())

    def bn(self, y, relu=True, name="bn"):
        return self._op(self.L.rfx_net_bn, y, int(relu), name.encode())

    def bn_add_relu(self, y, skip, name="bn_add"):
        return self._op(self.L.rfx_net_bn_add_relu, y, skip, name.encode())

    def relu(self, x, name="relu"):
        return self._op(self.L.rfx_net_relu, x, name.encode())

    def maxpool(self, x, k, stride, pad, name="maxpool"):
        return self._op(self.L.rfx_net_maxpool, x, k, stride, pad, name.encode())

    def avgpool(self, x, name="avgpool"):
        return self._op(self.L.rfx_net_avgpool, x, name.encode())

    def avgpool2d(self, x, k, stride, pad=0, name="avgpool2d"):
        return self._op(self.L.rfx_net_avgpool2d, x, k, stride, pad, name.encode())

    def linear(self, x, out_features, name="linear"):
        return self._op(self.L.rfx_net_linear, x, out_features, name.encode())

    def fc(self, x, classes, name="fc"):
        return self._op(self.L.rfx_net_fc, x, classes, name.encode())

    def concat(self, a, b, name="concat"):
        return self._op(self.L.rfx_net_concat, a, b, name.encode())

    def loss(self, logits, name="loss"):
        return self._op(self.L.rfx_net_loss, logits, name.encode())

    # ------------------------------------------------------------ introspection
    def tensors(self) -> List[TensorInfo]:
        out = []
        for t in range(self.L.rfx_net_num_tensors(self.h)):
            name = C.create_string_buffer(256)
            shp = (C.c_int32 * 4)()
            dt, cost, prod = C.c_int32(), C.c_int64(), C.c_int32()
            _check(self.L.rfx_net_tensor_info(self.h, t, name, 256, shp, C.byref(dt), C.byref(cost), C.byref(prod)))
            out.append(TensorInfo(t, name.value.decode(), tuple(shp), "bf16" if dt.value == 0 else "f32", cost.value,
                                  prod.value))
        return out

    def ops(self) -> List[OpInfo]:
        out = []
        for o in range(self.L.rfx_net_num_ops(self.h)):
            name = C.create_string_buffer(256)
            kind, ins, ot = C.c_int32(), (C.c_int32 * 2)(), C.c_int32()
            _check(self.L.rfx_net_op_info(self.h, o, name, 256, C.byref(kind), ins, C.byref(ot)))
            out.append(OpInfo(o, name.value.decode(), OP_KINDS[kind.value], [i for i in ins if i >= 0], ot.value))
        return out

    def op_attrs(self, op: int) -> Dict[str, int]:
        a = (C.c_int32 * 9)()
        _check(self.L.rfx_net_op_attrs(self.h, op, a))
        return dict(zip(("R", "S", "stride", "pad", "k", "classes", "cin_real", "cout", "pad_w"), list(a)))

    def graph(self) -> Tuple[List[Tuple[str, int]], List[Tuple[str, str]]]:
        """The tensor graph handed to the planner: (name, cost) vertices, named edges."""
        ts = self.tensors()
        verts = [(t.name, t.cost) for t in ts]
        edges = [(ts[i].name, ts[o.out].name) for o in self.ops() for i in o.inputs]
        return verts, edges

    def flops_per_step(self) -> int:
        return self.L.rfx_net_flops_per_step(self.h)

    # ------------------------------------------------------------ planning
    def plan(self, policy: str = "reforward") -> MemoryReport:
        _check(self.L.rfx_net_plan(self.h, policy.encode()))
        return self.report()

    def graph_key(self) -> str:
        """Hash of the tensor graph the planner sees (names, costs, edges)."""
        import hashlib
        verts, edges = self.graph()
        h = hashlib.sha256()
        for n, c in verts:
            h.update(f"{n}:{c};".encode())
        for a, b in edges:
            h.update(f"{a}>{b};".encode())
        return h.hexdigest()

    def plan_cached(self, policy: str, path: str) -> MemoryReport:
        """plan(policy), memoised in a JSON file keyed by the graph hash.

        A cached plan is replayed with plan_with_stored, which re-scores it
        (Eq. 1) on the current graph; the stored total must match the cache.
        Used for graphs whose exact plan takes minutes (Inception-v3)."""
        import json
        import os
        key = self.graph_key()
        if os.path.exists(path):
            with open(path) as f:
                c = json.load(f)
            if c.get("graph_key") == key and c.get("policy") == policy:
                names = {t.name: t.id for t in self.tensors()}
                rep = self.plan_with_stored([names[n] for n in c["stored"]], f"{policy} (cached)")
                if rep.planned_total != c["planned_total"]:
                    raise RuntimeError(f"cached plan {path} scores {rep.planned_total}, expected {c['planned_total']}")
                return rep
        import time
        t0 = time.time()
        rep = self.plan(policy)
        stored, _ = self.plan_sets()
        ts = self.tensors()
        os.makedirs(os.path.dirname(os.path.abspath(path)), exist_ok=True)
        with open(path, "w") as f:
            json.dump({"policy": policy, "graph_key": key, "planned_total": rep.planned_total,
                       "store_all_total": rep.store_all_total, "plan_seconds": time.time() - t0,
                       "stored": [ts[i].name for i in stored]}, f, indent=0)
        return rep

    def plan_with_stored(self, stored: Sequence[int], label: str = "custom") -> MemoryReport:
        n = self.L.rfx_net_num_tensors(self.h)
        m = (C.c_uint8 * n)()
        for v in stored:
            m[v] = 1
        _check(self.L.rfx_net_plan_with_stored(self.h, m, label.encode()))
        return self.report()

    def report(self) -> MemoryReport:
        r = MemoryReport()
        _check(self.L.rfx_net_plan_info(self.h, None, None, C.byref(r)))
        return r

    def plan_sets(self) -> Tuple[List[int], List[int]]:
        n = self.L.rfx_net_num_tensors(self.h)
        m = (C.c_uint8 * n)()
        s = (C.c_int32 * n)()
        _check(self.L.rfx_net_plan_info(self.h, m, s, None))
        return [i for i in range(n) if m[i]], list(s)

    def schedule(self) -> List[Tuple[str, int, int, bool, int]]:
        """(kind, op, segment, is_reforward, phase) per instruction of one step."""
        n = C.c_int32()
        _check(self.L.rfx_net_schedule(self.h, None, None, None, None, None, 0, C.byref(n)))
        k, o, s, r, ph = [(C.c_int32 * max(n.value, 1))() for _ in range(5)]
        _check(self.L.rfx_net_schedule(self.h, k, o, s, r, ph, n.value, C.byref(n)))
        names = ["forward", "backward", "release"]
        return [(names[k[i]], o[i], s[i], bool(r[i]), ph[i]) for i in range(n.value)]

    # ------------------------------------------------------------ runtime
    def setup(self, seed: int = 0) -> None:
        _check(self.L.rfx_net_setup(self.h, seed))

    def load_batch(self, images, labels, stream=None) -> None:
        """images: float32 NCHW, labels: int32 [batch]; torch tensors (host or cuda) or numpy."""
        import numpy as np
        try:
            import torch
        except Exception:  # pragma: no cover
            torch = None
        if torch is not None and isinstance(images, torch.Tensor):
            assert images.dtype == torch.float32 and images.is_contiguous()
            assert labels.dtype == torch.int32 and labels.is_contiguous()
            from_host = int(not images.is_cuda)
            _check(self.L.rfx_net_load_batch(self.h, C.c_void_p(images.data_ptr()), C.c_void_p(labels.data_ptr()),
                                             from_host, _stream(stream)))
            return
        im = np.ascontiguousarray(images, dtype=np.float32)
        lb = np.ascontiguousarray(labels, dtype=np.int32)
        _check(self.L.rfx_net_load_batch(self.h, im.ctypes.data_as(C.c_void_p), lb.ctypes.data_as(C.c_void_p), 1,
                                         _stream(stream)))

    def stage_batch(self, images, labels, slot: int, copy_stream=None) -> None:
        """Async H2D of a host batch (pinned torch tensors) into staging slot 0/1 on copy_stream."""
        assert not images.is_cuda and images.dtype == torch_float32() and images.is_contiguous()
        assert labels.dtype == torch_int32() and labels.is_contiguous()
        _check(self.L.rfx_net_stage_batch(self.h, C.c_void_p(images.data_ptr()), C.c_void_p(labels.data_ptr()),
                                          slot, _stream(copy_stream)))

    def use_batch(self, slot: int, stream=None) -> None:
        """Make `stream` wait for staging slot `slot`, pack it into the input, free the slot."""
        _check(self.L.rfx_net_use_batch(self.h, slot, _stream(stream)))

    def forward_backward(self, stream=None) -> None:
        _check(self.L.rfx_net_forward_backward(self.h, _stream(stream)))

    def update(self, lr=0.1, momentum=0.9, weight_decay=0.0, stream=None) -> None:
        _check(self.L.rfx_net_update(self.h, lr, momentum, weight_decay, _stream(stream)))

    def step(self, lr=0.1, momentum=0.9, weight_decay=0.0, use_graph=True, stream=None) -> None:
        _check(self.L.rfx_net_step(self.h, lr, momentum, weight_decay, int(use_graph), _stream(stream)))

    def run_phase(self, phase: int, lr=0.1, momentum=0.9, weight_decay=0.0, use_graph=True, stream=None) -> None:
        _check(self.L.rfx_net_run_phase(self.h, phase, lr, momentum, weight_decay, int(use_graph), _stream(stream)))

    def gemm_profile(self, iters: int = 10, stream=None) -> Tuple[float, float, int]:
        """(ms per step, algorithmic flops per step, launches) of the step's GEMMs replayed alone."""
        ms, fl, n = C.c_double(), C.c_double(), C.c_int64()
        _check(self.L.rfx_net_gemm_profile(self.h, iters, _stream(stream), C.byref(ms), C.byref(fl), C.byref(n)))
        return ms.value, fl.value, n.value

    def gemm_profile_detail(self, iters: int = 5, stream=None) -> List[Dict[str, float]]:
        """Per-launch timing of the step's GEMMs (CUDA events between eager launches)."""
        n = C.c_int32()
        _check(self.L.rfx_net_gemm_profile_detail(self.h, iters, _stream(stream), None, 0, C.byref(n)))
        buf = (C.c_double * (10 * max(n.value, 1)))()
        _check(self.L.rfx_net_gemm_profile_detail(self.h, iters, _stream(stream), buf, n.value, C.byref(n)))
        keys = ("M", "N", "K", "a_kind", "b_kind", "splits", "ms", "flops", "bytes", "block_n")
        return [dict(zip(keys, buf[10 * i: 10 * i + 10])) for i in range(n.value)]

    def arena_guard_intact(self) -> bool:
        """No kernel wrote past the Eq.-1-sized activation arena (canary band check)."""
        v = C.c_int32()
        _check(self.L.rfx_net_arena_guard(self.h, C.byref(v)))
        return bool(v.value)

    def gemm_try(self, idx: int, block_n: int, splits: int, iters: int = 5, stream=None) -> float:
        """ms of traced GEMM `idx` with a forced tile width and split count (tuning probe)."""
        ms = C.c_double()
        _check(self.L.rfx_net_gemm_try(self.h, idx, block_n, splits, iters, _stream(stream), C.byref(ms)))
        return ms.value

    def instr_profile(self, iters: int = 3, stream=None) -> List[float]:
        """In-stream ms of each schedule instruction, then of the SGD update (last entry)."""
        n = C.c_int32()
        _check(self.L.rfx_net_instr_profile(self.h, iters, _stream(stream), None, 0, C.byref(n)))
        buf = (C.c_double * max(n.value, 1))()
        _check(self.L.rfx_net_instr_profile(self.h, iters, _stream(stream), buf, n.value, C.byref(n)))
        return list(buf[:n.value])

    def copy_loss(self, host_dst, index: int = 0, stream=None) -> None:
        """Enqueue the D2H copy of the step's loss into host_dst[index] (a pinned
        float32 CPU tensor) without synchronising the host."""
        import torch
        if host_dst.dtype != torch.float32 or host_dst.device.type != "cpu":
            raise ValueError("host_dst must be a float32 CPU tensor")
        ptr = host_dst.data_ptr() + 4 * index
        _check(self.L.rfx_net_copy_loss(self.h, C.cast(C.c_void_p(ptr), C.POINTER(C.c_float)), _stream(stream)))

    def read_loss(self, stream=None) -> float:
        v = C.c_float()
        _check(self.L.rfx_net_read_loss(self.h, C.byref(v), _stream(stream)))
        return v.value

    # ------------------------------------------------------------ parameters
    def params(self) -> List[ParamInfo]:
        out = []
        for i in range(self.L.rfx_net_num_params(self.h)):
            name = C.create_string_buffer(256)
            shp = (C.c_int32 * 4)()
            nd, kind, cnt = C.c_int32(), C.c_int32(), C.c_int64()
            _check(self.L.rfx_net_param_info(self.h, i, name, 256, shp, C.byref(nd), C.byref(kind), C.byref(cnt)))
            out.append(ParamInfo(i, name.value.decode(), tuple(shp[: nd.value]), kind.value, cnt.value))
        return out

    def read_param(self, i: int, which: int = 0):
        import numpy as np
        p = self.params()[i]
        a = np.empty(p.shape, dtype=np.float32)
        _check(self.L.rfx_net_read_param(self.h, i, which, a.ctypes.data_as(C.c_void_p)))
        return a

    def write_param(self, i: int, value) -> None:
        import numpy as np
        a = np.ascontiguousarray(value, dtype=np.float32)
        p = self.params()[i]
        assert a.size == p.count, (p.name, a.shape, p.shape)
        _check(self.L.rfx_net_write_param(self.h, i, a.ctypes.data_as(C.c_void_p)))

    def param_slot(self, i: int) -> Tuple[int, int]:
        """(offset, count) of parameter i in the flat fp32 parameter / gradient buffers."""
        off, cnt = C.c_int64(), C.c_int64()
        _check(self.L.rfx_net_param_slot(self.h, i, C.byref(off), C.byref(cnt)))
        return off.value, cnt.value

    def pack_param(self, i: int, value):
        """Host-only: canonical tensor -> its flat-buffer slice (GEMM layout, zero padding)."""
        import numpy as np
        a = np.ascontiguousarray(value, dtype=np.float32)
        out = np.empty(self.param_slot(i)[1], dtype=np.float32)
        _check(self.L.rfx_net_pack_param(self.h, i, a.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
        return out

    def unpack_param(self, i: int, flat_slice):
        """Host-only: flat-buffer slice -> canonical tensor."""
        import numpy as np
        f = np.ascontiguousarray(flat_slice, dtype=np.float32)
        out = np.empty(self.params()[i].shape, dtype=np.float32)
        _check(self.L.rfx_net_unpack_param(self.h, i, f.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p)))
        return out

    def read_tensor(self, t: int):
        import numpy as np
        info = self.tensors()[t]
        a = np.empty(info.shape, dtype=np.float32)
        _check(self.L.rfx_net_read_tensor(self.h, t, a.ctypes.data_as(C.c_void_p)))
        return a

    def set_keep_grads(self, on: bool = True) -> None:
        _check(self.L.rfx_net_set_keep_grads(self.h, int(on)))

    def read_grad_tensor(self, t: int):
        import numpy as np
        info = self.tensors()[t]
        a = np.empty(info.shape, dtype=np.float32)
        _check(self.L.rfx_net_read_grad_tensor(self.h, t, a.ctypes.data_as(C.c_void_p)))
        return a

    def read_bn_running(self, op: int):
        import numpy as np
        o = self.ops()[op]
        c = self.tensors()[o.out].shape[3]
        m, v = np.empty(c, np.float32), np.empty(c, np.float32)
        _check(self.L.rfx_net_read_bn_running(self.h, op, m.ctypes.data_as(C.c_void_p), v.ctypes.data_as(C.c_void_p)))
        return m, v

    @staticmethod
    def comm_unique_id() -> bytes:
        """NCCL unique id (rank 0); broadcast it with torch.distributed."""
        buf = C.create_string_buffer(128)
        _check(_lib().rfx_comm_unique_id(buf))
        return buf.raw

    def set_comm(self, world: int, rank: int, uid: bytes, bucket_bytes: int = 25 << 20) -> int:
        """Average gradients across `world` ranks inside every step (NCCL,
        bucketed, overlapped with the backward).  Returns the bucket count."""
        assert len(uid) == 128
        _check(self.L.rfx_net_set_comm(self.h, world, rank, uid, bucket_bytes))
        return self.L.rfx_net_comm_buckets(self.h)

    def bucket_plan(self, bucket_bytes: int = 25 << 20) -> List[Tuple[int, int, int]]:
        """(after schedule instruction, lo, hi) float ranges of the all-reduce buckets."""
        n = C.c_int32()
        _check(self.L.rfx_net_bucket_plan(self.h, bucket_bytes, None, None, None, 0, C.byref(n)))
        a, lo, hi = (C.c_int32 * max(n.value, 1))(), (C.c_int64 * max(n.value, 1))(), (C.c_int64 * max(n.value, 1))()
        _check(self.L.rfx_net_bucket_plan(self.h, bucket_bytes, a, lo, hi, n.value, C.byref(n)))
        return [(a[i], lo[i], hi[i]) for i in range(n.value)]

    def param_offsets(self) -> List[Tuple[int, int]]:
        """(offset, count) of every parameter in the flat gradient buffer (dry, from the layout rules)."""
        out, off = [], 0
        for p in self.params():
            n = self._param_alloc_count(p)
            out.append((off, n))
            off += (n + 63) // 64 * 64
        return out

    def _param_alloc_count(self, p) -> int:
        if p.kind != 0:
            return p.count
        co, ci, r, s = p.shape
        if ci < 32:  # explicit-im2col layer: [Cout][Kpad]
            return co * ((r * s * ci + 63) // 64 * 64)
        return co * r * s * ((ci + 63) // 64 * 64)

    def grad_buffer(self) -> Tuple[int, int]:
        p, n = C.c_void_p(), C.c_int64()
        _check(self.L.rfx_net_grad_buffer(self.h, C.byref(p), C.byref(n)))
        return p.value, n.value
