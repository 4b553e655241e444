"""Storage tiers and expert placement (reference storage.py:1-243).

Two tiers feed the HBM ring:

* host tier — the container payload in pinned host memory; a page-in is one
  ``cudaMemcpyAsync`` H2D over PCIe on the kind's copy stream;
* device tier — tensors the placement puts on the "compressed device"
  backend are staged once into a separate HBM region; a page-in is a D2D copy.
  (The reference decompresses here; the codec is lossless so the bytes are
  identical.  The GPU decoder is the next row of the build — DESIGN.md.)

``plan_placement`` is host policy and keeps the reference's two rules
bit-for-bit: bandwidth-proportional greedy (storage.py:119-140) and the
alpha split of whole experts (storage.py:143-168).
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .errors import BackendMissError, CapacityExceededError, OutOfRangeError
from .geometry import ExpertTensorId, ModelSpec, TensorKind, WeightContainer, iter_tensor_ids, tensor_offset


class BackendKind(str, Enum):
    COMPRESSED_DEVICE = "compressed_device"
    HOST_OFFLOAD = "host_offload"


@dataclass(frozen=True)
class Backend:
    backend_id: int
    kind: BackendKind
    bandwidth: float
    capacity: int

    def __post_init__(self):
        if self.bandwidth <= 0:
            raise OutOfRangeError(f"backend {self.backend_id}: bandwidth must be > 0")
        if self.capacity < 0:
            raise OutOfRangeError(f"backend {self.backend_id}: negative capacity")


@dataclass
class PlacementPlan:
    fractions: dict
    assignment: dict
    per_layer_bytes: dict
    spec: ModelSpec = None

    def backend_for(self, tid: ExpertTensorId) -> int:
        if tid not in self.assignment:
            raise BackendMissError(f"{tid} is not in the placement plan")
        return self.assignment[tid]

    def layer_bytes(self, layer: int, backend_id: int) -> int:
        return self.per_layer_bytes.get((layer, backend_id), 0)


@dataclass(frozen=True)
class LoadEstimate:
    per_backend: tuple
    tau_load_layer: tuple
    tau_load: float


def _tensors_of_layer(spec: ModelSpec, layer: int):
    return [ExpertTensorId(layer, e, k) for e in range(1, spec.experts_per_layer + 1)
            for k in (TensorKind.GATE_UP, TensorKind.DOWN)]


def plan_placement(spec: ModelSpec, backends, alpha: float | None = None) -> PlacementPlan:
    if not backends:
        raise OutOfRangeError("need at least one backend")
    ids = [b.backend_id for b in backends]
    if len(set(ids)) != len(ids):
        raise OutOfRangeError("backend ids must be unique")
    plan = _alpha_split(spec, backends, alpha) if alpha is not None else _bandwidth_balanced(spec, backends)
    used = {}
    for (_layer, bid), n in plan.per_layer_bytes.items():
        used[bid] = used.get(bid, 0) + n
    for b in backends:
        if used.get(b.backend_id, 0) > b.capacity:
            raise CapacityExceededError(
                f"backend {b.backend_id} holds {used.get(b.backend_id, 0)} bytes, capacity {b.capacity}")
    return plan


def _bandwidth_balanced(spec: ModelSpec, backends) -> PlacementPlan:
    bw = {b.backend_id: b.bandwidth for b in backends}
    total = sum(bw.values())
    fractions = {bid: v / total for bid, v in bw.items()}
    order = sorted(bw)
    assignment, per_layer = {}, {}
    for layer in range(1, spec.num_layers + 1):
        load = dict.fromkeys(order, 0)
        # biggest tensors first; each goes where it would finish soonest (ties: lower id)
        for tid in sorted(_tensors_of_layer(spec, layer), key=lambda t: (-spec.sigma(t.kind), t.expert, int(t.kind))):
            size = spec.sigma(tid.kind)
            dest = min(order, key=lambda bid: ((load[bid] + size) / bw[bid], bid))
            load[dest] += size
            assignment[tid] = dest
        for bid in order:
            per_layer[(layer, bid)] = load[bid]
    return PlacementPlan(fractions, assignment, per_layer, spec)


def _alpha_split(spec: ModelSpec, backends, alpha: float) -> PlacementPlan:
    if not (0.0 < alpha <= 1.0):
        raise OutOfRangeError(f"alpha must lie in (0, 1], got {alpha}")
    dev = [b for b in backends if b.kind == BackendKind.COMPRESSED_DEVICE]
    host = [b for b in backends if b.kind == BackendKind.HOST_OFFLOAD]
    if len(dev) != 1 or len(host) != 1:
        raise OutOfRangeError("the residency split needs exactly one device and one host backend")
    d, h = dev[0].backend_id, host[0].backend_id
    L = spec.experts_per_layer
    m = min(L, max(1, round(alpha * L)))  # Python round(): banker's rounding, as the reference
    assignment, per_layer = {}, {}
    for layer in range(1, spec.num_layers + 1):
        on_dev = 0
        for tid in _tensors_of_layer(spec, layer):
            bid = d if tid.expert <= m else h
            assignment[tid] = bid
            on_dev += spec.sigma(tid.kind) if bid == d else 0
        per_layer[(layer, d)] = on_dev
        per_layer[(layer, h)] = spec.layer_bytes - on_dev
    return PlacementPlan({d: alpha, h: 1.0 - alpha}, assignment, per_layer, spec)


def estimate_load(plan: PlacementPlan, backends, spec: ModelSpec) -> LoadEstimate:
    bw = {b.backend_id: b.bandwidth for b in backends}
    per_backend, per_layer = [], []
    for layer in range(1, spec.num_layers + 1):
        taus = {bid: plan.layer_bytes(layer, bid) / v for bid, v in bw.items()}
        per_backend.append(taus)
        per_layer.append(max(taus.values()) if taus else 0.0)
    return LoadEstimate(tuple(per_backend), tuple(per_layer), float(sum(per_layer)))


def tau_layer_for_alpha(spec: ModelSpec, b_dev: float, b_host: float, alpha: float) -> float:
    return max(alpha * spec.layer_bytes / b_dev, (1.0 - alpha) * spec.layer_bytes / b_host)


def tau_load_for_alpha_layers(spec: ModelSpec, b_dev: float, b_host: float, alpha_layers) -> float:
    return sum(tau_layer_for_alpha(spec, b_dev, b_host, a) for a in alpha_layers)


class StorageHierarchy:
    """Serves exact tensor bytes from the planned tier.

    ``fetch(tid, dest)`` accepts a CUDA uint8 tensor (the normal case: a ring
    block's loading view) or a writable host buffer.  ``delay_fn`` is the
    reference's race-amplification hook; inside ``StreamedRunner`` it becomes
    a device-side spin on the copy stream before that tensor's DMA.
    """

    def __init__(self, container: WeightContainer, compressed, plan: PlacementPlan, backends, delay_fn=None):
        self.container = container
        self.compressed = compressed
        self.plan = plan
        self.backends = {b.backend_id: b for b in backends}
        self.delay_fn = delay_fn

    @property
    def spec(self) -> ModelSpec:
        return self.container.spec

    def on_device(self, tid: ExpertTensorId) -> bool:
        return self.backends[self.plan.backend_for(tid)].kind == BackendKind.COMPRESSED_DEVICE

    def backend_map(self) -> np.ndarray:
        """uint8 [N][L][2]: 1 where the tensor lives on the device tier."""
        s = self.spec
        out = np.zeros((s.num_layers, s.experts_per_layer, 2), dtype=np.uint8)
        for tid in iter_tensor_ids(s):
            out[tid.layer - 1, tid.expert - 1, int(tid.kind) - 1] = 1 if self.on_device(tid) else 0
        return out

    def delay_table(self):
        """float32 [N][L][2] seconds from delay_fn (None if no hook)."""
        if self.delay_fn is None:
            return None
        s = self.spec
        out = np.zeros((s.num_layers, s.experts_per_layer, 2), dtype=np.float32)
        for tid in iter_tensor_ids(s):
            out[tid.layer - 1, tid.expert - 1, int(tid.kind) - 1] = float(self.delay_fn(tid))
        return out

    def fetch(self, tid: ExpertTensorId, dest) -> None:
        self.plan.backend_for(tid)  # BackendMissError for unknown ids
        if self.delay_fn is not None:
            d = self.delay_fn(tid)
            if d > 0:
                time.sleep(d)
        n = self.spec.sigma(tid.kind)
        nbytes = int(dest.numel()) if hasattr(dest, "numel") else len(dest)
        if nbytes != n:
            raise BackendMissError(f"{tid}: fetched {n} bytes into a {nbytes}-byte block")
        off = tensor_offset(tid, self.spec)
        src = self.container.pinned[off:off + n]
        if hasattr(dest, "copy_"):
            dest.copy_(src, non_blocking=False)
        else:
            dest[:] = src.numpy().tobytes()
