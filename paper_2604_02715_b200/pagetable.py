"""PagedTensor over a fixed HBM ring of expert blocks (reference paging.py:1-271).

The reference keeps forward/reverse page<->block maps and a bytearray arena.
Here the arena is device memory owned by a libxpgb context; the host-side
bookkeeping (lowest-free-block-first allocation, the four-state lifecycle,
peak meter, trace lines) lives in C++ and a *device* slot table
(``int32 [2][N][L]``, entry = block<<2 | state) is what the GEMM kernels
read.  A compute kernel that reads a non-RESIDENT entry records a page fault
instead of returning garbage (``PageFaultError`` semantics, paging.py:228-237).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from enum import Enum

from . import _lib
from ._lib import call
from .device import Context, _torch
from .errors import OutOfRangeError
from .geometry import ExpertTensorId, ModelSpec, TensorKind, check_id, iter_tensor_ids

VADDR_BASE = 0x10_0000_0000
VADDR_GAP = 4096


def target_layer(i: int, n: int) -> int:
    """Layer whose blocks layer i recycles: the second preceding one, cyclically."""
    if n < 2:
        raise OutOfRangeError(f"need at least 2 layers, got {n}")
    if not (1 <= i <= n):
        raise OutOfRangeError(f"layer {i} outside [1, {n}]")
    return (i + n - 3) % n + 1


class PageState(Enum):
    UNMAPPED = "unmapped"
    LOADING = "loading"
    RESIDENT = "resident"
    EVICTING = "evicting"


_STATE_OF_CODE = {0: PageState.UNMAPPED, 1: PageState.LOADING, 2: PageState.RESIDENT, 3: PageState.EVICTING}


@dataclass(frozen=True)
class AddressSpace:
    """Stable per-kind virtual regions (Eq. 4); integers stand in for pointers."""

    spec: ModelSpec
    base_gate_up: int
    base_down: int

    @classmethod
    def for_spec(cls, spec: ModelSpec, base: int = VADDR_BASE) -> "AddressSpace":
        span = spec.num_layers * spec.experts_per_layer * spec.sigma_gate_up
        return cls(spec, base, base + span + VADDR_GAP)

    def base(self, kind) -> int:
        return self.base_gate_up if TensorKind(kind) == TensorKind.GATE_UP else self.base_down

    def extent(self, kind) -> int:
        return self.spec.num_layers * self.spec.experts_per_layer * self.spec.sigma(kind)


def page_vaddr(tid: ExpertTensorId, space: AddressSpace) -> int:
    check_id(tid, space.spec)
    s = space.spec
    return space.base(tid.kind) + ((tid.layer - 1) * s.experts_per_layer + (tid.expert - 1)) * s.sigma(tid.kind)


@dataclass
class PhysicalBlock:
    block_id: int
    kind: TensorKind
    capacity: int
    arena_offset: int
    bound_page: ExpertTensorId | None = None


class _DeviceBytes:
    """__cuda_array_interface__ wrapper so torch can view a raw device range."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3, "strides": None,
        }


def device_view(ptr: int, nbytes: int, device: int):
    torch = _torch()
    return torch.as_tensor(_DeviceBytes(ptr, nbytes), device=f"cuda:{device}")


class PageTable:
    """Page/block maps of one context's ring (or resident pool)."""

    def __init__(self, spec: ModelSpec, space: AddressSpace | None = None, trace=None, device: int = 0,
                 context: Context | None = None):
        self.spec = spec
        self.space = space or AddressSpace.for_spec(spec)
        self.ctx = context or Context(spec, _lib.POOL_RING, device)
        self.device = self.ctx.device
        self.trace = trace
        self._trace_seen = 0
        call("xpgb_pt_trace_enable", self.ctx.handle, 1 if trace is not None else 0)

    # ---- trace plumbing
    def sync_trace(self) -> None:
        if self.trace is None:
            return
        need = C.c_uint64()
        call("xpgb_pt_trace_get", self.ctx.handle, None, 0, C.byref(need))
        buf = C.create_string_buffer(need.value)
        call("xpgb_pt_trace_get", self.ctx.handle, buf, need.value, C.byref(need))
        lines = buf.value.decode().splitlines()
        for line in lines[self._trace_seen:]:
            self.trace.append(line)
        self._trace_seen = len(lines)

    def _ids(self, tid: ExpertTensorId):
        check_id(tid, self.spec)
        return (int(tid.layer), int(tid.expert), int(tid.kind))

    def _block(self, kind, block_id: int, tid) -> PhysicalBlock:
        ptr, nb = C.c_void_p(), C.c_uint64()
        call("xpgb_pt_block_ptr", self.ctx.handle, int(kind), block_id, C.byref(ptr), C.byref(nb))
        cap = self.spec.sigma(kind)
        offset = (block_id - 1) * cap
        if TensorKind(kind) == TensorKind.DOWN:
            offset += self.pool_blocks * self.spec.sigma_gate_up
        return PhysicalBlock(block_id, TensorKind(kind), cap, offset, tid)

    @property
    def pool_blocks(self) -> int:
        return self.pool_bytes // self.spec.expert_bytes

    # ---- lifecycle (paging.py:148-206)
    def map_page(self, tid: ExpertTensorId) -> PhysicalBlock:
        b = C.c_int32()
        try:
            call("xpgb_pt_map", self.ctx.handle, *self._ids(tid), C.byref(b))
        finally:
            self.sync_trace()
        return self._block(tid.kind, b.value, tid)

    def mark_resident(self, tid: ExpertTensorId) -> None:
        try:
            call("xpgb_pt_mark_resident", self.ctx.handle, *self._ids(tid))
        finally:
            self.sync_trace()

    def unmap_page(self, tid: ExpertTensorId) -> None:
        try:
            call("xpgb_pt_unmap", self.ctx.handle, *self._ids(tid))
        finally:
            self.sync_trace()

    def page_state(self, tid: ExpertTensorId) -> PageState:
        s = C.c_int32()
        call("xpgb_pt_state", self.ctx.handle, *self._ids(tid), C.byref(s))
        return _STATE_OF_CODE[s.value]

    def block_of(self, tid: ExpertTensorId) -> PhysicalBlock | None:
        b = C.c_int32()
        call("xpgb_pt_block", self.ctx.handle, *self._ids(tid), C.byref(b))
        return self._block(tid.kind, b.value, tid) if b.value else None

    def loading_view(self, tid: ExpertTensorId):
        """Writable uint8 CUDA tensor over the page's block while it is LOADING."""
        ptr, nb = C.c_void_p(), C.c_uint64()
        call("xpgb_pt_loading_view", self.ctx.handle, *self._ids(tid), C.byref(ptr), C.byref(nb))
        return device_view(ptr.value, nb.value, self.device)

    def read_page(self, tid: ExpertTensorId) -> bytes:
        """Bytes of a RESIDENT page (device -> host copy); faults otherwise."""
        n = self.spec.sigma(tid.kind)
        buf = C.create_string_buffer(n)
        call("xpgb_pt_read", self.ctx.handle, *self._ids(tid), buf, n)
        return buf.raw[:n]

    def arena_peak_bytes(self) -> int:
        v = C.c_uint64()
        call("xpgb_pt_peak_bytes", self.ctx.handle, C.byref(v))
        return int(v.value)

    @property
    def pool_bytes(self) -> int:
        v = C.c_uint64()
        call("xpgb_pt_pool_bytes", self.ctx.handle, C.byref(v))
        return int(v.value)

    def mapped_layers(self, kind) -> set:
        out = set()
        for tid in iter_tensor_ids(self.spec):
            if tid.kind == TensorKind(kind) and self.page_state(tid) != PageState.UNMAPPED:
                out.add(tid.layer)
        return out

    def resident_layers(self) -> set:
        return {tid.layer for tid in iter_tensor_ids(self.spec) if self.page_state(tid) == PageState.RESIDENT}

    def check_consistency(self) -> None:
        call("xpgb_pt_check_consistency", self.ctx.handle)
