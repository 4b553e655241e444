"""Thin owner of one ``xpgb_ctx`` (one device, one pool) plus tensor plumbing.

PyTorch is used only for device/pinned memory and the current CUDA stream;
every computation is a libxpgb kernel launched through the C ABI.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import call, lib
from .errors import OutOfRangeError, XpgError
from .geometry import ModelSpec


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise XpgError("no CUDA device: the B200 expert-paging path has no CPU fallback")
    return torch


def current_stream_ptr(device: int = 0) -> int:
    torch = _torch()
    return int(torch.cuda.current_stream(device).cuda_stream)


def as_device_f32(acts, device: int, rows: int, cols: int):
    """(tensor, was_numpy): a contiguous float32 CUDA tensor holding acts."""
    torch = _torch()
    if isinstance(acts, torch.Tensor):
        t = acts
        if t.device.type != "cuda":
            t = t.to(f"cuda:{device}", non_blocking=False)
        t = t.to(torch.float32).contiguous()
        was_numpy = False
    else:
        arr = np.ascontiguousarray(np.asarray(acts, dtype=np.float32))
        t = torch.from_numpy(arr).to(f"cuda:{device}")
        was_numpy = True
    if tuple(t.shape) != (rows, cols):
        raise OutOfRangeError(f"activations have shape {tuple(t.shape)}, expected {(rows, cols)}")
    return t, was_numpy


class Context:
    """One libxpgb context: pools, page table, streams, workspaces."""

    def __init__(self, spec: ModelSpec, pool: int = _lib.POOL_RING, device: int = 0, max_tokens: int = 16,
                 expert_shard=None):
        """expert_shard=(first, count): hold only those experts of every layer from the start."""
        _torch()
        self.spec = spec
        self.device = device
        self.pool = pool
        first, count = expert_shard if expert_shard is not None else (0, spec.experts_per_layer)
        self.expert_first, self.expert_count = int(first), int(count)
        s = _lib.Spec(spec.num_layers, spec.experts_per_layer, spec.hidden_dim, spec.intermediate_dim)
        h = C.c_void_p()
        call("xpgb_create_shard", C.byref(s), device, pool, max(1, int(max_tokens)), self.expert_first,
             self.expert_count, C.byref(h))
        self._h = h
        self._host_ref = None
        self._ring, self._depth = -1, 2  # mirror of the context's ring limit / depth

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().xpgb_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover - GC timing
        try:
            self.close()
        except Exception:
            pass

    # ---- storage
    def attach_host_pool(self, pinned_u8) -> None:
        """Use a (pinned) torch uint8 tensor holding this shard's payload as the host pool."""
        call("xpgb_host_pool_register", self._h, C.c_void_p(pinned_u8.data_ptr()), C.c_uint64(pinned_u8.numel()))
        self._host_ref = pinned_u8

    def set_placement(self, backend_of: np.ndarray) -> None:
        arr = np.ascontiguousarray(backend_of, dtype=np.uint8)
        call("xpgb_set_placement", self._h, arr.ctypes.data_as(C.POINTER(C.c_uint8)))

    def set_codec(self, cm, host_compressed: bool) -> None:
        """Attach a CompressedModel (exponent_codec) of this context's tensors."""
        p64 = C.POINTER(C.c_uint64)
        offs = np.ascontiguousarray(cm.rec_offsets, dtype=np.uint64)
        bits = np.ascontiguousarray(cm.bits_lens, dtype=np.uint64)
        lengths = cm.table.lengths_array()
        call("xpgb_set_codec", self._h, C.c_void_p(cm.pool.data_ptr()), C.c_uint64(cm.pool.numel()),
             offs.ctypes.data_as(p64), bits.ctypes.data_as(p64), lengths.ctypes.data_as(C.POINTER(C.c_uint8)),
             int(cm.chunk), 1 if host_compressed else 0)
        self._codec_ref = cm

    def set_expert_shard(self, first: int, count: int) -> None:
        call("xpgb_set_expert_shard", self._h, first, count)
        self.expert_first, self.expert_count = first, count

    def set_shared(self, shared) -> None:
        """Attach a geometry.SharedExperts (or None to remove): always-on, always-resident experts."""
        if shared is None:
            call("xpgb_set_shared", self._h, None, C.c_uint64(0), 0)
        else:
            call("xpgb_set_shared", self._h, C.c_void_p(shared.pinned.data_ptr()), C.c_uint64(shared.total_bytes),
                 int(shared.count))
        self._shared_ref = shared

    def set_shared_tokens(self, first: int = 0, count: int = -1) -> None:
        """Step rows [first, first+count) pass through the shared experts (count < 0: all)."""
        call("xpgb_set_shared_tokens", self._h, int(first), int(count))

    def set_ring_experts(self, ring_experts: int) -> None:
        """Sub-layer ring of ``ring_experts`` blocks per kind (-1: the reference's two layers)."""
        call("xpgb_set_ring_experts", self._h, int(ring_experts))
        self._ring = int(ring_experts)

    def set_ring_depth(self, depth: int) -> None:
        """Windows in flight on a sub-layer ring (window g recycles g - depth)."""
        call("xpgb_set_ring_depth", self._h, int(depth))
        self._depth = int(depth)

    def apply_residency(self, pinned_full, ring: int, depth: int) -> None:
        """Set a whole residency state from any previous one: the pinned mask [N][L] (always
        applied, so an empty mask clears earlier pins), then ring depth and size in the order
        the context accepts (a ring is never smaller than the depth in flight).  ring <= 0:
        the reference's two-layer ring at depth 2."""
        self.set_pinned(pinned_full)
        if ring <= 0:
            if self._ring != -1:
                self.set_ring_experts(-1)
            if self._depth != 2:
                self.set_ring_depth(2)
            return
        if ring >= self._depth:
            self.set_ring_experts(ring)
            self.set_ring_depth(depth)
        else:
            self.set_ring_depth(depth)
            self.set_ring_experts(ring)

    def set_hazard_checks(self, poison: bool = False, skip_war=None) -> None:
        """Debug: poison mapped ring blocks with NaN bytes; skip_war=(iteration, layer) drops
        that load's WAR wait (the WAR twin of the reference's RAW sabotage)."""
        it, layer = skip_war if skip_war else (0, 0)
        call("xpgb_set_hazard_checks", self._h, 1 if poison else 0, int(it), int(layer))

    def set_device_format(self, fmt: str) -> None:
        """Compressed device-tier records: "huffman" (the reference's codec) or "fx4" (fixed-width
        exponent offsets, fx4.cuh) -- re-stages the device tier."""
        if fmt not in ("huffman", "fx4"):
            raise XpgError(f"unknown device-tier format {fmt!r}")
        call("xpgb_set_device_format", self._h, 1 if fmt == "fx4" else 0)
        self._dev_fmt = fmt

    def set_device_formats(self, fx4_mask: np.ndarray) -> None:
        """Per-tensor device-tier format: ``fx4_mask`` [layers, experts, 2] (gate/up, down) true
        where the record is FX4, false for exponent-Huffman (xpgb_set_device_formats)."""
        arr = np.ascontiguousarray(fx4_mask, dtype=np.uint8)
        call("xpgb_set_device_formats", self._h, arr.ctypes.data_as(C.POINTER(C.c_uint8)))
        self._dev_fmt = "mixed" if 0 < arr.sum() < arr.size else ("fx4" if arr.size and arr.all() else "huffman")

    def set_host_staging(self, on: bool) -> None:
        """Allocate / release the compressed host tier's staging ring and chunk index."""
        call("xpgb_set_host_staging", self._h, 1 if on else 0)

    def set_fused_decode(self, on) -> None:
        """Decode-into-GEMM for the builtin compute: device-tier experts read in place
        (True / 1); 2 = only FX4 records in place, Huffman records decoded into the ring."""
        call("xpgb_set_fused_decode", self._h, int(on))

    def set_activation_planes(self, planes: int) -> None:
        """Activation planes of the decode-sized GEMMs: 2 (hi + lo, fp32-like; default) or 1
        (bf16 activations, half the MMAs) -- xpgb_set_activation_planes."""
        call("xpgb_set_activation_planes", self._h, int(planes))

    def set_stage_buffers(self, n: int) -> None:
        """Staging ring of the compressed host tier: ``n`` buffers per kind (link run-ahead)."""
        call("xpgb_set_stage_buffers", self._h, int(n))

    def set_pinned(self, mask: np.ndarray) -> None:
        arr = np.ascontiguousarray(mask, dtype=np.uint8)
        call("xpgb_set_pinned", self._h, arr.ctypes.data_as(C.POINTER(C.c_uint8)))

    def hbm_bytes(self) -> dict:
        r, st, dt = C.c_uint64(), C.c_uint64(), C.c_uint64()
        call("xpgb_hbm_bytes", self._h, C.byref(r), C.byref(st), C.byref(dt))
        return {"ring": int(r.value), "staging": int(st.value), "device_tier": int(dt.value)}

    def decode_stats(self) -> dict:
        """Exponent-decoder launches of the last profiled run (xpgb_decode_stats)."""
        n, ns, b = C.c_int64(), C.c_double(), C.c_int64()
        call("xpgb_decode_stats", self._h, C.byref(n), C.byref(ns), C.byref(b))
        return {"launches": int(n.value), "kernel_ns": float(ns.value), "algo_bytes": int(b.value)}

    def fused_stats(self) -> dict:
        """Decode-into-GEMM launches of the last profiled run (xpgb_fused_stats)."""
        n, ns, b = C.c_int64(), C.c_double(), C.c_int64()
        call("xpgb_fused_stats", self._h, C.byref(n), C.byref(ns), C.byref(b))
        return {"launches": int(n.value), "kernel_ns": float(ns.value), "record_bytes": int(b.value)}

    def make_resident(self) -> None:
        call("xpgb_make_resident", self._h)

    # ---- compute
    def layer_forward(self, layer: int, x, y, tokens: int, top_k: int, seed: int, stream: int | None = None):
        st = current_stream_ptr(self.device) if stream is None else stream
        call("xpgb_layer_forward", self._h, layer, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), tokens,
             top_k, C.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), C.c_void_p(st))

    def fault_ptr(self) -> int:
        """Device address of the context's fault word (int64; 0 = no fault)."""
        p = C.c_void_p()
        call("xpgb_fault_ptr", self._h, C.byref(p))
        return int(p.value or 0)

    def fault(self):
        f = C.c_int32()
        buf = C.create_string_buffer(512)
        call("xpgb_fault_get", self._h, C.byref(f), buf, 512)
        return (buf.value.decode() if f.value else None)

    def clear_fault(self):
        call("xpgb_fault_clear", self._h)

    def profile_layer(self, layer: int, x, y, tokens: int, top_k: int, seed: int, reps: int = 5):
        kt = _lib.KernelTimes()
        call("xpgb_profile_layer", self._h, layer, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), tokens,
             top_k, C.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), reps, C.byref(kt))
        return {name: getattr(kt, name) for name, _ in _lib.KernelTimes._fields_}

    def sync(self):
        call("xpgb_sync", self._h)


def kernel_launches() -> int:
    return int(lib().xpgb_kernel_launches())


def route_table(seed: int, tokens: int, num_layers: int, num_experts: int, top_k: int, device: int = 0,
                layer_first: int = 1):
    """Routing of layers [layer_first, layer_first+num_layers) as an int32 CUDA tensor [n, T, min(k, L)]."""
    torch = _torch()
    kk = min(top_k, num_experts)
    out = torch.empty((num_layers, tokens, kk), dtype=torch.int32, device=f"cuda:{device}")
    call("xpgb_route", C.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), layer_first, num_layers, tokens, num_experts,
         top_k, C.c_void_p(out.data_ptr()), C.c_void_p(current_stream_ptr(device)))
    return out
