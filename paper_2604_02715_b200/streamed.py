"""Streamed execution of the paged MoE stack on a B200 (reference pipeline.py:1-483).

Alg. 1 of the paper on CUDA streams instead of threads:

* loader(kind) threads  -> two copy streams (GATE_UP, DOWN), fed by the C++ schedule;
* compute thread        -> one compute stream running route/plan/gather/GEMM/combine;
* threading.Event       -> cudaEvent: RAW = compute waits on both load events of its
  step, WAR = the copy stream waits on the compute event of the layer it recycles;
* OrderingLog           -> device log appended by stream-ordered kernels with a global
  atomic counter, so the record order is the causal order the GPU executed.

``mode="sequential"`` enqueues the same task order but synchronises the host
after every task, the deterministic twin of the reference's inline mode.
"""

from __future__ import annotations

import os

import ctypes as C
import hashlib
import json
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import call
from .device import Context, _torch, as_device_f32, route_table
from .errors import XpgError
from .geometry import ExpertTensorId, ModelSpec, TensorKind, WeightContainer, initial_activations, iter_tensor_ids
from .pagetable import PageTable
from .tiers import StorageHierarchy

ROLE_LOAD = {TensorKind.GATE_UP: "load1", TensorKind.DOWN: "load2"}
ROLE_COMPUTE = "comp"


@dataclass(frozen=True)
class ForwardSpec:
    tokens_per_step: int = 4
    top_k: int = 2
    router_seed: int = 0


@dataclass(frozen=True)
class OrderingRecord:
    t: int
    event: str
    iteration: int
    layer: int
    kind: int | None = None
    target_iteration: int | None = None
    target_layer: int | None = None
    wall: float = 0.0
    group: int = 0                   # sub-layer ring window of the step (0: reference geometry)
    target_group: int | None = None  # recycles: the recycled step's window


def validate_ordering(records) -> list:
    """RAW/WAR replay of an ordering log (pipeline.py:119-147): one message per violation.
    The unit is the (iteration, layer) step -- or, with a sub-layer ring, its window."""
    first = {}
    for r in records:
        first.setdefault((r.event, r.iteration, r.layer, r.group, r.kind), r.t)

    def before(event, it, layer, group, kind, t):
        at = first.get((event, it, layer, group, kind))
        return at is not None and at < t

    def where(it, layer, group):
        return f"iter={it} layer={layer}" + (f" window={group}" if group else "")

    problems = []
    for r in records:
        if r.event == "compute-start":
            problems += [
                f"RAW: compute-start {where(r.iteration, r.layer, r.group)} before load-done kind={k}"
                for k in (1, 2) if not before("load-done", r.iteration, r.layer, r.group, k, r.t)
            ]
        elif r.event == "recycle" and not before("compute-done", r.target_iteration, r.target_layer,
                                                 r.target_group or 0, None, r.t):
            problems.append(f"WAR: recycle of {where(r.target_iteration, r.target_layer, r.target_group or 0)} "
                            f"kind={r.kind} before its compute-done")
    return problems


def _intervals(records) -> dict:
    """{(iteration, layer): {"load1"|"load2"|"compute": (start, done)}}; the windows of a
    sub-layer ring merge into their layer's span (first start .. last done)."""
    spans, opened = {}, {}
    for r in records:
        phase, _, edge = r.event.partition("-")
        if edge == "start":
            opened[(phase, r.iteration, r.layer, r.group, r.kind)] = r.wall
        elif edge == "done":
            t0 = opened.get((phase, r.iteration, r.layer, r.group, r.kind))
            if t0 is not None:
                name = f"load{r.kind}" if phase == "load" else "compute"
                layer = spans.setdefault((r.iteration, r.layer), {})
                a, b = layer.get(name, (t0, r.wall))
                layer[name] = (min(a, t0), max(b, r.wall))
    return spans


@dataclass
class RunReport:
    final_activations: object
    arena_peak_bytes: int
    stall_seconds: float
    war_wait_seconds: float
    violations: list
    records: list
    intervals: dict = field(default_factory=dict)
    page_fault: str | None = None
    # B200 additions
    h2d_bytes: int = 0
    d2d_bytes: int = 0
    copy_busy_seconds: tuple = (0.0, 0.0)
    elapsed_seconds: float = 0.0
    kernels: dict = field(default_factory=dict)
    decoded_bytes: int = 0

    @property
    def checksum(self) -> str:
        a = self.final_activations
        if hasattr(a, "detach"):
            a = a.detach().cpu().numpy()
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

    @property
    def page_in_gbps(self) -> float:
        busy = max(self.copy_busy_seconds) if self.copy_busy_seconds else 0.0
        return (self.h2d_bytes + self.d2d_bytes) / self.elapsed_seconds / 1e9 if self.elapsed_seconds > 0 else 0.0

    @property
    def exposed_fraction(self) -> float:
        return self.stall_seconds / self.elapsed_seconds if self.elapsed_seconds > 0 else 0.0

    def to_json(self) -> str:
        return json.dumps({
            "activation_checksum": self.checksum,
            "stall_ms": self.stall_seconds * 1e3,
            "war_wait_ms": self.war_wait_seconds * 1e3,
            "arena_peak_bytes": self.arena_peak_bytes,
            "violation_count": len(self.violations),
            "violations": self.violations,
            "page_fault": self.page_fault,
            "layer_intervals": {f"iter{it}.layer{ly}": v for (it, ly), v in sorted(self.intervals.items())},
            "h2d_bytes": self.h2d_bytes,
            "d2d_bytes": self.d2d_bytes,
            "elapsed_ms": self.elapsed_seconds * 1e3,
        }, indent=2)


def _records_from_log(ctx: Context):
    n = C.c_int32()
    call("xpgb_log_get", ctx.handle, None, 0, C.byref(n))
    arr = (_lib.Record * max(n.value, 1))()
    call("xpgb_log_get", ctx.handle, arr, n.value, C.byref(n))
    out = []
    t = 0
    base = None
    for i in range(n.value):
        r = arr[i]
        if r.event == _lib.EV_RUN_BEGIN:
            base = r.wall_ns
            continue
        if base is None:
            base = r.wall_ns
        kind = r.kind if r.kind > 0 else None
        out.append(OrderingRecord(
            t=t, event=_lib.EVENT_NAMES[r.event], iteration=r.iteration, layer=r.layer, kind=kind,
            target_iteration=r.target_iteration if r.target_iteration > 0 else None,
            target_layer=r.target_layer if r.target_layer > 0 else None,
            wall=(r.wall_ns - base) * 1e-9, group=r.group & 0xFFFF,
            target_group=((r.group >> 16) & 0xFFFF) if r.target_layer > 0 else None))
        t += 1
    return out


def _run_context(ctx: Context, spec: ModelSpec, fwd: ForwardSpec, iterations: int, acts, sequential: bool,
                 fetch_delay=None, compute_delay=None, sabotage=None, log: bool = True, profile: bool = False):
    torch = _torch()
    x, was_numpy = as_device_f32(acts, ctx.device, fwd.tokens_per_step, spec.hidden_dim)
    y = torch.empty_like(x)
    opts = _lib.RunOpts()
    opts.iterations = iterations
    opts.tokens = fwd.tokens_per_step
    opts.top_k = fwd.top_k
    opts.sequential = 1 if sequential else 0
    opts.router_seed = int(fwd.router_seed) & 0xFFFFFFFFFFFFFFFF
    opts.sabotage_iteration, opts.sabotage_layer = sabotage if sabotage else (0, 0)
    keep = []
    if fetch_delay is not None:
        fd = np.ascontiguousarray(fetch_delay, dtype=np.float32)
        keep.append(fd)
        opts.fetch_delay_s = fd.ctypes.data_as(C.POINTER(C.c_float))
    if compute_delay is not None:
        cd = np.ascontiguousarray(compute_delay, dtype=np.float32)
        keep.append(cd)
        opts.compute_delay_s = cd.ctypes.data_as(C.POINTER(C.c_float))
    opts.log_enable = 1 if log else 0
    opts.profile = int(profile) if not isinstance(profile, bool) else (1 if profile else 0)
    rep = _lib.Report()
    torch.cuda.current_stream(ctx.device).synchronize()
    call("xpgb_run", ctx.handle, C.byref(opts), C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), C.byref(rep))
    out = y.cpu().numpy() if was_numpy else y
    return out, rep


class StreamedRunner:
    """Paged pipeline for n iterations over N layers on one B200."""

    def __init__(self, spec: ModelSpec, hierarchy: StorageHierarchy, fwd: ForwardSpec, mode: str = "threaded",
                 compute_delay_fn=None, sabotage_skip_raw=None, trace=None, device: int = 0,
                 host_codec: bool = False, pinned=None, expert_shard=None, shared_tokens=None,
                 ring_experts=None, stage_buffers=None, ring_depth=None, fused_decode=None, device_format="huffman"):
        """expert_shard=(first, count): this device holds only experts [first, first+count) of
        every layer -- one expert-parallel rank's slice -- and ``hierarchy`` is built on that
        shard's container (ModelSpec(N, count, H, F), shard-local order); the router still
        spans all L experts and rows routed elsewhere are skipped.  shared_tokens=(first,
        count): the step rows that pass through the shared experts (default all).
        ring_experts: a sub-layer ring of that many expert blocks per kind (budgets below the
        reference's two layers; each layer then streams in windows of ring_experts/2).
        ring_depth: windows in flight on that ring (default 2; each window then holds
        ring_experts/ring_depth experts).
        stage_buffers: staging buffers per kind for the compressed host tier (2..16): how far
        the link runs ahead of the decoder.
        fused_decode: device-tier experts are read in place by the GEMM (decoder warps expand
        the records into the tensor-core tiles) instead of being decoded into the ring first;
        default off (XPGB_FUSED=1 turns it on).  Results are bit-identical either way.
        device_format: records of the compressed device tier -- "huffman" (the reference's
        exponent-Huffman, smallest) or "fx4" (fixed-width exponent offsets, fx4.cuh: ~13% more HBM,
        no serial decode chain, so the fused GEMM expands them near bandwidth)."""
        if mode not in ("threaded", "sequential"):
            raise XpgError(f"unknown mode {mode!r}")
        self.spec = spec
        self.hierarchy = hierarchy
        self.fwd = fwd
        self.mode = mode
        self.compute_delay_fn = compute_delay_fn
        self.sabotage_skip_raw = sabotage_skip_raw
        first, count = expert_shard if expert_shard is not None else (0, spec.experts_per_layer)
        self.ctx = Context(spec, _lib.POOL_RING, device, max_tokens=fwd.tokens_per_step, expert_shard=(first, count))
        self.ctx.attach_host_pool(hierarchy.container.pinned)
        if getattr(hierarchy.container, "shared", None) is not None:
            self.ctx.set_shared(hierarchy.container.shared)
        if shared_tokens is not None:
            self.ctx.set_shared_tokens(*shared_tokens)
        placement = _full_width(spec, hierarchy.backend_map(), first, count)
        cm = _codec_model(hierarchy, host_codec or bool(placement.any()))
        if cm is not None:
            # compressed tiers (codec.py): device-tier tensors live compressed in HBM; with
            # host_codec the host tier also ships compressed records over PCIe.  Both are
            # decoded on the GPU straight into the ring block.
            self.ctx.set_codec(cm, host_compressed=host_codec)
        if stage_buffers is not None:
            self.ctx.set_stage_buffers(int(stage_buffers))
        if fused_decode is None:
            fused_decode = os.environ.get("XPGB_FUSED", "0") == "1"
        self.ctx.set_fused_decode(bool(fused_decode))
        self.device_format = device_format
        if device_format != "huffman":
            self.ctx.set_device_format(device_format)
        self.ctx.set_placement(placement)
        if ring_depth is not None:
            self.ctx.set_ring_depth(int(ring_depth))
        if ring_experts is not None:
            self.ctx.set_ring_experts(int(ring_experts))
        if pinned is not None:
            # residency tier x > 0: these experts never leave HBM; the ring streams the rest
            self.ctx.set_pinned(pinned_mask(spec, pinned, first, count))
        self.table = PageTable(spec, trace=trace, context=self.ctx)
        self.stall_seconds = 0.0
        self.war_wait_seconds = 0.0
        self.host_codec = host_codec
        self._shard = (first, count)
        self._codec_on = cm is not None
        self.device_experts = None  # per-layer device-tier experts once set_device_experts ran

    # ---- residency control (residency.LiveResidencyController)
    def _compressed(self):
        cm = _codec_model(self.hierarchy, True)
        if not self._codec_on:
            self.ctx.set_codec(cm, host_compressed=self.host_codec)
            self._codec_on = True
        return cm

    def device_tier_bytes(self, m: int) -> int:
        """HBM bytes of the device tier holding experts 1..m of every layer (compressed records)."""
        spec, total = self.hierarchy.container.spec, 0
        if self.device_format == "fx4":
            # fx4.cuh layout with no escapes (N(0, s) weights escape ~1e-4 of values; the exact
            # size after staging is ctx.hbm_bytes()["device_tier"])
            r16 = lambda x: (x + 15) // 16 * 16
            for tid in iter_tensor_ids(spec):
                if tid.expert <= m:
                    n = spec.value_count(tid.kind)
                    total += r16(n) + r16(n // 2) + r16(4 * (n // 256 + 1)) + 16 + 256
            return total
        cm = self._compressed()
        from ._lib import lib

        for i, tid in enumerate(iter_tensor_ids(spec)):
            if tid.expert <= m:
                total += int(lib().xpgb_codec_record_bytes(spec.value_count(tid.kind), int(cm.bits_lens[i]),
                                                           int(cm.chunk)))
        return total

    def set_device_mask(self, mask) -> None:
        """Placement by an explicit bool [N][L] mask of device-tier experts (the reference's
        alpha split puts experts 1..m there; spreading them lets every window of a sub-layer
        ring mix device-tier and host-tier experts, so the link never idles on a window)."""
        spec = self.hierarchy.container.spec
        mask = np.asarray(mask, dtype=bool).reshape(spec.num_layers, spec.experts_per_layer)
        if mask.any():
            self._compressed()
        shard_map = np.repeat(mask[:, :, None], 2, axis=2).astype(np.uint8)
        first, count = self._shard
        self.ctx.set_placement(_full_width(self.spec, shard_map, first, count))
        self.device_experts = [int(v) for v in mask.sum(axis=1)]

    def set_device_format(self, device_format: str, fused_decode: bool | None = None) -> None:
        """Switch the device tier's record format ("huffman" / "fx4", re-staging it) and,
        optionally, decode-into-GEMM for the builtin compute."""
        self.ctx.set_device_format(device_format)
        self.device_format = device_format
        if fused_decode is not None:
            self.ctx.set_fused_decode(bool(fused_decode))

    def apply_plan(self, plan) -> None:
        """Apply a budget.ResidencyPlan -- pinned experts, ring size and depth, device-tier
        experts (and, for budget.plan_tiers plans, the device tier's record format and
        decode-into-GEMM) -- replacing whatever residency state an earlier plan left."""
        spec = self.hierarchy.container.spec
        first, count = self._shard
        fmt = getattr(plan, "device_format", None)
        if fmt == "mixed":
            # per-expert record format (both tensors of an expert alike), FX4 read in place
            fx4 = np.zeros((self.spec.num_layers, self.spec.experts_per_layer), dtype=bool)
            fx4[:, first:first + count] = np.asarray(plan.fx4_mask).reshape(spec.num_layers, spec.experts_per_layer)
            self.ctx.set_device_formats(np.repeat(fx4[:, :, None], 2, axis=2))
            self.device_format = "mixed"
        elif fmt and fmt != self.device_format:
            self.set_device_format(fmt)
        if getattr(plan, "fused", None) is not None:
            self.ctx.set_fused_decode(int(plan.fused))
        full = np.zeros((self.spec.num_layers, self.spec.experts_per_layer), dtype=np.uint8)
        full[:, first:first + count] = plan.pinned_mask.reshape(spec.num_layers, spec.experts_per_layer)
        streamed = spec.experts_per_layer - plan.pinned_mask.sum(axis=1).min()
        depth = getattr(plan, "depth", 2)
        # a ring below the reference's two layers, or any ring with one window in flight
        sub = 0 < plan.ring and (plan.ring < 2 * streamed or depth != 2)
        self.ctx.apply_residency(full, int(plan.ring) if sub else 0, depth)
        self.set_device_mask(plan.device_mask)
        if self.host_codec:
            # no expert left on the host tier: the staging ring and chunk index go back to the budget
            host = int(plan.device_mask.size - plan.device_mask.sum() - plan.pinned_mask.sum())
            self.ctx.set_host_staging(host > 0)

    def set_device_experts(self, m_layers) -> None:
        """Placement: experts 1..m_l of layer l on the compressed device tier, the rest on the
        host tier (the reference's alpha split per layer, storage.py:143-168).  Re-stages the
        device tier between runs; results are unchanged (the codec is lossless)."""
        spec = self.hierarchy.container.spec
        m_layers = [int(m) for m in m_layers]
        if len(m_layers) != spec.num_layers or min(m_layers) < 0 or max(m_layers) > spec.experts_per_layer:
            raise XpgError(f"bad per-layer device experts {m_layers}")
        if any(m_layers):
            self._compressed()
        shard_map = np.zeros((spec.num_layers, spec.experts_per_layer, 2), dtype=np.uint8)
        for l, m in enumerate(m_layers):
            shard_map[l, :m] = 1
        first, count = self._shard
        self.ctx.set_placement(_full_width(self.spec, shard_map, first, count))
        self.device_experts = m_layers

    def run(self, iterations: int, acts=None, profile: bool = False) -> RunReport:
        if iterations < 1:
            raise XpgError("need at least one iteration")
        if acts is None:
            acts = initial_activations(self.spec, self.fwd, 0)
        cd = None
        if self.compute_delay_fn is not None:
            cd = np.array([[self.compute_delay_fn(it, ly) for ly in range(1, self.spec.num_layers + 1)]
                           for it in range(1, iterations + 1)], dtype=np.float32)
        out, rep = _run_context(self.ctx, self.spec, self.fwd, iterations, acts, self.mode == "sequential",
                                fetch_delay=self.hierarchy.delay_table(), compute_delay=cd,
                                sabotage=self.sabotage_skip_raw, profile=profile)
        return self._report(out, rep)

    def _report(self, out, rep) -> RunReport:
        self.table.sync_trace()
        records = _records_from_log(self.ctx)
        self.stall_seconds = rep.stall_ns * 1e-9
        self.war_wait_seconds = rep.war_wait_ns * 1e-9
        return RunReport(
            final_activations=out,
            arena_peak_bytes=int(rep.arena_peak_bytes),
            stall_seconds=self.stall_seconds,
            war_wait_seconds=self.war_wait_seconds,
            violations=validate_ordering(records),
            records=records,
            intervals=_intervals(records),
            page_fault=self.ctx.fault() if rep.page_fault else None,
            h2d_bytes=int(rep.h2d_bytes),
            d2d_bytes=int(rep.d2d_bytes),
            copy_busy_seconds=(rep.copy_busy_ns[0] * 1e-9, rep.copy_busy_ns[1] * 1e-9),
            elapsed_seconds=rep.elapsed_ns * 1e-9,
            kernels=_kernel_stats(rep),
            decoded_bytes=int(rep.decoded_bytes),
        )

    def open_session(self, max_iterations: int, log: bool = True) -> "DecodeSession":
        """A serving session: ``step(acts)`` runs one decode iteration on new activations while
        the copy streams keep prefetching the next iteration's first layers in the background."""
        return DecodeSession(self, max_iterations, log=log)


class DecodeSession:
    """One long schedule of up to ``max_iterations`` decode steps, fed one step at a time.

    ``run(iterations)`` starts every call from an empty ring, so the first two layers of
    each call page in with nothing to overlap.  A session keeps the schedule open between
    calls: while the caller prepares step i+1 (attention, sampling), layers 1-2 of step
    i+1 are already paging in -- the reference's lookahead carried across decode steps.
    Each step copies its inputs into the device activation buffer on the library's compute
    stream (H2D from pinned memory when given a pinned tensor), runs the step's layers, and
    copies the output back (``out=`` pinned tensor, or a new numpy array).
    """

    def __init__(self, runner: StreamedRunner, max_iterations: int, log: bool = True):
        torch = _torch()
        if max_iterations < 1:
            raise XpgError("need at least one iteration")
        self.runner, self.max_iterations = runner, max_iterations
        spec, fwd, ctx = runner.spec, runner.fwd, runner.ctx
        self.acts = torch.zeros(fwd.tokens_per_step, spec.hidden_dim, dtype=torch.float32,
                                device=f"cuda:{ctx.device}")
        opts = _lib.RunOpts()
        opts.iterations = max_iterations
        opts.tokens = fwd.tokens_per_step
        opts.top_k = fwd.top_k
        opts.router_seed = int(fwd.router_seed) & 0xFFFFFFFFFFFFFFFF
        opts.log_enable = 1 if log else 0
        opts.fresh_inputs = 1
        h = ctx.handle
        call("xpgb_session_begin", h, C.byref(opts), C.c_void_p(self.acts.data_ptr()))
        total, per_it, stream = C.c_int32(), C.c_int32(), C.c_void_p()
        call("xpgb_session_info", h, C.byref(total), C.byref(per_it), C.byref(stream))
        self.steps_total, self.steps_per_iteration = total.value, per_it.value
        self._stream_ptr = stream.value
        self.stream = torch.cuda.ExternalStream(stream.value, device=f"cuda:{ctx.device}")
        self.g = 0
        self.iteration = 0
        self.closed = False
        try:
            call("xpgb_session_materialize", h, 0)
            call("xpgb_session_materialize", h, 1)
        except Exception:
            _lib.lib().xpgb_session_abort(h)
            raise

    def step(self, acts, out=None):
        torch = _torch()
        if self.closed:
            raise XpgError("session is closed")
        if self.iteration >= self.max_iterations:
            raise XpgError(f"session holds {self.max_iterations} iterations")
        h = self.runner.ctx.handle
        src = torch.from_numpy(np.ascontiguousarray(acts, dtype=np.float32)) if isinstance(acts, np.ndarray) else acts
        # host copies run on torch's stream (its pinned-memory allocator tracks only its own
        # streams) and are ordered against the library's compute stream by events
        cur = torch.cuda.current_stream(self.acts.device)
        self.acts.copy_(src, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(cur)
        self.stream.wait_event(ev)
        try:  # the iteration's steps in one call (acquire / compute / release / materialize(g+2))
            call("xpgb_session_run_steps", h, self.g, self.steps_per_iteration, C.c_void_p(self._stream_ptr))
            self.g += self.steps_per_iteration
        except Exception:
            self.closed = True  # the library aborted the session
            raise
        self.iteration += 1
        dst = out if out is not None else torch.empty(self.acts.shape, dtype=torch.float32,
                                                      pin_memory=True)
        done = torch.cuda.Event()
        done.record(self.stream)
        cur.wait_event(done)
        dst.copy_(self.acts, non_blocking=True)
        cur.synchronize()
        return dst if out is not None else dst.numpy()

    def close(self) -> RunReport:
        """End the schedule (pages still bound are released) and report over the steps run."""
        if self.closed:
            raise XpgError("session is closed")
        rep = _lib.Report()
        call("xpgb_session_end", self.runner.ctx.handle, C.byref(rep))
        self.closed = True
        return self.runner._report(self.acts, rep)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        if not self.closed:
            if exc[0] is None:
                self.close()
            else:
                _lib.lib().xpgb_session_abort(self.runner.ctx.handle)
                self.closed = True


def _kernel_stats(rep) -> dict:
    return {
        "gate_up_ns": rep.kern_gate_up_ns, "down_ns": rep.kern_down_ns, "aux_ns": rep.kern_aux_ns,
        "gate_up_bytes": int(rep.gate_up_bytes), "down_bytes": int(rep.down_bytes),
        "down_splits": int(rep.down_splits), "active_experts": int(rep.active_experts),
    }


def _full_width(spec: ModelSpec, shard_map: np.ndarray, first: int, count: int) -> np.ndarray:
    """A shard's [N][count][2] placement map widened to the context's [N][L][2] indexing."""
    if count == spec.experts_per_layer:
        return shard_map
    out = np.zeros((spec.num_layers, spec.experts_per_layer, 2), dtype=np.uint8)
    out[:, first:first + count] = shard_map.reshape(spec.num_layers, count, 2)
    return out


def pinned_mask(spec: ModelSpec, pinned, first: int = 0, count: int | None = None) -> np.ndarray:
    """uint8 [N][L] mask: an int m pins the first m experts (of the shard) of every layer;
    arrays pass through."""
    if isinstance(pinned, (int, np.integer)):
        m = np.zeros((spec.num_layers, spec.experts_per_layer), dtype=np.uint8)
        m[:, first:first + int(pinned)] = 1
        return m
    m = np.asarray(pinned, dtype=np.uint8).reshape(spec.num_layers, spec.experts_per_layer)
    return np.ascontiguousarray(m)


def _codec_model(hierarchy: StorageHierarchy, needed: bool):
    """The hierarchy's CompressedModel (built on demand) when a compressed tier is in use."""
    if not needed:
        return None
    from .exponent_codec import CompressedModel

    cm = hierarchy.compressed
    if not isinstance(cm, CompressedModel):
        cm = CompressedModel.from_container(hierarchy.container)
        hierarchy.compressed = cm
    return cm


def run_iterations(iterations: int, spec: ModelSpec, hierarchy: StorageHierarchy, fwd: ForwardSpec,
                   mode: str = "threaded", acts=None, **runner_kwargs) -> RunReport:
    return StreamedRunner(spec, hierarchy, fwd, mode=mode, **runner_kwargs).run(iterations, acts=acts)


class ResidentModel:
    """Every expert tensor of a container resident in HBM (one block per tensor).

    The fully-resident comparator: the same kernels read the same device slot
    table, which simply never changes (pipeline.py:216-230).
    """

    def __init__(self, spec: ModelSpec, container: WeightContainer, device: int = 0, max_tokens: int = 16,
                 expert_shard=None, shared_tokens=None):
        self.spec = spec
        self.container = container
        # container = the shard's payload when expert_shard is set (see StreamedRunner)
        self.ctx = Context(spec, _lib.POOL_RESIDENT, device, max_tokens=max_tokens, expert_shard=expert_shard)
        self.ctx.attach_host_pool(container.pinned)
        self.ctx.make_resident()
        if getattr(container, "shared", None) is not None:
            self.ctx.set_shared(container.shared)
        if shared_tokens is not None:
            self.ctx.set_shared_tokens(*shared_tokens)

    def forward(self, layer: int, acts, fwd: ForwardSpec):
        torch = _torch()
        x, was_numpy = as_device_f32(acts, self.ctx.device, acts.shape[0], self.spec.hidden_dim)
        y = torch.empty_like(x)
        self.ctx.clear_fault()
        self.ctx.layer_forward(layer, x, y, x.shape[0], fwd.top_k, fwd.router_seed)
        fault = self.ctx.fault()
        if fault:
            from .errors import PageFaultError

            raise PageFaultError(fault)
        return y.cpu().numpy() if was_numpy else y

    def run(self, iterations: int, fwd: ForwardSpec, acts, log: bool = False, profile: bool = False):
        return _run_context(self.ctx, self.spec, fwd, iterations, acts, sequential=False, log=log, profile=profile)


_RESIDENT_CACHE: dict = {}


def _resident_for(spec: ModelSpec, weights_of) -> ResidentModel:
    if isinstance(weights_of, ResidentModel):
        return weights_of
    owner = getattr(weights_of, "__self__", None)
    if isinstance(owner, WeightContainer):
        key = id(owner)
        hit = _RESIDENT_CACHE.get(key)
        if hit is None or hit[0] is not owner:
            hit = (owner, ResidentModel(spec, owner))
            _RESIDENT_CACHE.clear()
            _RESIDENT_CACHE[key] = hit
        return hit[1]
    # generic callable: materialise bf16 words of every tensor (exact for bf16-valued weights)
    from .geometry import float32_to_bf16, tensor_offset

    words = np.zeros(spec.total_bytes // 2, dtype=np.uint16)
    for tid in iter_tensor_ids(spec):
        w = np.asarray(weights_of(tid), dtype=np.float32).reshape(-1)
        off = tensor_offset(tid, spec) // 2
        words[off:off + w.size] = float32_to_bf16(w)
    return ResidentModel(spec, WeightContainer(spec, words))


def layer_forward(weights_of, spec: ModelSpec, fwd: ForwardSpec, layer: int, acts):
    """One MoE layer (pipeline.py:192-208) on the GPU.

    ``weights_of`` may be a ``ResidentModel``, a ``PageTable`` whose layer
    pages are RESIDENT, ``WeightContainer.tensor_f32`` (as in the reference's
    ``resident_baseline``), or any tid -> float32 matrix callable.
    """
    if isinstance(weights_of, PageTable):
        torch = _torch()
        ctx = weights_of.ctx
        x, was_numpy = as_device_f32(acts, ctx.device, np.shape(acts)[0], spec.hidden_dim)
        y = torch.empty_like(x)
        ctx.clear_fault()
        ctx.layer_forward(layer, x, y, x.shape[0], fwd.top_k, fwd.router_seed)
        fault = ctx.fault()
        if fault:
            from .errors import PageFaultError

            raise PageFaultError(fault)
        return y.cpu().numpy() if was_numpy else y
    model = _resident_for(spec, weights_of)
    return model.forward(layer, acts, fwd)


def resident_baseline(iterations: int, spec: ModelSpec, container, fwd: ForwardSpec, acts=None):
    """Fully-resident oracle path on the GPU: same kernels, every page resident."""
    if acts is None:
        acts = initial_activations(spec, fwd, 0)
    model = container if isinstance(container, ResidentModel) else _resident_for(spec, container.tensor_f32)
    out, _ = model.run(iterations, fwd, acts)
    return out


def routed_experts(seed: int, token: int, layer: int, num_experts: int, top_k: int, device: int = 0):
    """Experts of one token (ascending, 1-based) from the GPU router kernel."""
    tab = route_table(seed, token + 1, 1, num_experts, top_k, device=device, layer_first=layer)
    return [int(v) for v in tab[0, token].tolist()]
