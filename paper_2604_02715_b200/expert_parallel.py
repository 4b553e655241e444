"""Expert parallelism over G GPUs: one rank per GPU, experts sharded contiguously.

No reference counterpart (the reference is single-process).  The
partition follows the north star: rank r owns experts
``[first_r, first_r + count_r)`` of every layer — its own HBM ring, its own
pinned host pool holding only its shard, its own copy streams — and a layer
exchanges tokens twice:

* dispatch: each (token, routed expert) row goes, as bf16, to the expert's owner;
* combine: the owner's fp32 expert outputs come back and the token's owner sums
  them in ascending expert order with weight f32(1/top_k) (pipeline.py:198-207).

Rank r's T tokens are rows ``[r*T, (r+1)*T)`` of the global step batch, so the
router's token index is the global row and a G-rank step computes exactly what
one GPU computes on the concatenated batch.  The router is a pure function of
(seed, token, layer), so every rank computes the global routing table locally
and derives send/receive counts and every permutation from it — no count
exchange.  The exchange itself is ``all_to_all_single`` (NCCL over NVLink on
GPUs, gloo in the CPU tests); the expert GEMMs are libxpgb's tcgen05 kernels.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import XpgError
from ._lib import call
from .geometry import ModelSpec, tensor_offset, ExpertTensorId, TensorKind
from .streamed import ForwardSpec, RunReport, _kernel_stats, _records_from_log, _intervals, validate_ordering


def shard_bounds(num_experts: int, world: int):
    """Contiguous, balanced expert blocks: [(first, count)] per rank (0-based first)."""
    base, rem = divmod(num_experts, world)
    out, first = [], 0
    for r in range(world):
        n = base + (1 if r < rem else 0)
        out.append((first, n))
        first += n
    return out


def shard_payload(container, first: int, count: int):
    """Pinned uint8 tensor with experts [first, first+count) of every layer, in
    shard-local container order (layer, local expert, kind)."""
    from .geometry import _pinned_bytes

    spec = container.spec
    eb = spec.expert_bytes
    out = _pinned_bytes(spec.num_layers * count * eb, True)
    for layer in range(1, spec.num_layers + 1):
        src = tensor_offset(ExpertTensorId(layer, first + 1, TensorKind.GATE_UP), spec)
        dst = (layer - 1) * count * eb
        out[dst:dst + count * eb].copy_(container.pinned[src:src + count * eb])
    return out


@dataclass
class DispatchPlan:
    """Index bookkeeping of one layer's dispatch/combine on one rank (torch tensors)."""

    send_counts: list      # rows this rank sends to each rank
    recv_counts: list      # rows this rank receives from each rank
    send_rows: object      # [n_send] local token row of each sent pair, in send order
    to_expert: object      # [n_recv] arrival index of each expert-major row
    from_expert: object    # [n_recv] expert-major index of each arrival row
    offsets: object        # [count+1] expert-major row offsets of the local experts (int32)
    ret_index: object      # [T, kk] position of each (token, slot) in the returned buffer (int32)
    # peer-memory exchange (PeerExchange): where each row goes, computed from the global routing
    p2p_src_rows: object = None   # [T*kk] local token of each of my pairs, in send order (int32)
    p2p_dst_rank: object = None   # [T*kk] owner rank of each of my pairs
    p2p_dst_row: object = None    # [T*kk] its row in the owner's expert-major input
    c_rank: object = None         # [n_own] token-owner rank of each of my expert-major rows
    c_row: object = None          # [n_own] its row in that rank's return buffer (= its send position)
    # a plan built on the device (DevicePlanner): c_* / to_expert / from_expert are sized for the
    # worst case and n_own lives in counts[2*world]; the host counts are read only when the NCCL
    # transport needs split sizes (one device->host copy per layer)
    counts: object = None         # int32 [2*world+1] device: sent to r, received from r, n_own
    cap_rows: int = 0             # upper bound of n_own (rows of the c_* buffers)

    @property
    def n_dev(self):
        """Device pointer of n_own (None for a host-built plan)."""
        return None if self.counts is None else self.counts.data_ptr() + 4 * (self.counts.numel() - 1)

    def resolve_counts(self) -> None:
        """Host split sizes of a device plan (NCCL transport only: synchronises once)."""
        if self.send_counts is None:
            c = [int(v) for v in self.counts.tolist()]
            G = (len(c) - 1) // 2
            self.send_counts, self.recv_counts, n_own = c[:G], c[G:2 * G], c[2 * G]
            self.to_expert = self.to_expert[:n_own].to(self.send_rows.dtype)
            self.from_expert = self.from_expert[:n_own].to(self.send_rows.dtype)


def build_plan(routes, rank: int, world: int, tokens: int, bounds) -> DispatchPlan:
    """routes: [world*tokens, kk] int tensor of 1-based ids (ascending per row)."""
    import torch

    dev = routes.device
    G, T = world, tokens
    kk = routes.shape[1]
    L = sum(n for _, n in bounds)
    owner = torch.empty(L, dtype=torch.int64, device=dev)
    for r, (f, n) in enumerate(bounds):
        owner[f:f + n] = r
    e0 = routes.to(torch.int64) - 1                      # [G*T, kk] 0-based expert
    dst = owner[e0]                                      # owner rank per pair
    g_tok = torch.arange(G * T, device=dev).unsqueeze(1).expand(G * T, kk)
    slot = torch.arange(kk, device=dev).unsqueeze(0).expand(G * T, kk)
    src = g_tok // T
    local_tok = g_tok - src * T
    # canonical pair order inside a (src -> dst) message: (expert, local token, slot)
    inner = (e0 * T + local_tok) * kk + slot
    span = L * T * kk

    # ---- send side: my tokens, ordered by (dst, expert, token, slot)
    mine = slice(rank * T, (rank + 1) * T)
    key = (dst[mine] * span + inner[mine]).reshape(-1)
    send_order = torch.argsort(key, stable=True)
    send_counts = torch.bincount(dst[mine].reshape(-1), minlength=G)
    send_rows = (send_order // kk)
    ret_index = torch.empty(T * kk, dtype=torch.int64, device=dev)
    ret_index[send_order] = torch.arange(T * kk, device=dev)

    # ---- receive side: every pair I own, in arrival order (src, expert, token, slot)
    own = (dst == rank).reshape(-1)
    akey = (src.reshape(-1) * span + inner.reshape(-1))[own]
    arrival = torch.argsort(akey, stable=True)
    a_src = src.reshape(-1)[own][arrival]
    a_exp = e0.reshape(-1)[own][arrival]
    recv_counts = torch.bincount(a_src, minlength=G)
    to_expert = torch.argsort(a_exp, stable=True)        # expert-major row i <- arrival to_expert[i]
    from_expert = torch.empty_like(to_expert)
    from_expert[to_expert] = torch.arange(to_expert.numel(), device=dev)
    first, count = bounds[rank]
    per_exp = torch.bincount(a_exp - first, minlength=count) if a_exp.numel() else torch.zeros(count, dtype=torch.int64, device=dev)
    offsets = torch.zeros(count + 1, dtype=torch.int32, device=dev)
    offsets[1:] = torch.cumsum(per_exp, 0).to(torch.int32)
    plan = DispatchPlan(
        send_counts=[int(v) for v in send_counts.tolist()],
        recv_counts=[int(v) for v in recv_counts.tolist()],
        send_rows=send_rows,
        to_expert=to_expert,
        from_expert=from_expert,
        offsets=offsets,
        ret_index=ret_index.reshape(T, kk).to(torch.int32),
    )
    # ---- peer-memory exchange: every pair's row at its owner and at its sender, for all ranks
    P = G * T * kk
    ar = torch.arange(P, device=dev)
    src_f, dst_f, e_f, in_f = src.reshape(-1), dst.reshape(-1), e0.reshape(-1), inner.reshape(-1)
    order_s = torch.argsort((src_f * G + dst_f) * span + in_f)          # each sender's send order
    pos_s = torch.empty_like(ar)
    pos_s[order_s] = ar
    send_pos = pos_s - src_f * (T * kk)
    order_e = torch.argsort((e_f * G + src_f) * span + in_f)            # each owner's expert-major order
    pos_e = torch.empty_like(ar)
    pos_e[order_e] = ar
    n_dst = torch.bincount(dst_f, minlength=G)
    before = torch.cumsum(n_dst, 0) - n_dst
    em_pos = pos_e - before[dst_f]
    mine_s = order_s[rank * T * kk:(rank + 1) * T * kk]
    b0, n_own = int(before[rank]), int(n_dst[rank])
    own_e = order_e[b0:b0 + n_own]
    plan.p2p_src_rows = (mine_s // kk - rank * T).to(torch.int32)
    plan.p2p_dst_rank = dst_f[mine_s].to(torch.int32)
    plan.p2p_dst_row = em_pos[mine_s].to(torch.int32)
    plan.c_rank = src_f[own_e].to(torch.int32)
    plan.c_row = send_pos[own_e].to(torch.int32)
    return plan


class DevicePlanner:
    """The per-step dispatch plan of one rank on the GPU: the router kernel writes the global
    routing table (xpgb_route) and one CTA derives every row position from it (xpgb_ep_plan),
    for the layer about to run -- the reference routes on every forward (pipeline.py:200-203),
    and so does this: nothing is cached across steps, and nothing crosses to the host on the
    peer-memory transport.  Buffers are sized once for `tokens` tokens per rank."""

    def __init__(self, spec: ModelSpec, fwd: ForwardSpec, rank: int, world: int, tokens: int, device: int = 0):
        import torch

        L = spec.experts_per_layer
        self.spec, self.fwd, self.rank, self.world, self.T = spec, fwd, rank, world, int(tokens)
        self.kk = min(fwd.top_k, L)
        self.device = device
        first, count = shard_bounds(L, world)[rank]
        dev = f"cuda:{device}"
        i32 = dict(dtype=torch.int32, device=dev)
        G, T, kk = world, self.T, self.kk
        self.cap = G * T * kk
        self.routes = torch.empty(max(1, G * T * kk), **i32)
        self.src_rows = torch.empty(max(1, T * kk), **i32)
        self.dst_rank = torch.empty(max(1, T * kk), **i32)
        self.dst_row = torch.empty(max(1, T * kk), **i32)
        self.ret_index = torch.empty((T, kk), **i32)
        self.c_rank = torch.empty(max(1, self.cap), **i32)
        self.c_row = torch.empty(max(1, self.cap), **i32)
        self.to_arr = torch.empty(max(1, self.cap), **i32)
        self.from_arr = torch.empty(max(1, self.cap), **i32)
        self.offsets = torch.empty(count + 1, **i32)
        self.counts = torch.empty(2 * G + 1, **i32)
        words = int(_lib.lib().xpgb_ep_plan_scratch_words(G, max(1, T), L))
        self.scratch = torch.empty(words, **i32)
        self.bufs = _lib.EpPlanBufs(*[C.c_void_p(t.data_ptr()) for t in (
            self.src_rows, self.dst_rank, self.dst_row, self.ret_index, self.c_rank, self.c_row, self.to_arr,
            self.from_arr, self.offsets, self.counts)])

    def plan(self, layer: int, tokens: int, seed=None) -> DispatchPlan:
        """Route layer `layer` for world x tokens global rows and build this rank's plan, both on
        torch's current stream.  seed: the step's router seed (default fwd.router_seed)."""
        from .device import current_stream_ptr

        if tokens > self.T:
            raise XpgError(f"{tokens} tokens per rank exceed the {self.T} the expert-parallel runner was built for")
        st = C.c_void_p(current_stream_ptr(self.device))
        seed = self.fwd.router_seed if seed is None else seed
        G, L, kk = self.world, self.spec.experts_per_layer, self.kk
        if tokens:
            call("xpgb_route", C.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), int(layer), 1, G * tokens, L,
                 self.fwd.top_k, C.c_void_p(self.routes.data_ptr()), st)
        call("xpgb_ep_plan", C.c_void_p(self.routes.data_ptr()), int(tokens), G, self.rank, kk, L,
             C.c_void_p(self.scratch.data_ptr()), C.byref(self.bufs), st)
        n = tokens * kk
        return DispatchPlan(send_counts=None, recv_counts=None, send_rows=self.src_rows[:n].long(),
                            to_expert=self.to_arr, from_expert=self.from_arr, offsets=self.offsets,
                            ret_index=self.ret_index[:tokens], p2p_src_rows=self.src_rows[:n],
                            p2p_dst_rank=self.dst_rank[:n], p2p_dst_row=self.dst_row[:n], c_rank=self.c_rank,
                            c_row=self.c_row, counts=self.counts, cap_rows=G * tokens * kk)


class PeerExchange:
    """Dispatch/combine over peer memory: one window per rank (CUDA IPC, opened by every
    other rank), one scatter kernel per exchange writing rows straight into the owner's
    expert-major input / the sender's return buffer, an epoch flag per (rank, peer) released
    by the scatter's last CTA and acquired by the receiver's stream (xpgb_ep_*)."""

    FLAG_BYTES = 512  # int32 flags[16] at 0, the scatter's CTA counter at 256; rows from 512

    MAX_WORLD = 16   # kMaxEpWorld (ep_p2p.cuh): flag slots per window

    def __init__(self, rank: int, world: int, tokens: int, kk: int, hidden: int, group=None, device: int = 0,
                 fault_ptr: int = 0):
        """Collective: every rank of the group must construct its PeerExchange together.  Any
        rank's failure (allocation, IPC open) makes every rank raise, so the ranks never end
        up on different transports.  fault_ptr: the rank's context fault word (a faulted step
        raises the peers' fault words; a wait that times out or sees one sets it)."""
        import torch
        import torch.distributed as dist

        if world > self.MAX_WORLD:  # before any allocation: "auto" then takes the collective
            raise XpgError(f"peer exchange supports at most {self.MAX_WORLD} ranks, not {world}")
        torch.cuda.set_device(device)  # the window and every launch belong to this rank's GPU
        self.rank, self.world, self.H = rank, world, hidden
        self.group = group
        self.tokens = tokens
        self.fault_ptr = fault_ptr
        self.in_rows = world * tokens * kk           # worst case: every pair of the step lands here
        self.ret_rows = tokens * kk
        self.xp_off = self.FLAG_BYTES
        # expert-major input rows as two bf16 planes: hi rows, then lo rows in_rows later
        self.ret_off = self.xp_off + ((2 * self.in_rows * hidden * 2 + 255) // 256) * 256
        size = self.ret_off + self.ret_rows * hidden * 4
        self._own, self._opened, err = 0, [], None
        handle = (C.c_uint8 * 64)()
        try:
            base = C.c_void_p()
            call("xpgb_ep_window_alloc", C.c_uint64(size), C.byref(base), handle)
            self._own = base.value
        except Exception as exc:  # noqa: BLE001 -- reported to every rank below
            err = f"rank {rank}: window alloc failed: {exc}"

        def agree(mine):
            if world == 1:
                return [mine]
            out = [None] * world
            dist.all_gather_object(out, mine, group=group)
            return out

        handles = agree(bytes(handle) if err is None else None)
        bases = []
        if err is None and all(h is not None for h in handles):
            try:
                for r in range(world):
                    if r == rank:
                        bases.append(self._own)
                        continue
                    p = C.c_void_p()
                    call("xpgb_ep_window_open", (C.c_uint8 * 64).from_buffer_copy(handles[r]), C.byref(p))
                    self._opened.append(p.value)
                    bases.append(p.value)
            except Exception as exc:  # noqa: BLE001
                err = f"rank {rank}: peer window open failed: {exc}"
        elif err is None:
            err = "a peer could not allocate its window"
        errors = [e for e in agree(err) if e]
        if errors:
            self.close()
            raise RuntimeError("; ".join(errors))
        self.bases = bases
        self._xp = (C.c_void_p * world)(*[b + self.xp_off for b in bases])
        self._ret = (C.c_void_p * world)(*[b + self.ret_off for b in bases])
        self._flags = (C.c_void_p * world)(*bases)
        self.counter = self._own + 256
        self.epoch = 0

    @property
    def xp(self) -> int:
        """This rank's expert-major bf16 input rows (device pointer)."""
        return self._own + self.xp_off

    @property
    def ret(self) -> int:
        """This rank's returned fp32 rows, in send order (device pointer)."""
        return self._own + self.ret_off

    def agree_epoch(self) -> None:
        """Collective (every rank, at session begin): continue from the largest epoch any rank
        reached, so a rank that raised mid-step (and skipped some exchanges) cannot pass a
        later wait early on stale flags or wait for an epoch nobody publishes."""
        import torch
        import torch.distributed as dist

        if self.world == 1:
            return
        on_gpu = dist.get_backend(self.group) == "nccl"
        t = torch.tensor([self.epoch], dtype=torch.int64, device=f"cuda:{torch.cuda.current_device()}" if on_gpu
                         else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group)
        self.epoch = int(t.item())

    def _scatter(self, src, src_rows, dst_rank, dst_row, n, n_dev, to_bf16, regions, stream):
        self.epoch += 1
        call("xpgb_ep_scatter_rows", C.c_void_p(src.data_ptr()),
             C.c_void_p(src_rows.data_ptr()) if src_rows is not None else None,
             C.c_void_p(dst_rank.data_ptr()), C.c_void_p(dst_row.data_ptr()), int(n),
             C.c_void_p(n_dev) if n_dev else None, self.H, 1 if to_bf16 else 0, self.in_rows, regions, self._flags,
             self.world, self.rank, self.epoch, C.c_void_p(self.fault_ptr) if self.fault_ptr else None,
             C.c_void_p(self.counter), C.c_void_p(stream))
        call("xpgb_ep_wait", C.c_void_p(self._own), self.world, self.epoch,
             C.c_void_p(self.fault_ptr) if self.fault_ptr else None, C.c_void_p(stream))

    def _check_rows(self, x) -> None:
        if x.shape[0] > self.tokens:
            raise XpgError(f"{x.shape[0]} tokens per rank overflow the peer windows sized for {self.tokens}")

    def dispatch(self, x, plan, stream) -> int:
        """x fp32 [T, H] -> every owner's expert-major rows (two bf16 planes, lo in_rows later);
        returns this rank's xp."""
        self._check_rows(x)
        self._scatter(x, plan.p2p_src_rows, plan.p2p_dst_rank, plan.p2p_dst_row, plan.p2p_src_rows.numel(), None,
                      True, self._xp, stream)
        return self.xp

    def reduce_combine(self, ctx, plan, stream) -> int:
        """The combine fused with the owner's split-K reduction (xpgb_ep_reduce_scatter): the
        rows of the last experts_forward_range(reduce=0) go from the partial planes straight
        into the token owners' return buffers."""
        self.epoch += 1
        n = plan.cap_rows if plan.counts is not None else int(plan.c_rank.numel())
        call("xpgb_ep_reduce_scatter", ctx.handle, C.c_void_p(plan.c_rank.data_ptr()),
             C.c_void_p(plan.c_row.data_ptr()), int(n), C.c_void_p(plan.n_dev) if plan.n_dev else None, self._ret,
             self._flags, self.world, self.rank, self.epoch, C.c_void_p(self.counter), C.c_void_p(stream))
        call("xpgb_ep_wait", C.c_void_p(self._own), self.world, self.epoch,
             C.c_void_p(self.fault_ptr) if self.fault_ptr else None, C.c_void_p(stream))
        return self.ret

    def combine(self, out, plan, stream) -> int:
        """This rank's expert outputs fp32 [n_own, H] -> the token owners' return buffers."""
        n = plan.cap_rows if plan.counts is not None else int(plan.c_rank.numel())
        self._scatter(out, None, plan.c_rank, plan.c_row, n, plan.n_dev, False, self._ret, stream)
        return self.ret

    def close(self):
        import torch

        torch.cuda.synchronize()
        for p in self._opened:
            _lib.lib().xpgb_ep_window_close(C.c_void_p(p))
        self._opened = []
        if self._own:
            _lib.lib().xpgb_ep_window_free(C.c_void_p(self._own))
            self._own = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ExpertParallelMoE:
    """One rank's MoE layer under expert parallelism.

    route_fn(seed, n_tokens, layer, L, k) -> int [n_tokens, kk] (default: libxpgb router kernel);
    expert_fn(layer, rows fp32 [n, H], offsets int32 [count+1]) -> fp32 [n, H] unscaled expert outputs
    (default: libxpgb grouped SwiGLU through this rank's page table, the rows as their hi/lo bf16 planes);
    combine_fn(rows fp32, index int32 [T, kk], top_k) -> fp32 [T, H] (default: libxpgb ordered combine);
    shared_fn(layer, x fp32 [T, H], y fp32 [T, H]) adds the shared experts' outputs to y in place (each
    rank applies its replica to its own tokens after the routed combine; default: libxpgb when the
    context holds shared experts, else none).
    The defaults need a CUDA device; the CPU tests inject oracle-backed functions.
    """

    def __init__(self, spec: ModelSpec, fwd: ForwardSpec, rank: int, world: int, group=None, ctx=None,
                 route_fn=None, expert_fn=None, combine_fn=None, shared_fn=None, has_shared: bool = False):
        self.spec = spec
        self.fwd = fwd
        self.rank = rank
        self.world = world
        self.group = group
        self.ctx = ctx
        self.bounds = shard_bounds(spec.experts_per_layer, world)
        self.route_fn = route_fn or self._gpu_route
        self.expert_fn = expert_fn or self._gpu_experts
        self.combine_fn = combine_fn or self._gpu_combine
        self.shared_fn = shared_fn or (self._gpu_shared if has_shared else None)
        self.planner = None  # DevicePlanner: per-step plans on the GPU (set by the runner)

    # ---- defaults on the GPU
    def _gpu_route(self, seed, n_tokens, layer, L, k):
        from .device import route_table

        return route_table(seed, n_tokens, 1, L, k, device=self.ctx.device, layer_first=layer)[0]

    @staticmethod
    def planes(rows):
        """fp32 rows [n, H] -> bf16 [2, n, H]: hi = bf16_rn(x), lo = bf16_rn(x - hi)
        (moe_kernels.cuh split_bf16; torch's bf16 cast rounds to nearest even)."""
        import torch

        out = torch.empty((2,) + tuple(rows.shape), dtype=torch.bfloat16, device=rows.device)
        out[0].copy_(rows)
        out[1].copy_(rows - out[0].float())
        return out

    def _gpu_experts(self, layer, rows, offsets):
        import torch

        from .device import current_stream_ptr

        out = torch.empty((rows.shape[0], self.spec.hidden_dim), dtype=torch.float32, device=rows.device)
        if rows.shape[0]:
            planes = self.planes(rows)
            call("xpgb_experts_forward", self.ctx.handle, layer, C.c_void_p(planes.data_ptr()), int(rows.shape[0]),
                 C.c_void_p(offsets.data_ptr()), int(rows.shape[0]), C.c_void_p(out.data_ptr()),
                 C.c_void_p(current_stream_ptr(self.ctx.device)))
        return out

    def _gpu_combine(self, rows, index, top_k):
        import torch

        from .device import current_stream_ptr

        T, kk = index.shape
        y = torch.empty((T, self.spec.hidden_dim), dtype=torch.float32, device=index.device)
        if T:
            call("xpgb_combine_rows", C.c_void_p(rows.data_ptr()), C.c_void_p(index.data_ptr()), T, kk, top_k,
                 self.spec.hidden_dim, C.c_void_p(y.data_ptr()), C.c_void_p(current_stream_ptr(self.ctx.device)))
        return y

    def _gpu_shared(self, layer, x, y):
        from .device import current_stream_ptr

        call("xpgb_shared_forward", self.ctx.handle, layer, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
             int(x.shape[0]), C.c_void_p(current_stream_ptr(self.ctx.device)))

    # ---- one layer
    def plan(self, layer: int, tokens: int, seed=None) -> DispatchPlan:
        """This step's plan for `layer` (routing recomputed every call, as the reference routes
        every forward): on the GPU with a DevicePlanner, else from route_fn on the host."""
        seed = self.fwd.router_seed if seed is None else seed
        if self.planner is not None:
            return self.planner.plan(layer, tokens, seed)
        routes = self.route_fn(seed, self.world * tokens, layer, self.spec.experts_per_layer, self.fwd.top_k)
        return build_plan(routes, self.rank, self.world, tokens, self.bounds)

    def forward(self, layer: int, x, plan: DispatchPlan | None = None):
        plan = plan or self.plan(layer, x.shape[0])
        rows = self.dispatch(x, plan)
        return self.combine(layer, x, self.expert_fn(layer, rows, plan.offsets), plan)

    def dispatch(self, x, plan: DispatchPlan):
        """Send this rank's (token, expert) rows to the owners; returns the rows of its own
        experts, expert-major (fp32 [n_recv, H]: as many bytes as the two bf16 planes the
        expert GEMMs take, and the receiver splits them)."""
        import torch

        if plan.counts is not None:
            plan.resolve_counts()
        send = x.index_select(0, plan.send_rows)
        recv = torch.empty((sum(plan.recv_counts), x.shape[1]), dtype=torch.float32, device=x.device)
        self._a2a(recv, send, plan.recv_counts, plan.send_counts)
        return recv.index_select(0, plan.to_expert)

    def combine(self, layer: int, x, out, plan: DispatchPlan):
        """Return the owners' fp32 expert outputs to their tokens; ordered weighted sum
        (+ this rank's shared-expert replica on its own tokens)."""
        import torch

        back = out.index_select(0, plan.from_expert)
        ret = torch.empty((plan.send_rows.shape[0], x.shape[1]), dtype=torch.float32, device=x.device)
        self._a2a(ret, back, plan.send_counts, plan.recv_counts)
        y = self.combine_fn(ret, plan.ret_index, self.fwd.top_k)
        if self.shared_fn is not None:
            self.shared_fn(layer, x, y)  # after the routed sum, weight 1 (single-device slot order)
        return y

    def _a2a(self, out, inp, out_splits, in_splits):
        import torch
        import torch.distributed as dist

        if self.world == 1:
            out.copy_(inp)
            return
        if out.device.type == "cuda" and dist.get_backend(self.group) == "gloo":
            # gloo moves host memory only (the multi-rank-on-one-GPU test harness); NCCL is
            # the GPU path
            host = torch.empty(out.shape, dtype=out.dtype)
            self._a2a(host, inp.cpu(), out_splits, in_splits)
            out.copy_(host)
            return
        if out.dtype == torch.bfloat16 and out.device.type == "cpu":
            # gloo has no 16-bit all_to_all: move pairs of bf16 words as int32 (H is even)
            dist.all_to_all_single(out.view(torch.int32), inp.contiguous().view(torch.int32), out_splits, in_splits,
                                   group=self.group)
        else:
            dist.all_to_all_single(out, inp.contiguous(), out_splits, in_splits, group=self.group)


class ExpertParallelRunner:
    """The paged decode loop of one rank under EP (StreamedRunner semantics per rank).

    The rank's libxpgb context pages its expert shard through its own 2-layer ring
    (session API: RAW/WAR events, ordering log); the compute of each step is the
    EP dispatch -> grouped SwiGLU -> combine of ExpertParallelMoE on torch's stream.
    """

    def __init__(self, spec: ModelSpec, container, fwd: ForwardSpec, rank: int, world: int, device: int = 0,
                 group=None, shard_pool=None, shared=None, host_codec: bool = False, transport: str = "nccl"):
        """host_codec: the rank's shard pages in as exponent-Huffman records over its own host
        link, decoded on its GPU (as StreamedRunner(host_codec=True)).
        transport: "nccl" (all_to_all_single), "p2p" (PeerExchange: scatter kernels into the
        peers' windows over NVLink), or "auto" (p2p when every window opens, else nccl)."""
        from .device import Context

        shared = shared if shared is not None else getattr(container, "shared", None)
        self.spec = spec
        self.fwd = fwd
        self.rank, self.world = rank, world
        first, count = shard_bounds(spec.experts_per_layer, world)[rank]
        self.shard = (first, count)
        self._codec = None
        self.ctx = Context(spec, _lib.POOL_RING, device, max_tokens=world * fwd.tokens_per_step,
                           expert_shard=(first, count))
        pool = shard_pool if shard_pool is not None else shard_payload(container, first, count)
        self.ctx.attach_host_pool(pool)
        if host_codec:
            from .exponent_codec import CompressedModel
            from .geometry import WeightContainer

            shard = WeightContainer._adopt(ModelSpec(spec.num_layers, count, spec.hidden_dim, spec.intermediate_dim),
                                           pool)
            self._codec = CompressedModel.from_container(shard)
            self.ctx.set_codec(self._codec, host_compressed=True)
        if shared is not None:
            self.ctx.set_shared(shared)  # every rank holds a replica (resident, never paged)
        self.moe = ExpertParallelMoE(spec, fwd, rank, world, group=group, ctx=self.ctx,
                                     has_shared=shared is not None)
        self.peer = None
        self.transport = "nccl"
        self.transport_note = None
        if transport not in ("nccl", "p2p", "auto"):
            raise ValueError(f"unknown transport {transport!r}")
        # the dispatch plan is rebuilt on the GPU for every layer of every step
        self.moe.planner = DevicePlanner(spec, fwd, rank, world, fwd.tokens_per_step, device)
        if transport in ("p2p", "auto"):
            kk = min(fwd.top_k, spec.experts_per_layer)
            try:
                self.peer = PeerExchange(rank, world, fwd.tokens_per_step, kk, spec.hidden_dim, group=group,
                                         device=device, fault_ptr=self.ctx.fault_ptr())
                self.transport = "p2p"
            except Exception as exc:  # noqa: BLE001 -- auto falls back to the collective
                if transport == "p2p":
                    raise
                self.transport_note = f"p2p unavailable ({exc}); nccl all_to_all"

    def close(self) -> None:
        """Release the peer windows (collective: every rank closes its mappings first)."""
        if self.peer is not None:
            import torch.distributed as dist

            peer, self.peer = self.peer, None
            for p in peer._opened:
                _lib.lib().xpgb_ep_window_close(C.c_void_p(p))
            peer._opened = []
            if self.world > 1:
                dist.barrier(group=self.moe.group)
            peer.close()
            self.transport = "nccl"  # later runs fall back to the collective

    def device_tier_bytes(self, m: int) -> int:
        from ._lib import lib
        from .geometry import iter_tensor_ids

        cm, total = self._codec, 0
        for i, tid in enumerate(iter_tensor_ids(cm.spec)):
            if tid.expert <= m:
                total += int(lib().xpgb_codec_record_bytes(cm.spec.value_count(tid.kind), int(cm.bits_lens[i]),
                                                           int(cm.chunk)))
        return total

    def apply_plan(self, plan) -> None:
        """A budget.ResidencyPlan for this rank's shard (pinned, device tier, ring)."""
        from .streamed import _full_width

        N, L = self.spec.num_layers, self.spec.experts_per_layer
        first, count = self.shard
        full = np.zeros((N, L), dtype=np.uint8)
        full[:, first:first + count] = plan.pinned_mask
        streamed = count - plan.pinned_mask.sum(axis=1).min()
        depth = getattr(plan, "depth", 2)
        # a ring below the reference's two layers, or any ring with one window in flight
        sub = 0 < plan.ring and (plan.ring < 2 * streamed or depth != 2)
        self.ctx.apply_residency(full, int(plan.ring) if sub else 0, depth)
        shard_map = np.repeat(plan.device_mask[:, :, None], 2, axis=2).astype(np.uint8)
        self.ctx.set_placement(_full_width(self.spec, shard_map, first, count))

    def _begin(self, iterations: int, tokens: int, profile: bool = False, log: bool = True):
        import torch

        opts = _lib.RunOpts()
        opts.iterations = iterations
        opts.tokens = self.world * tokens
        opts.top_k = self.fwd.top_k
        opts.router_seed = int(self.fwd.router_seed) & 0xFFFFFFFFFFFFFFFF
        opts.log_enable = 1 if log else 0
        opts.profile = 1 if profile else 0  # decoder launch timing (xpgb_decode_stats)
        opts.fresh_inputs = 1
        h = self.ctx.handle
        if self.peer is not None:
            self.peer.agree_epoch()  # collective: every rank begins its session together
        torch.cuda.synchronize(self.ctx.device)
        call("xpgb_session_begin", h, C.byref(opts), None)
        try:
            call("xpgb_session_materialize", h, 0)
            call("xpgb_session_materialize", h, 1)
            total, per_iter = C.c_int32(), C.c_int32()
            call("xpgb_session_info", h, C.byref(total), C.byref(per_iter), None)
        except Exception:
            _lib.lib().xpgb_session_abort(h)
            raise
        return int(total.value), int(per_iter.value)

    def _steps(self, x, g0: int, g1: int, seed=None):
        """Session steps [g0, g1) (whole layers: route + plan and dispatch at a layer's first
        window, the window's grouped GEMMs, combine after its last) on torch's current
        stream.  The plan is rebuilt on the GPU for every layer of every step (no host sync
        on the peer-memory transport; NCCL reads the split sizes once per layer)."""
        import torch

        from .device import current_stream_ptr

        h = self.ctx.handle
        T = x.shape[0]
        info = (C.c_int32 * 7)()
        out = None
        n_rows, rows_ptr, lo_rows, planes = 0, 0, 0, None
        plan = None
        peer = self.peer
        kk = min(self.fwd.top_k, self.spec.experts_per_layer)
        H = self.spec.hidden_dim
        for g in range(g0, g1):  # steps are layers, or windows of a sub-layer ring
            call("xpgb_session_step", h, g, info)
            layer, e0, e1, first, last = info[1], info[3], info[4], info[5], info[6]
            stream = current_stream_ptr(self.ctx.device)
            st = C.c_void_p(stream)
            if first:
                plan = self.moe.plan(layer, T, seed)
                if peer is not None:
                    # rows land expert-major in my window (n_own stays on the device)
                    n_rows, lo_rows = plan.cap_rows, peer.in_rows
                    rows_ptr = peer.dispatch(x, plan, stream)
                    out = None
                else:
                    rows = self.moe.dispatch(x, plan)
                    n_rows = int(rows.shape[0])
                    planes = ExpertParallelMoE.planes(rows)
                    rows_ptr, lo_rows = planes.data_ptr(), max(1, n_rows)
                    out = torch.empty((n_rows, H), dtype=torch.float32, device=x.device)
            call("xpgb_session_acquire", h, g, st)
            if n_rows and e1 > e0:
                # peer windows: the last window leaves its split-K partials for the fused
                # reduce + combine scatter; NCCL reduces into `out` here
                reduce = 1 if (last and peer is None) else 0
                call("xpgb_experts_forward_range", h, layer, C.c_void_p(rows_ptr), int(lo_rows),
                     C.c_void_p(plan.offsets.data_ptr()), n_rows, e0, e1, reduce,
                     C.c_void_p(out.data_ptr() if out is not None else 0), st)
            call("xpgb_session_release", h, g, st)
            call("xpgb_session_materialize", h, g + 2)
            if last:
                if peer is not None:
                    ret = peer.reduce_combine(self.ctx, plan, stream)
                    y = torch.empty((T, H), dtype=torch.float32, device=x.device)
                    if T:
                        call("xpgb_combine_rows", C.c_void_p(ret), C.c_void_p(plan.ret_index.data_ptr()), T, kk,
                             self.fwd.top_k, H, C.c_void_p(y.data_ptr()), st)
                    if self.moe.shared_fn is not None:
                        self.moe.shared_fn(layer, x, y)
                    x = y
                else:
                    x = self.moe.combine(layer, x, out, plan)
        return x

    def _end(self, x) -> RunReport:
        h = self.ctx.handle
        rep = _lib.Report()
        call("xpgb_session_end", h, C.byref(rep))
        records = _records_from_log(self.ctx)
        return RunReport(
            final_activations=x, arena_peak_bytes=int(rep.arena_peak_bytes), stall_seconds=rep.stall_ns * 1e-9,
            war_wait_seconds=rep.war_wait_ns * 1e-9, violations=validate_ordering(records), records=records,
            intervals=_intervals(records), page_fault=self.ctx.fault() if rep.page_fault else None,
            h2d_bytes=int(rep.h2d_bytes), d2d_bytes=int(rep.d2d_bytes),
            copy_busy_seconds=(rep.copy_busy_ns[0] * 1e-9, rep.copy_busy_ns[1] * 1e-9),
            elapsed_seconds=rep.elapsed_ns * 1e-9, kernels=_kernel_stats(rep), decoded_bytes=int(rep.decoded_bytes))

    def run(self, iterations: int, acts, profile: bool = False) -> RunReport:
        import torch

        x = acts if isinstance(acts, torch.Tensor) else torch.from_numpy(np.asarray(acts, np.float32))
        x = x.to(f"cuda:{self.ctx.device}", torch.float32).contiguous()
        if x.shape[0] > self.fwd.tokens_per_step:
            raise XpgError(f"{x.shape[0]} tokens per rank exceed the runner's {self.fwd.tokens_per_step} "
                           "(every rank steps the same number of tokens)")
        total, _ = self._begin(iterations, x.shape[0], profile=profile)
        try:
            x = self._steps(x, 0, total)
        except Exception:
            _lib.lib().xpgb_session_abort(self.ctx.handle)
            raise
        return self._end(x)

    def open_session(self, max_iterations: int, log: bool = False) -> "EPDecodeSession":
        """Serving loop under EP (as StreamedRunner.open_session): one decode iteration per
        step(acts) on fresh activations; the schedule stays open between steps, so the next
        step's first windows page in while the caller holds the result."""
        return EPDecodeSession(self, max_iterations, log)


class EPDecodeSession:
    def __init__(self, runner: ExpertParallelRunner, max_iterations: int, log: bool = False):
        self.runner = runner
        self.max_iterations = max_iterations
        self.T = runner.fwd.tokens_per_step
        self.total, self.per_iter = runner._begin(max_iterations, self.T, log=log)
        self.g = 0
        self.steps_run = 0
        self.x = None
        self.closed = False

    def step(self, acts, out=None, router_seed=None):
        """acts: [T, H] fp32 (numpy, pinned CPU tensor or CUDA tensor); returns the layer
        stack's output (into `out` when given, e.g. pinned host memory).  Every step routes
        afresh on the GPU; router_seed (default fwd.router_seed) stands in for a gate whose
        decisions change from step to step."""
        import torch

        if self.closed or self.steps_run >= self.max_iterations:
            raise XpgError("session is closed or out of iterations")
        if np.shape(acts)[0] != self.T:
            raise XpgError(f"a session step takes {self.T} tokens per rank, got {np.shape(acts)[0]}")
        dev = f"cuda:{self.runner.ctx.device}"
        x = acts if isinstance(acts, torch.Tensor) else torch.from_numpy(np.asarray(acts, np.float32))
        x = x.to(dev, torch.float32, non_blocking=True).contiguous()
        try:
            y = self.runner._steps(x, self.g, self.g + self.per_iter, router_seed)
        except Exception:
            self.abort()
            raise
        self.g += self.per_iter
        self.steps_run += 1
        self.x = y
        if out is not None:
            out.copy_(y, non_blocking=False)
            return out
        return y

    def abort(self):
        if not self.closed:
            _lib.lib().xpgb_session_abort(self.runner.ctx.handle)
            self.closed = True

    def close(self) -> RunReport:
        """End the session (the unused iterations' pages are released)."""
        if self.closed:
            raise XpgError("session already closed")
        self.closed = True
        return self.runner._end(self.x)

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        if not self.closed:
            self.close() if exc[0] is None else self.abort()
