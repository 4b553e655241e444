"""Live residency control: the reference planner's dead-zone rule, fed by measured times.

Reference: xpg planner.py (``PlannerState``/``MemoryBudget`` 44-91, ``compute_rho``
94-100, ``plan_step`` 103-131, ``ResidencyController`` 148-233, ``run_landscape_loop``
262-340).  The decision rule is restated here unchanged -- it is host policy, a few
comparisons per cooldown period -- so its outputs are pinned to the reference's
own traces (tests/golden/make_planner_golden.py).  What changes on the B200 is the
signal: the reference drives the rule from a *simulator* (simulate.py), this module
drives it from a real decode loop on the GPU:

* tau_comp  = sum over layers of the compute span (compute-start -> compute-done,
  device timestamps of the ordering log), i.e. the forward with no page-in stall;
* tau_load  = sum over layers of the page-in span (load-start -> load-done of the
  slower kind), i.e. what the copy/decode streams needed for the layer;
* rho       = tau_comp / tau_load, averaged over the cooldown window.

The control variable is the device tier of the placement (experts 1..m of every
layer kept compressed in HBM, decoded on-GPU into the ring -- storage.py:143-168),
exactly the reference's alpha = m / L.  A change is applied one layer per decode
step (io_balance, planner.py:185-196) through ``StreamedRunner.set_device_experts``;
the descent guard estimates rho at the destination from the measured per-tier
bandwidths (``tiers.tau_layer_for_alpha``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from .errors import OutOfRangeError
from .tiers import tau_layer_for_alpha

THETA_DEFAULT = 0.9      # planner.py:40
COOLDOWN_DEFAULT = 300   # planner.py:41


@dataclass(frozen=True)
class PlannerState:
    """Residency m / L of the device tier plus the loop's knobs (planner.py:44-68)."""

    experts_per_layer: int
    device_experts: int
    theta: float = THETA_DEFAULT
    step_experts: int = 1
    cooldown: int = COOLDOWN_DEFAULT
    io_balance: bool = True

    def __post_init__(self):
        if not (0.0 < self.theta <= 1.0 + 1e-12):
            raise OutOfRangeError(f"theta must lie in (0, 1], got {self.theta}")
        if min(self.step_experts, self.cooldown) < 1:
            raise OutOfRangeError("step_experts and cooldown must be >= 1")
        if not (1 <= self.device_experts <= self.experts_per_layer):
            raise OutOfRangeError(
                f"device_experts {self.device_experts} outside [1, {self.experts_per_layer}]")

    @property
    def alpha(self) -> float:
        return self.device_experts / self.experts_per_layer


@dataclass(frozen=True)
class MemoryBudget:
    """Bytes the resident experts may use once the KV cache is served (planner.py:71-91)."""

    c_gpu: float
    c_kv: float
    expert_pool_bytes: float  # device-tier size at alpha = 1

    @property
    def c_res(self) -> float:
        return self.c_gpu - self.c_kv

    def c_exp(self, alpha: float) -> float:
        return alpha * self.expert_pool_bytes

    def max_feasible_m(self, experts_per_layer: int) -> int:
        if self.expert_pool_bytes <= 0:
            return experts_per_layer
        quantum = self.expert_pool_bytes / experts_per_layer
        return int(math.floor(self.c_res / quantum + 1e-9))


def compute_rho(tau_comp: float, tau_load: float) -> float:
    """tau_comp / tau_load; a free load reads as +inf (planner.py:94-100)."""
    if tau_load < 0:
        raise OutOfRangeError(f"negative tau_load {tau_load}")
    return math.inf if tau_load == 0 else tau_comp / tau_load


def plan_step(state: PlannerState, rho: float, budget: MemoryBudget, rho_estimator=None) -> PlannerState:
    """One decision (planner.py:103-131): dead zone [theta, 1], guarded descent, budget clamp."""
    L, m = state.experts_per_layer, state.device_experts
    if rho > 1.0:                              # compute-bound: give memory back ...
        down = max(1, m - state.step_experts)
        # ... unless the destination would already be load-bound (descent guard)
        if down != m and (rho_estimator is None or rho_estimator(down / L) >= 1.0):
            m = down
    elif rho < state.theta:                    # load-bound: keep more experts on the device
        m = min(L, m + state.step_experts)
    m = max(1, min(L, m, budget.max_feasible_m(L)))  # never displace the KV cache
    return state if m == state.device_experts else replace(state, device_experts=m)


# --------------------------------------------------------------------------- landscape harness


@dataclass(frozen=True)
class LandscapeResult:
    alphas: tuple
    adjustments: tuple
    reversals: int
    final_m: int

    @property
    def oscillated(self) -> bool:
        return self.reversals > 0


def run_landscape_loop(tau_by_m, tau_comp_theory: float, planner: PlannerState, iterations: int,
                       noise_amplitude: float = 0.0, seed: int = 0, budget: MemoryBudget | None = None):
    """The planner against a synthetic tau_load(m) curve (planner.py:262-340): measurements
    are tau_by_m[m] * (1 + U(-a, a)) averaged since the last decision; the descent guard
    sees the noiseless curve."""
    L = planner.experts_per_layer
    budget = budget or MemoryBudget(float("inf"), 0.0, 0.0)
    rng = np.random.default_rng(seed)
    state, window, alphas, adjustments, since = planner, [], [], [], 0

    def guard(alpha):
        return compute_rho(tau_comp_theory, tau_by_m[round(alpha * L)])

    for it in range(1, iterations + 1):
        tau = tau_by_m[state.device_experts]
        if noise_amplitude:
            tau *= 1.0 + rng.uniform(-noise_amplitude, noise_amplitude)
        window.append(tau)
        since += 1
        if since >= state.cooldown:
            nxt = plan_step(state, compute_rho(tau_comp_theory, sum(window) / len(window)), budget, guard)
            if nxt.device_experts != state.device_experts:
                adjustments.append((it, 1 if nxt.device_experts > state.device_experts else -1))
                state = nxt
            window.clear()
            since = 0
        alphas.append(state.alpha)
    reversals = sum(1 for (_, a), (_, b) in zip(adjustments, adjustments[1:]) if a != b)
    return LandscapeResult(tuple(alphas), tuple(adjustments), reversals, state.device_experts)


# --------------------------------------------------------------------------- live loop on the GPU


@dataclass
class LiveSample:
    """One decode step of the live loop."""

    iteration: int
    m_layers: tuple          # device-tier experts per layer during the step
    tau_comp: float          # measured, seconds
    tau_load: float          # measured, seconds
    rho: float
    step_seconds: float
    tokens_per_second: float
    migration_bytes: int = 0
    adjusted: int = 0        # +1 / -1 when a decision changed m


def measured_taus(report) -> tuple:
    """(tau_comp, tau_load) of one iteration from a RunReport's device-timestamped spans."""
    comp = load = 0.0
    for spans in report.intervals.values():
        if "compute" in spans:
            t0, t1 = spans["compute"]
            comp += t1 - t0
        ls = [spans[k][1] - spans[k][0] for k in ("load1", "load2") if k in spans]
        load += max(ls) if ls else 0.0
    return comp, load


@dataclass
class LiveResidencyController:
    """Closed-loop residency on a running StreamedRunner (planner.py:148-233 on real times).

    ``hbm_budget_bytes`` is the device memory the expert tiers may use beside the ring
    (c_gpu - non_expert - window in the reference); ``kv_bytes_fn(iteration)`` the KV demand
    to keep free (default none).  ``b_dev``/``b_host`` (raw-equivalent B/s of the device and
    host tiers) feed the descent guard; measure them with ``calibrate``.
    """

    runner: object
    planner: PlannerState
    hbm_budget_bytes: float
    b_dev: float
    b_host: float
    kv_bytes_fn: object = None
    samples: list = field(default_factory=list)

    def __post_init__(self):
        spec = self.runner.spec
        self.n_layers = spec.num_layers
        self.L = spec.experts_per_layer
        self.pool_bytes = float(self.runner.device_tier_bytes(self.L))  # device tier at alpha = 1
        m0 = min(self.planner.device_experts, self._budget(0).max_feasible_m(self.L))
        self.state = replace(self.planner, device_experts=max(1, m0))
        self.m_layers = [self.state.device_experts] * self.n_layers
        self.runner.set_device_experts(self.m_layers)
        self.pending = []
        self.window = []
        self.since = 0

    def _budget(self, iteration: int) -> MemoryBudget:
        horizon = self.planner.cooldown + self.n_layers  # planner.py:172-177
        kv = float(self.kv_bytes_fn(iteration + horizon)) if self.kv_bytes_fn else 0.0
        return MemoryBudget(self.hbm_budget_bytes, kv, self.pool_bytes)

    def _rho_estimate(self, tau_comp: float):
        spec = self.runner.spec

        def est(alpha: float) -> float:
            return compute_rho(tau_comp, self.n_layers * tau_layer_for_alpha(spec, self.b_dev, self.b_host, alpha))

        return est

    def step(self, acts) -> LiveSample:
        it = len(self.samples) + 1
        migration = 0
        if self.pending:  # staggered migration: one layer per step (all at once without io_balance)
            moves = [self.pending.pop(0)] if self.state.io_balance else [self.pending.pop(0) for _ in
                                                                          range(len(self.pending))]
            for layer_idx, m in moves:
                migration += abs(self.m_layers[layer_idx] - m) * self.runner.device_tier_bytes(1) // self.n_layers
                self.m_layers[layer_idx] = m
            self.runner.set_device_experts(self.m_layers)
        rep = self.runner.run(1, acts=acts)
        tau_comp, tau_load = measured_taus(rep)
        rho = compute_rho(tau_comp, tau_load)
        self.window.append((tau_comp, tau_load))
        self.since += 1
        adjusted = 0
        if self.since >= self.state.cooldown and not self.pending:
            tc = sum(w[0] for w in self.window) / len(self.window)
            tl = sum(w[1] for w in self.window) / len(self.window)
            nxt = plan_step(self.state, compute_rho(tc, tl), self._budget(it), self._rho_estimate(tc))
            if nxt.device_experts != self.state.device_experts:
                adjusted = 1 if nxt.device_experts > self.state.device_experts else -1
                self.pending = [(l, nxt.device_experts) for l in range(self.n_layers)]
                self.state = nxt
            self.window.clear()
            self.since = 0
        sec = rep.elapsed_seconds
        s = LiveSample(it, tuple(self.m_layers), tau_comp, tau_load, rho, sec,
                       self.runner.fwd.tokens_per_step / sec if sec > 0 else 0.0, int(migration), adjusted)
        self.samples.append(s)
        return s


def calibrate_bandwidths(runner, acts, reps: int = 3) -> tuple:
    """(b_dev, b_host) in raw-equivalent B/s, measured on this GPU.

    b_host: a host-only paged stack (link-bound), raw model bytes per second of its run.
    b_dev: the on-GPU exponent decoder expanding a device-resident record (the device tier's
    page-in), best of ``reps``."""
    import ctypes as C

    import torch

    from ._lib import call
    from .exponent_codec import CompressedModel

    spec = runner.spec
    saved = list(runner.device_experts) if runner.device_experts is not None else None
    runner.set_device_experts([0] * spec.num_layers)
    # host-only stack: link-bound, so the raw bytes streamed per second of wall time are the
    # link's raw-equivalent rate (the per-layer load spans of one cold iteration overstate the
    # link time: they include the first layers' start-up and staging waits)
    runner.run(1, acts=acts)
    rep = runner.run(3, acts=acts)
    b_host = 3 * spec.total_bytes / rep.elapsed_seconds if rep.elapsed_seconds > 0 else float("inf")
    cm = runner.hierarchy.compressed
    if not isinstance(cm, CompressedModel):
        cm = CompressedModel.from_container(runner.hierarchy.container)
        runner.hierarchy.compressed = cm
    rec = torch.from_numpy(np.ascontiguousarray(cm._rec(0))).cuda(runner.ctx.device)
    n = spec.value_count(1)
    out = torch.empty(n, dtype=torch.int16, device=rec.device)
    lengths = cm.table.lengths_array()
    stream = torch.cuda.current_stream(rec.device).cuda_stream
    best = float("inf")
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call("xpgb_codec_decode", C.c_void_p(rec.data_ptr()), C.c_uint64(n), C.c_uint64(int(cm.bits_lens[0])),
             int(cm.chunk), lengths.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_void_p(out.data_ptr()),
             C.c_void_p(stream))
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    if saved is not None:
        runner.set_device_experts(saved)
    return 2.0 * n / best, b_host
