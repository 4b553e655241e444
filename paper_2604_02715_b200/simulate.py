"""The reference's decode performance model, fed with B200 measurements.

Restates xpg simulate.py (``SimConfig`` 20-66, ``simulate_decode`` 96-146,
``steady_tau_load``/``knee_alpha``/``sweep_alpha`` 149-181) and the closed loop of
planner.py (``ResidencyController`` 142-233, ``run_control_loop``/``check_trace_safety``/
``write_trace_csv`` 236-268) with the same arithmetic, so its outputs are pinned to the
reference's own (tests/golden/make_sim_golden.py, tests/test_simulate_cpu.py).

What is new is where the inputs come from: ``calibrated_config`` takes b_host, b_dev and
tau_comp measured on the GPU (``python -m paper_2604_02715_b200 calibrate``), and
``predict_tiered`` extends the per-layer load model to the tiers this implementation adds
(pinned experts that load nothing, host records that cross the link compressed) so the
model's step time can be checked against a measured budget sweep
(``tools/sim_calibration.py``).
"""

from __future__ import annotations

import csv
import math
from collections import deque
from dataclasses import dataclass, replace

from .errors import InfeasibleConfigError, OutOfRangeError
from .geometry import ModelSpec
from .residency import MemoryBudget, PlannerState, compute_rho, plan_step
from .tiers import tau_layer_for_alpha, tau_load_for_alpha_layers


@dataclass(frozen=True)
class SimConfig:
    spec: ModelSpec
    b_dev: float                  # effective device (decompression) bandwidth, raw B/s
    b_host: float                 # host transfer bandwidth, raw-equivalent B/s
    tau_comp_theory: float        # per-iteration forward ceiling, seconds
    batch_size: int
    context_start: int
    max_new_tokens: int
    kv_bytes_per_token: int
    c_gpu: int                    # device byte budget
    non_expert_bytes: int
    swap_bandwidth: float
    compression_ratio: float = 0.8

    def __post_init__(self):
        if self.b_dev <= 0 or self.b_host <= 0 or self.swap_bandwidth <= 0:
            raise OutOfRangeError("bandwidths must be positive")
        if self.tau_comp_theory <= 0:
            raise OutOfRangeError("tau_comp_theory must be positive")
        if self.batch_size < 1 or self.max_new_tokens < 1:
            raise OutOfRangeError("batch_size and max_new_tokens must be >= 1")
        if not 0 < self.compression_ratio <= 1:
            raise OutOfRangeError("compression_ratio must lie in (0, 1]")
        if self.c_gpu <= self.non_expert_bytes + self.window_bytes:
            raise InfeasibleConfigError("device budget cannot hold the mandatory two-layer window")

    @property
    def window_bytes(self) -> int:
        return 2 * self.spec.experts_per_layer * self.spec.expert_bytes

    @property
    def compressed_expert_bytes(self) -> float:
        return self.compression_ratio * self.spec.total_bytes

    def resident_bytes(self, alpha: float) -> float:
        return alpha * self.compressed_expert_bytes

    def kv_bytes(self, iteration: int) -> int:
        return self.batch_size * (self.context_start + iteration) * self.kv_bytes_per_token

    def kv_free_bytes(self, alpha: float) -> float:
        return self.c_gpu - self.non_expert_bytes - self.window_bytes - self.resident_bytes(alpha)


@dataclass(frozen=True)
class IterationSample:
    iteration: int
    kv_bytes: int
    alpha: float
    tau_load: float
    tau_comp_actual: float
    iteration_time: float
    throughput: float
    rho: float
    kv_overflow: float = 0.0
    migration_bytes: float = 0.0


class FixedAlphaPolicy:
    def __init__(self, alpha: float):
        if not 0 < alpha <= 1:
            raise OutOfRangeError(f"alpha must lie in (0, 1], got {alpha}")
        self.alpha = alpha

    def begin(self, config: SimConfig):
        self._layers = [self.alpha] * config.spec.num_layers

    def step(self, iteration: int, kv_bytes: int, last_sample):
        return self._layers, 0.0


def simulate_decode(config: SimConfig, policy) -> list:
    """Decode loop under an alpha policy: iteration time = max(tau_comp + swap, tau_load)."""
    if isinstance(policy, (int, float)):
        policy = FixedAlphaPolicy(float(policy))
    policy.begin(config)
    spec = config.spec
    samples, prev_overflow, last = [], None, None
    for it in range(1, config.max_new_tokens + 1):
        kv = config.kv_bytes(it)
        alpha_layers, migration_bytes = policy.step(it, kv, last)
        alpha = sum(alpha_layers) / len(alpha_layers)
        if prev_overflow is None:
            prev_overflow = max(0.0, config.kv_bytes(0) - config.kv_free_bytes(alpha))
        overflow = max(0.0, kv - config.kv_free_bytes(alpha))
        tau_swap = 2.0 * max(0.0, overflow - prev_overflow) / config.swap_bandwidth
        prev_overflow = overflow
        tau_comp_actual = config.tau_comp_theory + tau_swap
        tau_load = tau_load_for_alpha_layers(spec, config.b_dev, config.b_host, alpha_layers)
        tau_load += migration_bytes / config.b_host
        rho = config.tau_comp_theory / tau_load if tau_load > 0 else math.inf
        iteration_time = max(tau_comp_actual, tau_load)
        last = IterationSample(iteration=it, kv_bytes=kv, alpha=alpha, tau_load=tau_load,
                               tau_comp_actual=tau_comp_actual, iteration_time=iteration_time,
                               throughput=config.batch_size / iteration_time, rho=rho, kv_overflow=overflow,
                               migration_bytes=migration_bytes)
        samples.append(last)
    return samples


def steady_tau_load(config: SimConfig, alpha: float) -> float:
    return config.spec.num_layers * tau_layer_for_alpha(config.spec, config.b_dev, config.b_host, alpha)


def knee_alpha(config: SimConfig) -> float:
    """alpha* where the host-branch tau_load crosses tau_comp_theory, clipped to [0, 1]."""
    n, p_layer = config.spec.num_layers, config.spec.layer_bytes
    return min(1.0, max(0.0, 1.0 - config.tau_comp_theory * config.b_host / (n * p_layer)))


def sweep_alpha(config: SimConfig, alphas) -> list:
    rows = []
    for alpha in alphas:
        if not 0 < alpha <= 1:
            raise OutOfRangeError(f"alpha grid value {alpha} outside (0, 1]")
        tau_load = steady_tau_load(config, alpha)
        rows.append({"alpha": alpha, "tau_load": tau_load, "tau_comp": max(config.tau_comp_theory, tau_load)})
    return rows


def write_samples_csv(samples, path) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["iter", "alpha", "tau_load", "tau_comp", "iter_time", "throughput", "rho", "kv_bytes"])
        for s in samples:
            w.writerow([s.iteration, f"{s.alpha:.6f}", f"{s.tau_load:.9f}", f"{s.tau_comp_actual:.9f}",
                        f"{s.iteration_time:.9f}", f"{s.throughput:.6f}", f"{s.rho:.6f}", s.kv_bytes])


def write_sweep_csv(rows, path) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["alpha", "tau_load", "tau_comp"])
        for r in rows:
            w.writerow([f"{r['alpha']:.6f}", f"{r['tau_load']:.9f}", f"{r['tau_comp']:.9f}"])


# ---------------------------------------------------------------- closed loop over the model

@dataclass(frozen=True)
class TraceRow:
    iteration: int
    rho: float
    alpha: float
    c_kv: float
    c_exp: float
    throughput: float
    adjusted: int


class ResidencyController:
    """Policy object for simulate_decode implementing the planner's closed loop
    (planner.py:142-233): a dead-zone decision every cooldown iterations, applied one layer
    per iteration (io_balance), migrations charged to the host link."""

    def __init__(self, planner: PlannerState, tau_load_noise=None):
        self.initial = planner
        self.tau_load_noise = tau_load_noise

    def begin(self, config: SimConfig):
        self.config = config
        spec = config.spec
        self.l, self.n = spec.experts_per_layer, spec.num_layers
        self.expert_compressed = config.compression_ratio * spec.expert_bytes
        self.pool_bytes = config.compressed_expert_bytes
        self.effective_gpu = config.c_gpu - config.non_expert_bytes - config.window_bytes
        state = self.initial
        m0 = min(state.device_experts, self._budget(0).max_feasible_m(self.l))
        self.state = replace(state, device_experts=max(1, m0))
        self.m_layers = [self.state.device_experts] * self.n
        self.pending = deque()
        self.since_adjust = 0
        self.meta = []

    def _budget(self, iteration: int) -> MemoryBudget:
        horizon = self.initial.cooldown + self.n
        return MemoryBudget(self.effective_gpu, self.config.kv_bytes(iteration + horizon), self.pool_bytes)

    def _estimated_tau_load(self, m: int) -> float:
        return tau_load_for_alpha_layers(self.config.spec, self.config.b_dev, self.config.b_host,
                                         [m / self.l] * self.n)

    def _rho_estimator(self, alpha: float) -> float:
        return compute_rho(self.config.tau_comp_theory, self._estimated_tau_load(round(alpha * self.l)))

    def step(self, iteration: int, kv_bytes: int, last_sample):
        migration_bytes = 0.0
        if self.pending:
            moves = [self.pending.popleft()]
            if not self.state.io_balance:
                while self.pending:
                    moves.append(self.pending.popleft())
            for layer_idx, new_m in moves:
                migration_bytes += abs(self.m_layers[layer_idx] - new_m) * self.expert_compressed
                self.m_layers[layer_idx] = new_m
        adjusted = 0
        rho = self._rho_estimator(self.state.alpha)
        if self.tau_load_noise is not None:
            rho = compute_rho(self.config.tau_comp_theory,
                              self._estimated_tau_load(self.state.device_experts) * self.tau_load_noise(iteration))
        self.since_adjust += 1
        if self.since_adjust >= self.state.cooldown and not self.pending:
            new_state = plan_step(self.state, rho, self._budget(iteration), self._rho_estimator)
            if new_state.device_experts != self.state.device_experts:
                adjusted = 1 if new_state.device_experts > self.state.device_experts else -1
                for layer_idx in range(self.n):
                    self.pending.append((layer_idx, new_state.device_experts))
                self.state = new_state
                self.since_adjust = 0
        self.meta.append((rho, adjusted))
        return [m / self.l for m in self.m_layers], migration_bytes

    def trace(self, samples) -> list:
        return [TraceRow(iteration=s.iteration, rho=rho, alpha=s.alpha, c_kv=float(s.kv_bytes),
                         c_exp=s.alpha * self.pool_bytes, throughput=s.throughput, adjusted=adj)
                for s, (rho, adj) in zip(samples, self.meta)]


def run_control_loop(config: SimConfig, planner: PlannerState, tau_load_noise=None):
    controller = ResidencyController(planner, tau_load_noise=tau_load_noise)
    samples = simulate_decode(config, controller)
    return samples, controller.trace(samples)


def check_trace_safety(config: SimConfig, trace) -> None:
    effective = config.c_gpu - config.non_expert_bytes - config.window_bytes
    for row in trace:
        if row.c_exp > effective - row.c_kv + 1e-6:
            raise AssertionError(f"iteration {row.iteration}: resident experts {row.c_exp:.0f} exceed "
                                 f"budget {effective - row.c_kv:.0f}")


def write_trace_csv(trace, path) -> None:
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["iter", "rho", "alpha", "c_kv", "c_exp", "throughput"])
        for r in trace:
            w.writerow([r.iteration, f"{r.rho:.6f}", f"{r.alpha:.6f}", f"{r.c_kv:.0f}", f"{r.c_exp:.0f}",
                        f"{r.throughput:.6f}"])


# ---------------------------------------------------------------- calibration (B200 measurements)

def calibrated_config(spec: ModelSpec, measured: dict, *, batch_size: int, max_new_tokens: int = 64,
                      context_start: int = 0, kv_bytes_per_token: int = 0, c_gpu: int | None = None,
                      non_expert_bytes: int = 0, swap_bandwidth: float = 50e9) -> SimConfig:
    """A SimConfig whose b_host, b_dev, tau_comp_theory and compression ratio are the ones
    ``calibrate`` measured on the GPU (raw-equivalent B/s; tau per decode iteration).  The
    KV terms default to zero: this path has no attention, so only the residency terms
    matter.  c_gpu defaults to room for the whole model compressed plus the window."""
    if c_gpu is None:
        c_gpu = int(2 * spec.experts_per_layer * spec.expert_bytes + spec.total_bytes + non_expert_bytes + 1)
    return SimConfig(spec=spec, b_dev=float(measured["b_dev"]), b_host=float(measured["b_host"]),
                     tau_comp_theory=float(measured["tau_comp_theory"]), batch_size=batch_size,
                     context_start=context_start, max_new_tokens=max_new_tokens,
                     kv_bytes_per_token=kv_bytes_per_token, c_gpu=c_gpu, non_expert_bytes=non_expert_bytes,
                     swap_bandwidth=swap_bandwidth,
                     compression_ratio=float(measured.get("compression_ratio", 0.8)))


def predict_tiered(config: SimConfig, device_per_layer: float, pinned_per_layer: float = 0.0) -> dict:
    """The reference's iteration time max(tau_comp, N * tau_layer) with this implementation's
    tiers (our extension of tau_layer_for_alpha, storage.py:190-196): per layer, alpha = the
    device-tier share (decoded at b_dev), the pinned share loads nothing, and the rest crosses
    the host link (b_host is raw-equivalent, so compressed host records are already in it)."""
    spec = config.spec
    L, P = spec.experts_per_layer, spec.layer_bytes
    alpha = device_per_layer / L
    host = max(0.0, 1.0 - alpha - pinned_per_layer / L)
    tau_layer = max(alpha * P / config.b_dev, host * P / config.b_host)
    tau_load = spec.num_layers * tau_layer
    t = max(config.tau_comp_theory, tau_load)
    return {"alpha": alpha, "pinned_fraction": pinned_per_layer / L, "tau_load": tau_load, "iteration_time": t,
            "tok_s": config.batch_size / t, "bound": "load" if tau_load >= config.tau_comp_theory else "compute"}


def predict_sm_shared(config: SimConfig, device_per_layer: float, pinned_per_layer: float = 0.0, *,
                      b_dec: float | None = None, b_fused: float | None = None, fx4_per_layer: float | None = None,
                      host_exposed: float = 0.0) -> dict:
    """Step time of this implementation's tiered decode step (our model, not the reference's).

    The reference overlaps every page-in with compute (``max(tau_comp, N * tau_layer)``,
    simulate.py:96-146).  On the GPU only the host link is a separate engine: the exponent
    decoder runs on the same SMs as the GEMMs.  So a step costs the slower of
      link  = host share x model bytes / b_host          (copy engines, compressed records)
      SMs   = tau_comp + streamed-compressed share x model bytes / b_dec
    where the streamed-compressed share is every non-pinned expert (device-tier records and
    host records are both expanded on the SMs).  With decode-into-GEMM (``b_fused``), the
    FX4 device-tier experts -- all of them, or ``fx4_per_layer`` of them in a mixed device tier
    whose other records are Huffman -- instead cost model bytes / b_fused each *in place of*
    their share of tau_comp (their GEMM reads the record directly); every other streamed expert
    pays b_dec.  ``host_exposed``: share of the link time an SM-bound step cannot hide (the
    staging ring holds about one record ahead; budget.HOST_EXPOSED).  Rates are raw-equivalent
    B/s; ``b_dec`` defaults to the calibrated b_dev."""
    spec = config.spec
    L = spec.experts_per_layer
    total = spec.num_layers * spec.layer_bytes
    dev = device_per_layer / L
    pin = pinned_per_layer / L
    host = max(0.0, 1.0 - dev - pin)
    b_dec = config.b_dev if b_dec is None else b_dec
    link = host * total / config.b_host
    if b_fused:
        fx = dev if fx4_per_layer is None else fx4_per_layer / L
        sm = config.tau_comp_theory * (1.0 - fx) + fx * total / b_fused + (host + dev - fx) * total / b_dec
    else:
        sm = config.tau_comp_theory + (dev + host) * total / b_dec
    t = max(link, sm + host_exposed * link)
    return {"link_s": link, "sm_s": sm, "iteration_time": t, "tok_s": config.batch_size / t,
            "bound": "link" if link >= sm else "sm"}
