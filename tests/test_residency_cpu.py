"""Live residency planner: the decision rule pinned to the reference's own outputs
(tests/golden/planner_v1.json from tests/golden/make_planner_golden.py)."""

import json
import math
import os

import pytest

from paper_2604_02715_b200 import residency as R
from paper_2604_02715_b200.errors import OutOfRangeError

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "planner_v1.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def _est(kind):
    return {"none": None, "steep": (lambda a: 0.2 + 2.0 * a), "flat": (lambda a: 5.0)}[kind]


def test_plan_step_matches_reference_grid(golden):
    bad = []
    for c in golden["plan_step"]:
        st = R.PlannerState(c["L"], c["m"], theta=c["theta"], step_experts=c["step"])
        b = R.MemoryBudget(float("inf"), 0.0, 0.0) if c["budget"] is None else R.MemoryBudget(*c["budget"])
        rho = math.inf if c["rho"] == "inf" else c["rho"]
        got = R.plan_step(st, rho, b, _est(c["est"])).device_experts
        if got != c["out_m"]:
            bad.append((c, got))
    assert not bad, bad[:3]
    assert len(golden["plan_step"]) > 5000


def test_landscape_loops_match_reference(golden):
    for c in golden["landscape"]:
        st = R.PlannerState(8, c["m0"], cooldown=c["cooldown"])
        curve = [None] + c["tau_by_m"][1:]
        res = R.run_landscape_loop(curve, 4.0, st, 60, noise_amplitude=c["noise"], seed=c["seed"])
        assert list(res.alphas) == c["alphas"], c["curve"]
        assert [list(a) for a in res.adjustments] == c["adjustments"]
        assert res.reversals == c["reversals"] and res.final_m == c["final_m"]


def test_state_validation_and_rho():
    with pytest.raises(OutOfRangeError):
        R.PlannerState(8, 0)
    with pytest.raises(OutOfRangeError):
        R.PlannerState(8, 2, theta=1.5)
    with pytest.raises(OutOfRangeError):
        R.compute_rho(1.0, -1.0)
    assert R.compute_rho(1.0, 0.0) == math.inf
    assert R.MemoryBudget(10.0, 4.0, 8.0).max_feasible_m(8) == 6


class _FakeReport:
    def __init__(self, comp, load):
        self.intervals = {(1, l): {"compute": (0.0, comp), "load1": (0.0, load), "load2": (0.0, load / 2)}
                          for l in (1, 2)}
        self.elapsed_seconds = 2 * max(comp, load)


class _FakeRunner:
    """Stands in for StreamedRunner: tau_load falls as more experts sit on the device tier."""

    def __init__(self):
        from paper_2604_02715_b200 import ForwardSpec, ModelSpec

        self.spec = ModelSpec(2, 8, 64, 128)
        self.fwd = ForwardSpec(16, 2, 1)
        self.device_experts = None
        self.applied = []

    def device_tier_bytes(self, m):
        return 1000 * m * self.spec.num_layers

    def set_device_experts(self, m_layers):
        self.device_experts = list(m_layers)
        self.applied.append(tuple(m_layers))

    def run(self, iterations, acts=None):
        m = sum(self.device_experts) / len(self.device_experts)
        return _FakeReport(comp=1.0, load=4.0 * (1 - m / 8) + 0.05)


def test_live_controller_climbs_to_budget_with_staggered_migration():
    runner = _FakeRunner()
    ctl = R.LiveResidencyController(runner, R.PlannerState(8, 1, cooldown=2), hbm_budget_bytes=5 * 2000 + 1,
                                    b_dev=1e12, b_host=1e9)
    for _ in range(30):
        ctl.step(None)
    # the loop raises m while load-bound, one layer per step, and stops at the budget (m = 5)
    assert ctl.state.device_experts == 5
    assert runner.applied[0] == (1, 1)
    assert (2, 1) in runner.applied and (2, 2) in runner.applied  # staggered: one layer per step
    assert all(s.rho > 0 for s in ctl.samples)
    assert sum(s.adjusted for s in ctl.samples) == 4
