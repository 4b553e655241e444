"""The simulator restatement (paper_2604_02715_b200.simulate) against golden vectors dumped
from the reference's own simulate.py / planner.py closed loop (tests/golden/make_sim_golden.py):
knee alpha*, alpha sweeps, fixed-alpha decode samples with KV swap, and the controller trace."""
import json
import os

import numpy as np
import pytest

import paper_2604_02715_b200 as X
from paper_2604_02715_b200 import simulate as S
from paper_2604_02715_b200.residency import PlannerState

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "sim_golden.json")


def _cases():
    with open(GOLD) as fh:
        return json.load(fh)["cases"]


@pytest.mark.parametrize("ci", range(9))
def test_simulator_matches_reference(ci):
    case = _cases()[ci]
    spec = X.ModelSpec(*case["spec"])
    c = S.SimConfig(spec=spec, **case["config"])
    assert S.knee_alpha(c) == pytest.approx(case["knee"], rel=1e-12)
    grid = [r["alpha"] for r in case["sweep"]]
    for got, want in zip(S.sweep_alpha(c, grid), case["sweep"]):
        assert got["tau_load"] == pytest.approx(want["tau_load"], rel=1e-12)
        assert got["tau_comp"] == pytest.approx(want["tau_comp"], rel=1e-12)
    samples = S.simulate_decode(c, 0.25)
    got = np.array([[s.iteration, s.kv_bytes, s.alpha, s.tau_load, s.tau_comp_actual, s.iteration_time,
                     s.throughput, s.rho, s.kv_overflow] for s in samples])
    np.testing.assert_allclose(got, np.array(case["fixed_alpha_samples"]), rtol=1e-12)
    st = PlannerState(experts_per_layer=spec.experts_per_layer, device_experts=max(1, spec.experts_per_layer // 4),
                      cooldown=5)
    _, trace = S.run_control_loop(c, st)

    got = np.array([[r.iteration, r.rho, r.alpha, r.c_kv, r.c_exp, r.throughput, r.adjusted] for r in trace])
    np.testing.assert_allclose(got, np.array(case["loop_trace"]), rtol=1e-12)


def test_tiered_prediction_reduces_to_reference_without_pinned():
    spec = X.ModelSpec(8, 8, 4096, 14336)
    c = S.calibrated_config(spec, {"b_dev": 900e9, "b_host": 80e9, "tau_comp_theory": 0.004,
                                   "compression_ratio": 0.66}, batch_size=256)
    for m in range(1, 9):
        p = S.predict_tiered(c, m, 0)
        assert p["tau_load"] == pytest.approx(S.steady_tau_load(c, m / 8), rel=1e-12)
    assert S.predict_tiered(c, 0, 8)["tau_load"] == 0.0  # everything pinned: nothing to load
    assert S.predict_tiered(c, 0, 8)["bound"] == "compute"
