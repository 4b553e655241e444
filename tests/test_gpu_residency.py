"""Live residency controller on the GPU: measured tau_comp / tau_load drive the device tier.
Needs a B200."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_live_controller_moves_experts_and_stays_exact():
    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200 import residency as R

    spec = X.ModelSpec(4, 8, 1024, 2048)  # 12.6 MB experts: page-in dominates a T=16 step
    fwd = X.ForwardSpec(16, 2, 7)
    c = X.generate_fast_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    hier = X.StorageHierarchy(c, None, X.plan_placement(spec, backends), backends)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=True)
    x = X.initial_activations(spec, fwd, 7)
    want = X.resident_baseline(1, spec, c, fwd, acts=x.copy())
    b_dev, b_host = R.calibrate_bandwidths(runner, x.copy())
    assert b_dev > 0 and b_host > 0  # (tiny tensors: launch-bound, either may be larger)
    budget = runner.device_tier_bytes(8) * 3.5 / 8  # room for 3 (average) experts per layer
    ctl = R.LiveResidencyController(runner, R.PlannerState(8, 1, cooldown=1), budget, b_dev, b_host)
    for _ in range(14):
        s = ctl.step(x.copy())
        assert s.tau_load > 0 and s.tau_comp > 0
    # decode at T=16 is load-bound (rho < theta): the loop fills the budget and stops there
    assert all(s.rho < 0.9 for s in ctl.samples), [s.rho for s in ctl.samples]
    assert ctl.state.device_experts == 3
    assert runner.device_experts == [3, 3, 3, 3]
    assert any(s.adjusted == 1 for s in ctl.samples)
    rep = runner.run(1, acts=x.copy())
    assert rep.violations == [] and rep.page_fault is None
    assert rep.final_activations.tobytes() == np.asarray(want).tobytes()
    assert rep.decoded_bytes > 0
