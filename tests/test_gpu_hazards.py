"""Race hardening: recycled ring blocks poisoned with NaN bytes (xpgb_set_hazard_checks).

A correct schedule never reads a block before its load lands or after a later window recycled
it, so poisoning every mapped block changes nothing.  Dropping one WAR wait (the WAR twin of
the reference's RAW sabotage, pipeline.py:369-370) must show up twice: as a WAR violation in
the replayed ordering log, and on the device -- the recycle unmaps the victim's slot-table
entries before its blocks are poisoned and refilled, so a GEMM that starts after it faults
(the device PageFault), and one already streaming the block reads NaN bytes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def X():
    import paper_2604_02715_b200 as X

    return X


def _hier(X, spec, seed, alpha=None):
    container = X.generate_synthetic_model(spec, seed)
    if alpha is None:
        backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    else:
        backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 40),
                    X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    return container, X.StorageHierarchy(container, None, X.plan_placement(spec, backends, alpha=alpha), backends)


@pytest.mark.parametrize("alpha,host_codec,ring", [(None, False, None), (None, True, None), (0.5, True, None),
                                                   (None, True, 4), (0.5, False, 4)])
def test_poisoned_blocks_change_nothing(X, alpha, host_codec, ring):
    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(16, 2, 7)
    container, hier = _hier(X, spec, 7, alpha)
    x = X.initial_activations(spec, fwd, 7)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=host_codec, ring_experts=ring)
    runner.ctx.set_hazard_checks(poison=True)
    rep = runner.run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    assert np.asarray(rep.final_activations).tobytes() == np.asarray(base).tobytes()


def test_dropped_war_wait_is_caught_twice(X):
    spec = X.ModelSpec(4, 2, 64, 128)
    fwd = X.ForwardSpec(4, 2, 5)
    _, hier = _hier(X, spec, 2)
    # layer 3's load recycles layer 1's blocks (2-layer ring): hold layer 1's compute for
    # 50 ms and layer 3's copies for 100 ms, so the poisoned blocks sit under layer 1's GEMMs
    hier.delay_fn = lambda tid: 0.1 if tid.layer == 3 else 0.0
    runner = X.StreamedRunner(spec, hier, fwd, compute_delay_fn=lambda it, ly: 0.05 if (it, ly) == (1, 1) else 0.0)
    runner.ctx.set_hazard_checks(poison=True, skip_war=(1, 3))
    rep = runner.run(1)
    assert any(v.startswith("WAR") for v in rep.violations), rep.violations
    assert rep.page_fault is not None or np.isnan(np.asarray(rep.final_activations)).any()
    # the same run with the wait in place is clean and finite
    runner = X.StreamedRunner(spec, hier, fwd, compute_delay_fn=lambda it, ly: 0.05 if (it, ly) == (1, 1) else 0.0)
    runner.ctx.set_hazard_checks(poison=True)
    rep = runner.run(1)
    assert rep.violations == [] and rep.page_fault is None
    assert np.isfinite(np.asarray(rep.final_activations)).all()
