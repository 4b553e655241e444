"""Parity of the CUDA path (through the C ABI) with the reference oracle.  Needs a B200.

Bars (north star): routing and slot ids bit-exact; layer outputs within
rel-L2 <= 1e-2 of the reference (bf16 tensor-core inputs, fp32 accumulate);
GPU-streamed == GPU-resident bit-identical.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-2  # north-star bf16 tolerance, relative L2


@pytest.fixture(scope="module")
def X():
    import paper_2604_02715_b200 as X

    return X


@pytest.fixture(scope="module")
def O():
    from oracle import xpg_oracle as O

    return O


def test_router_bit_exact_golden(X, golden):
    from paper_2604_02715_b200.device import route_table

    arrays, meta = golden
    for key, c in meta["cases"].items():
        if not key.startswith("route_"):
            continue
        got = route_table(int(c["seed"]), c["T"], c["N"], c["L"], c["k"]).cpu().numpy()
        np.testing.assert_array_equal(got, arrays[key], err_msg=key)


@pytest.mark.parametrize("L,k,T,N", [(8, 2, 256, 8), (128, 8, 256, 4), (256, 8, 256, 8), (1024, 32, 64, 2), (33, 5, 77, 3)])
def test_router_bit_exact_oracle_full_sizes(X, O, L, k, T, N):
    from paper_2604_02715_b200.device import route_table

    for seed in (7, 0, 2**64 - 1, -12345):
        got = route_table(seed, T, N, L, k).cpu().numpy()
        want = O.route_all(seed, T, N, L, k)
        np.testing.assert_array_equal(got, want)


def test_routed_experts_single_token(X):
    assert X.routed_experts(7, 0, 1, 8, 2) == [2, 6]
    assert X.routed_experts(0, 0, 1, 1, 2) == [1]
    assert X.routed_experts(2**64 + 7, 3, 1, 8, 2) == X.routed_experts(7, 3, 1, 8, 2)


@pytest.mark.parametrize("ci", range(8))
def test_layer_forward_golden(X, O, golden, ci):
    arrays, meta = golden
    c = meta["cases"][f"fwd_{ci}"]
    spec = X.ModelSpec(c["N"], c["L"], c["H"], c["F"])
    container = X.generate_synthetic_model(spec, c["wseed"])
    fwd = X.ForwardSpec(c["T"], c["k"], int(c["rseed"]))
    y = X.layer_forward(container.tensor_f32, spec, fwd, c["layer"], arrays[f"fwd_x_{ci}"])
    err = O.rel_l2(y, arrays[f"fwd_y_{ci}"])
    assert err <= TOL, err


@pytest.mark.parametrize("ci", range(2))
def test_resident_stack_golden(X, O, golden, ci):
    arrays, meta = golden
    c = meta["cases"][f"stack_{ci}"]
    spec = X.ModelSpec(c["N"], c["L"], c["H"], c["F"])
    container = X.generate_synthetic_model(spec, c["wseed"])
    fwd = X.ForwardSpec(c["T"], c["k"], c["wseed"])
    y = X.resident_baseline(c["iterations"], spec, container, fwd, acts=arrays[f"stack_x_{ci}"])
    assert O.rel_l2(y, arrays[f"stack_y_{ci}"]) <= TOL * c["N"] * c["iterations"]


def _hier(X, spec, seed=1, alpha=None, delay_fn=None):
    container = X.generate_synthetic_model(spec, seed)
    if alpha is None:
        backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    else:
        backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 40),
                    X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    plan = X.plan_placement(spec, backends, alpha=alpha)
    return container, X.StorageHierarchy(container, None, plan, backends, delay_fn)


@pytest.mark.parametrize("mode", ["sequential", "threaded"])
@pytest.mark.parametrize("alpha", [None, 0.5])
def test_streamed_equals_resident_bit_exact(X, mode, alpha):
    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(16, 2, 7)
    container, hier = _hier(X, spec, seed=7, alpha=alpha)
    x = X.initial_activations(spec, fwd, 7)
    rep = X.run_iterations(3, spec, hier, fwd, mode=mode, acts=x.copy())
    base = X.resident_baseline(3, spec, container, fwd, acts=x.copy())
    assert rep.page_fault is None
    assert rep.violations == []
    assert rep.final_activations.tobytes() == base.tobytes()
    assert rep.arena_peak_bytes == 2 * spec.experts_per_layer * spec.expert_bytes


def test_streamed_parity_with_oracle_per_layer(X, O, golden):
    """A 1-iteration streamed run layer by layer against the oracle on fresh inputs."""
    spec = X.ModelSpec(2, 8, 256, 512)
    fwd = X.ForwardSpec(64, 2, 3)
    container, hier = _hier(X, spec, seed=7)
    pool = O.WordPool(2, 8, 256, 512, container.words)
    x = np.random.default_rng(5).standard_normal((64, 256), dtype=np.float32)
    rep = X.run_iterations(1, spec, hier, fwd, mode="threaded", acts=x)
    want = O.resident_stack(pool, x, 2, 3, 1)
    assert O.rel_l2(rep.final_activations, want) <= 2 * TOL


@pytest.mark.parametrize("N,L", [(2, 1), (2, 3), (3, 1), (4, 2), (5, 3), (6, 2), (8, 4), (4, 8), (3, 5)])
def test_slot_ids_and_log_match_reference(X, O, golden, N, L):
    arrays, meta = golden
    ci = next(k.split("_")[1] for k, c in meta["cases"].items()
              if k.startswith("slots_") and c["N"] == N and c["L"] == L)
    spec = X.ModelSpec(N, L, 16, 16)
    _, hier = _hier(X, spec, seed=1)
    trace = []
    runner = X.StreamedRunner(spec, hier, X.ForwardSpec(2, 2, 1), mode="sequential", trace=trace)
    rep = runner.run(3)
    maps = []
    for line in trace:
        f = dict(kv.split("=") for kv in line.split())
        if f["event"] == "map":
            maps.append((int(f["layer"]), int(f["expert"]), int(f["kind"]), int(f["block"])))
    assert maps == [tuple(r) for r in arrays[f"slots_{ci}"].tolist()]
    ev = {0: "recycle", 1: "load-start", 2: "load-done", 3: "compute-start", 4: "compute-done"}
    want = [(ev[r[0]], r[1], r[2], None if r[3] < 0 else r[3], None if r[4] < 0 else r[4], None if r[5] < 0 else r[5])
            for r in arrays[f"order_{ci}"].tolist()]
    got = [(r.event, r.iteration, r.layer, r.kind, r.target_iteration, r.target_layer) for r in rep.records]
    assert got == want
    assert rep.violations == []


def test_threaded_log_is_clean_and_overlaps(X):
    spec = X.ModelSpec(6, 2, 64, 64)
    _, hier = _hier(X, spec, seed=5, alpha=0.5, delay_fn=lambda tid: 0.002)
    runner = X.StreamedRunner(spec, hier, X.ForwardSpec(3, 2, 5), mode="threaded",
                              compute_delay_fn=lambda it, ly: 0.004)
    rep = runner.run(2)
    assert rep.violations == []
    overlaps = 0
    for (it, ly), spans in rep.intervals.items():
        nxt = (it, ly + 1) if ly < spec.num_layers else (it + 1, 1)
        ns = rep.intervals.get(nxt)
        if ns and "load1" in ns and "compute" in spans and ns["load1"][0] < spans["compute"][1]:
            overlaps += 1
    assert overlaps > 0
    kind_overlaps = sum(1 for s in rep.intervals.values()
                        if "load1" in s and "load2" in s and s["load1"][0] < s["load2"][1] and s["load2"][0] < s["load1"][1])
    assert kind_overlaps > 0


def test_injected_delays_stall_but_stay_exact(X):
    spec = X.ModelSpec(4, 2, 64, 128)
    fwd = X.ForwardSpec(3, 2, 5)
    container, hier = _hier(X, spec, seed=3, alpha=0.5, delay_fn=lambda tid: 0.001)
    x = X.initial_activations(spec, fwd, 3)
    rep = X.run_iterations(2, spec, hier, fwd, mode="threaded", acts=x.copy())
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert rep.final_activations.tobytes() == base.tobytes()
    assert rep.violations == []
    assert rep.stall_seconds > 0


def test_sabotage_reports_raw_violation_and_page_fault(X):
    spec = X.ModelSpec(4, 2, 64, 128)
    _, hier = _hier(X, spec, seed=2, alpha=0.5, delay_fn=lambda tid: 0.03 if tid.layer == 3 else 0.0)
    runner = X.StreamedRunner(spec, hier, X.ForwardSpec(3, 2, 5), mode="threaded", sabotage_skip_raw=(1, 3))
    rep = runner.run(2)
    assert rep.page_fault is not None
    assert any(v.startswith("RAW") for v in rep.violations)


def test_cold_start_and_war_targets(X):
    spec = X.ModelSpec(4, 2, 64, 128)
    _, hier = _hier(X, spec, seed=2)
    rep = X.run_iterations(2, spec, hier, X.ForwardSpec(3, 2, 5), mode="threaded")
    rec = [r for r in rep.records if r.event == "recycle"]
    assert [r for r in rec if r.iteration == 1 and r.layer <= 2] == []
    assert {(r.target_iteration, r.target_layer) for r in rec if r.iteration == 1 and r.layer == 3} == {(1, 1)}
    assert {(r.target_iteration, r.target_layer) for r in rec if r.iteration == 2 and r.layer == 1} == {(1, 3)}


def test_per_kind_window_never_exceeds_two_layers(X):
    spec = X.ModelSpec(6, 2, 16, 32)
    trace = []
    _, hier = _hier(X, spec, seed=4, alpha=0.5)
    X.StreamedRunner(spec, hier, X.ForwardSpec(3, 2, 5), mode="threaded", trace=trace).run(3)
    mapped = {1: set(), 2: set()}
    for line in trace:
        f = dict(kv.split("=") for kv in line.split())
        kind, layer = int(f["kind"]), int(f["layer"])
        if f["event"] == "map":
            mapped[kind].add(layer)
        elif f["event"] == "unmap":
            mapped[kind].discard(layer)
        assert len(mapped[kind]) <= 2, line


def test_zero_input_stays_zero(X):
    spec = X.ModelSpec(4, 2, 64, 128)
    _, hier = _hier(X, spec, seed=2)
    zeros = np.zeros((3, 64), dtype=np.float32)
    rep = X.run_iterations(1, spec, hier, X.ForwardSpec(3, 2, 5), mode="sequential", acts=zeros)
    assert not rep.final_activations.any()


def test_report_json_fields(X):
    import json

    spec = X.ModelSpec(4, 2, 64, 128)
    _, hier = _hier(X, spec, seed=2)
    doc = json.loads(X.run_iterations(1, spec, hier, X.ForwardSpec(3, 2, 5)).to_json())
    for key in ("activation_checksum", "stall_ms", "arena_peak_bytes", "violation_count", "layer_intervals"):
        assert key in doc
    assert doc["violation_count"] == 0


@pytest.mark.parametrize("shared,host_codec", [(0, False), (1, False), (0, True)])
def test_expert_parallel_runner_world1_matches_resident(X, O, shared, host_codec):
    """The EP runner (session API + experts_forward + ordered combine [+ the rank's shared
    expert replica on its own tokens]) on one GPU."""
    from paper_2604_02715_b200.expert_parallel import ExpertParallelRunner

    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(16, 2, 7)
    container = X.generate_synthetic_model(spec, 7, shared_experts=shared)
    x = X.initial_activations(spec, fwd, 7)
    runner = ExpertParallelRunner(spec, container, fwd, rank=0, world=1, host_codec=host_codec)
    rep = runner.run(2, x)
    assert rep.page_fault is None and rep.violations == []
    assert rep.arena_peak_bytes == 2 * spec.experts_per_layer * spec.expert_bytes
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert O.rel_l2(rep.final_activations.cpu().numpy(), base) <= 1e-3


@pytest.mark.parametrize("tokens,pair", [(1024, None), (96, "1")])
def test_expert_parallel_runner_pair_gemm(X, O, monkeypatch, tokens, pair):
    """EP owners with prefill-sized groups (>= 128 rows per expert) run the CTA-pair GEMMs
    in experts_forward_range (forced on for a small batch too)."""
    from paper_2604_02715_b200.expert_parallel import ExpertParallelRunner

    if pair is not None:
        monkeypatch.setenv("XPGB_PAIR_GEMM", pair)
    spec = X.ModelSpec(2, 8, 256, 512)
    fwd = X.ForwardSpec(tokens, 2, 5)
    container = X.generate_synthetic_model(spec, 5)
    x = X.initial_activations(spec, fwd, 5)
    runner = ExpertParallelRunner(spec, container, fwd, rank=0, world=1, host_codec=True)
    rep = runner.run(1, x)
    assert rep.page_fault is None and rep.violations == []
    base = X.resident_baseline(1, spec, container, fwd, acts=x.copy())
    assert O.rel_l2(rep.final_activations.cpu().numpy(), base) <= 1e-3


def test_expert_parallel_runner_windows_and_device_tier(X, O):
    """EP runner on a budget plan: sub-layer ring windows (experts_forward_range per window,
    dispatch before the first, combine after the last) + compressed device tier + pinned."""
    from paper_2604_02715_b200.budget import plan_residency
    from paper_2604_02715_b200.expert_parallel import ExpertParallelRunner

    spec = X.ModelSpec(3, 8, 128, 256)
    fwd = X.ForwardSpec(24, 2, 5)
    container = X.generate_synthetic_model(spec, 5)
    x = X.initial_activations(spec, fwd, 5)
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    for budget in (0.3, 0.7):
        runner = ExpertParallelRunner(spec, container, fwd, rank=0, world=1, host_codec=True)
        ceb = runner.device_tier_bytes(8) / 24 * 1.002
        plan = plan_residency(3, 8, spec.expert_bytes, ceb, budget * spec.total_bytes, min_window_bytes=1)
        assert plan.ring < 16  # a sub-layer ring: several windows per layer
        runner.apply_plan(plan)
        rep = runner.run(2, x)
        assert rep.page_fault is None and rep.violations == []
        assert O.rel_l2(rep.final_activations.cpu().numpy(), base) <= 1e-3


def test_session_api_external_compute_matches_run(X):
    """begin/materialize/acquire/compute/release/end reproduces run() bit for bit."""
    import ctypes as C

    import torch

    from paper_2604_02715_b200 import _lib
    from paper_2604_02715_b200._lib import call

    spec = X.ModelSpec(4, 4, 128, 256)
    fwd = X.ForwardSpec(8, 2, 3)
    container, hier = _hier(X, spec, seed=3)
    x = X.initial_activations(spec, fwd, 3)
    runner = X.StreamedRunner(spec, hier, fwd)
    want = runner.run(2, acts=x.copy()).final_activations
    acts = torch.from_numpy(x.copy()).cuda()
    opts = _lib.RunOpts()
    opts.iterations, opts.tokens, opts.top_k, opts.router_seed, opts.log_enable = 2, 8, 2, 3, 1
    h = runner.ctx.handle
    torch.cuda.synchronize()
    call("xpgb_session_begin", h, C.byref(opts), C.c_void_p(acts.data_ptr()))
    total, per_it, st = C.c_int32(), C.c_int32(), C.c_void_p()
    call("xpgb_session_info", h, C.byref(total), C.byref(per_it), C.byref(st))
    assert (total.value, per_it.value) == (2 * spec.num_layers, spec.num_layers)
    call("xpgb_session_materialize", h, 0)
    call("xpgb_session_materialize", h, 1)
    for g in range(2 * spec.num_layers):  # built-in compute runs on the session's compute stream
        call("xpgb_session_acquire", h, g, st)
        call("xpgb_session_compute", h, g)
        call("xpgb_session_release", h, g, st)
        call("xpgb_session_materialize", h, g + 2)
    rep = _lib.Report()
    call("xpgb_session_end", h, C.byref(rep))
    assert acts.cpu().numpy().tobytes() == want.tobytes()
    assert rep.page_fault == 0


@pytest.mark.parametrize("pinned,host_codec", [(2, False), (5, True), (7, False)])
def test_pinned_experts_budget_tier(X, pinned, host_codec):
    """Residency tier x > 0: pinned experts stay resident, the ring streams the rest; results unchanged."""
    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(16, 2, 7)
    container, hier = _hier(X, spec, seed=7)
    x = X.initial_activations(spec, fwd, 7)
    runner = X.StreamedRunner(spec, hier, fwd, pinned=pinned, host_codec=host_codec)
    rep = runner.run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    assert rep.final_activations.tobytes() == base.tobytes()
    streamed = spec.experts_per_layer - pinned
    hbm = runner.ctx.hbm_bytes()
    assert hbm["ring"] == (2 * streamed + spec.num_layers * pinned) * spec.expert_bytes
    if not host_codec:
        assert rep.h2d_bytes == 2 * spec.num_layers * streamed * spec.expert_bytes
    # a second run on the same context still finds its pinned experts resident
    rep2 = runner.run(1, acts=x.copy())
    assert rep2.page_fault is None and rep2.violations == []


@pytest.mark.parametrize("L,k,T", [(8, 2, 1500), (128, 8, 300), (64, 4, 4097), (3, 5, 700), (4, 2, 2001)])
def test_multi_cta_plan_layer_forward_vs_oracle(X, O, L, k, T):
    """T*k above the single-CTA plan threshold: route+count / scan+place over many CTAs.
    Layer output within tolerance of the oracle, and the resident run of the same step
    (all layers planned at once) bit-identical to layer_forward."""
    spec = X.ModelSpec(2, L, 64, 128)
    container = X.generate_synthetic_model(spec, 5)
    pool = O.WordPool(2, L, 64, 128, container.words)
    x = np.random.default_rng(T).standard_normal((T, 64), dtype=np.float32)
    fwd = X.ForwardSpec(T, k, 9)
    y1 = X.layer_forward(container.tensor_f32, spec, fwd, 1, x)
    assert O.rel_l2(y1, O.layer_forward(pool, 1, x, k, 9)) <= TOL
    y2 = X.layer_forward(container.tensor_f32, spec, fwd, 2, y1)
    # resident run of the same step (both layers planned at once, fused next-layer gather)
    model = X.ResidentModel(spec, container, max_tokens=T)
    out, _ = model.run(1, fwd, x.copy())
    assert np.asarray(out).tobytes() == np.asarray(y2).tobytes()


@pytest.mark.parametrize("ring,host_codec", [(None, False), (4, True)])
def test_decode_session_steps_equal_resident(X, ring, host_codec):
    """A serving session: each step runs one decode iteration on fresh inputs while the next
    step's first layers prefetch; every output equals the resident model on that input."""
    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(16, 2, 7)
    container, hier = _hier(X, spec, seed=7)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=host_codec, ring_experts=ring)
    model = X.ResidentModel(spec, container, max_tokens=16)
    rng = np.random.default_rng(0)
    sess = runner.open_session(max_iterations=5)
    for i in range(3):  # closes early: 3 of 5
        x = rng.standard_normal((16, 256), dtype=np.float32)
        got = sess.step(x)
        want, _ = model.run(1, fwd, x.copy())
        assert np.asarray(got).tobytes() == np.asarray(want).tobytes(), i
    rep = sess.close()
    assert rep.violations == [] and rep.page_fault is None
    assert sum(1 for r in rep.records if r.event == "compute-start") == 3 * sess.steps_per_iteration
    with pytest.raises(X.XpgError):
        sess.close()
    # the runner is reusable afterwards, also through the context-manager form
    x = rng.standard_normal((16, 256), dtype=np.float32)
    with runner.open_session(max_iterations=1) as s2:
        assert np.asarray(s2.step(x)).tobytes() == np.asarray(model.run(1, fwd, x.copy())[0]).tobytes()
    r2 = runner.run(1, acts=x.copy())
    assert r2.violations == [] and r2.final_activations.tobytes() == np.asarray(model.run(1, fwd, x.copy())[0]).tobytes()


def test_empty_step_and_single_expert_edge_cases(X, O):
    """T = 0 (an empty decode step) pages like any other step and returns an empty batch;
    L = 1 with top_k > L routes every token to the one expert with scale 1/top_k."""
    spec = X.ModelSpec(3, 4, 64, 128)
    container, hier = _hier(X, spec, seed=2)
    fwd0 = X.ForwardSpec(0, 2, 1)
    rep = X.StreamedRunner(spec, hier, fwd0).run(2, acts=np.zeros((0, 64), np.float32))
    assert rep.final_activations.shape == (0, 64)
    assert rep.violations == [] and rep.page_fault is None
    assert rep.arena_peak_bytes == 2 * spec.experts_per_layer * spec.expert_bytes
    y0 = X.layer_forward(container.tensor_f32, spec, fwd0, 1, np.zeros((0, 64), np.float32))
    assert np.asarray(y0).shape == (0, 64)
    spec1 = X.ModelSpec(2, 1, 64, 128)
    c1 = X.generate_synthetic_model(spec1, 3)
    pool = O.WordPool(2, 1, 64, 128, c1.words)
    x = np.random.default_rng(0).standard_normal((9, 64), dtype=np.float32)
    y = X.layer_forward(c1.tensor_f32, spec1, X.ForwardSpec(9, 3, 5), 2, x)
    assert O.rel_l2(y, O.layer_forward(pool, 2, x, 3, 5)) <= TOL
