"""GPU exponent decoder (k_exp_decode): bit-exact with the reference codec; compressed tiers."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def XC():
    from paper_2604_02715_b200 import exponent_codec as XC

    return XC


@pytest.fixture(scope="module")
def X():
    import paper_2604_02715_b200 as X

    return X


def test_roundtrip_adversarial_patterns(XC):
    data = np.arange(65536, dtype=np.uint16).astype("<u2").tobytes()  # NaN, Inf, subnormals, every exponent
    t = XC.build_table(XC.build_histogram(data))
    for chunk in (8, 64, 1024):
        assert XC.decompress(XC.compress(data, t, chunk=chunk), t) == data


@pytest.mark.parametrize("n", [1, 7, 8, 9, 1023, 1024, 1025, 200_000])
def test_roundtrip_random_and_gaussian(XC, X, n):
    rng = np.random.default_rng(n)
    for data in (rng.integers(0, 65536, n, dtype=np.uint16).astype("<u2").tobytes(),
                 X.float32_to_bf16(rng.standard_normal(n).astype(np.float32) * 0.02).astype("<u2").tobytes()):
        t = XC.build_table(XC.build_histogram(data))
        assert XC.decompress(XC.compress(data, t), t) == data


def test_roundtrip_long_codes(XC):
    # a skewed histogram forces codes up to the 32-bit cap (LUT misses take the slow path)
    counts = [0] * 256
    for i in range(40):
        counts[i] = 2 ** min(i, 40)
    t = XC.build_table(XC.ExponentHistogram(tuple(counts)))
    rng = np.random.default_rng(3)
    exps = rng.integers(0, 40, 100_000)
    words = ((exps.astype(np.uint16) << 7) | rng.integers(0, 128, exps.size).astype(np.uint16)).astype("<u2")
    data = words.tobytes()
    assert XC.decompress(XC.compress(data, t, chunk=64), t) == data


def test_compressed_model_tensor_bytes_and_xpgc_roundtrip(XC, X, tmp_path):
    spec = X.ModelSpec(3, 2, 32, 64)
    c = X.generate_synthetic_model(spec, 4)
    cm = XC.CompressedModel.from_container(c)
    for tid in X.iter_tensor_ids(spec):
        assert cm.tensor_bytes(tid) == c.tensor_bytes(tid)
    path = tmp_path / "m.xpgc"
    cm.write(path)
    loaded = XC.CompressedModel.read(path)  # no chunk index in XPGC: rebuilt on the host
    for tid in X.iter_tensor_ids(spec):
        assert loaded.tensor_bytes(tid) == c.tensor_bytes(tid)
    assert loaded.to_bytes() == cm.to_bytes()


def _runner(X, spec, seed, alpha, host_codec):
    container = X.generate_synthetic_model(spec, seed)
    if alpha is None:
        backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    else:
        backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 40),
                    X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    hier = X.StorageHierarchy(container, None, X.plan_placement(spec, backends, alpha=alpha), backends)
    return container, hier


@pytest.mark.parametrize("alpha,host_codec", [(None, True), (0.25, False), (0.5, True), (1.0, False)])
def test_compressed_tiers_streamed_equals_resident(X, alpha, host_codec):
    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(16, 2, 7)
    container, hier = _runner(X, spec, 7, alpha, host_codec)
    x = X.initial_activations(spec, fwd, 7)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=host_codec)
    rep = runner.run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    assert rep.final_activations.tobytes() == base.tobytes()
    if host_codec:
        assert rep.decoded_bytes > 0
        assert rep.h2d_bytes < 0.8 * (2 * spec.total_bytes)  # compressed records cross the link


def test_host_codec_sabotage_still_faults(X):
    spec = X.ModelSpec(4, 2, 64, 128)
    _, hier = _runner(X, spec, 2, None, True)
    hier.delay_fn = lambda tid: 0.03 if tid.layer == 3 else 0.0
    runner = X.StreamedRunner(spec, hier, X.ForwardSpec(3, 2, 5), host_codec=True, sabotage_skip_raw=(1, 3))
    rep = runner.run(2)
    assert rep.page_fault is not None
    assert any(v.startswith("RAW") for v in rep.violations)


def test_host_codec_small_staging_pieces(X, monkeypatch):
    """Records streamed through a 16 KiB staging buffer (many pieces per tensor) stay exact."""
    monkeypatch.setenv("XPGB_STAGE_BYTES", "16384")
    spec = X.ModelSpec(4, 4, 128, 256)
    fwd = X.ForwardSpec(8, 2, 3)
    container, hier = _runner(X, spec, 3, None, True)
    x = X.initial_activations(spec, fwd, 3)
    rep = X.StreamedRunner(spec, hier, fwd, host_codec=True).run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert rep.violations == [] and rep.page_fault is None
    assert rep.final_activations.tobytes() == base.tobytes()


@pytest.mark.parametrize("alpha,host_codec,pinned", [(None, True, None), (None, True, 5), (1.0, False, None),
                                                     (0.5, True, 3)])
def test_grouped_record_runs_exact(X, alpha, host_codec, pinned):
    """More experts than one multi-tensor decode launch holds (64): runs of consecutive
    records split at the launch limit, at pinned experts and at the tier boundary."""
    spec = X.ModelSpec(3, 80, 64, 128)
    fwd = X.ForwardSpec(32, 4, 11)
    container, hier = _runner(X, spec, 11, alpha, host_codec)
    x = X.initial_activations(spec, fwd, 11)
    rep = X.StreamedRunner(spec, hier, fwd, host_codec=host_codec, pinned=pinned).run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert rep.violations == [] and rep.page_fault is None
    assert rep.final_activations.tobytes() == base.tobytes()
    iterations, streamed_experts = 2, spec.num_layers * (spec.experts_per_layer - (pinned or 0))
    assert rep.decoded_bytes == iterations * streamed_experts * spec.expert_bytes  # every streamed tensor decoded



def test_mmap_container_pages_in_exactly(X, tmp_path):
    """A container ingested by mmap + in-place page-locking streams like the pinned copy."""
    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(16, 2, 7)
    c = X.generate_synthetic_model(spec, 7)
    path = tmp_path / "m.xpgw"
    c.write(path)
    o = X.open_container(path)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    for host_codec in (False, True):
        hier = X.StorageHierarchy(o, None, X.plan_placement(spec, backends), backends)
        x = X.initial_activations(spec, fwd, 7)
        rep = X.StreamedRunner(spec, hier, fwd, host_codec=host_codec).run(2, acts=x.copy())
        base = X.resident_baseline(2, spec, c, fwd, acts=x.copy())
        assert rep.violations == [] and rep.page_fault is None
        assert rep.final_activations.tobytes() == base.tobytes()


def test_device_mask_spread_with_sub_layer_ring_exact(X):
    """The bench's tiering: device-tier experts spread over the windows of a sub-layer ring,
    host tier as compressed records -- still bit-identical to the resident model."""
    import numpy as np

    spec = X.ModelSpec(3, 12, 128, 256)
    fwd = X.ForwardSpec(40, 3, 5)
    container, hier = _runner(X, spec, 5, None, True)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=True, ring_experts=6)
    mask = np.zeros((3, 12), dtype=bool)
    mask[:, [0, 4, 5, 9]] = True
    runner.set_device_mask(mask)
    assert runner.device_experts == [4, 4, 4]
    x = X.initial_activations(spec, fwd, 5)
    rep = runner.run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert rep.violations == [] and rep.page_fault is None
    assert rep.final_activations.tobytes() == base.tobytes()
    hbm = runner.ctx.hbm_bytes()
    assert hbm["device_tier"] > 0 and hbm["ring"] == 6 * spec.expert_bytes


@pytest.mark.parametrize("budget", [0.2, 0.6, 0.9, 1.0])
def test_residency_plan_applied_stays_exact(X, budget):
    """budget.plan_residency -> StreamedRunner.apply_plan (sub-layer ring + compressed device
    tier + pinned experts in one context): bit-identical to resident, footprint in budget."""
    from paper_2604_02715_b200.budget import plan_residency

    spec = X.ModelSpec(3, 8, 128, 256)
    fwd = X.ForwardSpec(24, 2, 9)
    container, hier = _runner(X, spec, 9, None, True)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=True)
    ceb = runner.device_tier_bytes(8) / 24 * 1.002
    plan = plan_residency(3, 8, spec.expert_bytes, ceb, budget * spec.total_bytes, min_window_bytes=1)
    runner.apply_plan(plan)
    x = X.initial_activations(spec, fwd, 9)
    rep = runner.run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert rep.violations == [] and rep.page_fault is None
    assert rep.final_activations.tobytes() == base.tobytes()
    hbm = runner.ctx.hbm_bytes()
    assert hbm["ring"] + hbm["device_tier"] <= budget * spec.total_bytes * 1.001


@pytest.mark.parametrize("L,budget", [(1, 0.25), (2, 0.3), (2, 0.7)])
def test_residency_plan_whole_layer_windows(X, L, budget):
    """Plans whose window is a whole layer (an EP rank with 1-2 experts per layer): a ring of
    one layer at depth 1 or two at depth 2, applied and run exactly, within budget."""
    from paper_2604_02715_b200.budget import plan_residency

    spec = X.ModelSpec(4, L, 128, 256)
    fwd = X.ForwardSpec(8, min(2, L), 3)
    container, hier = _runner(X, spec, 3, None, True)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=True)
    ceb = runner.device_tier_bytes(L) / (4 * L) * 1.002
    plan = plan_residency(4, L, spec.expert_bytes, ceb, budget * spec.total_bytes)
    runner.apply_plan(plan)
    x = X.initial_activations(spec, fwd, 3)
    rep = runner.run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert rep.violations == [] and rep.page_fault is None
    assert rep.final_activations.tobytes() == base.tobytes()
    hbm = runner.ctx.hbm_bytes()
    assert hbm["ring"] + hbm["device_tier"] <= budget * spec.total_bytes * 1.001


@pytest.mark.parametrize("stage_buffers", [2, 3, 16])
def test_staging_ring_sizes_exact_and_profiled(X, stage_buffers):
    """Any staging-ring size (link run-ahead) pages in the same bytes; with profile on, every
    decoder launch is timed on its own stream (xpgb_decode_stats) and its algorithmic bytes
    cover what it produced."""
    from paper_2604_02715_b200.errors import OutOfRangeError

    spec = X.ModelSpec(4, 4, 128, 256)
    fwd = X.ForwardSpec(8, 2, 3)
    container, hier = _runner(X, spec, 3, None, True)
    x = X.initial_activations(spec, fwd, 3)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=True, stage_buffers=stage_buffers)
    rep = runner.run(2, acts=x.copy(), profile=True)
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert rep.violations == [] and rep.page_fault is None
    assert rep.final_activations.tobytes() == base.tobytes()
    st = runner.ctx.decode_stats()
    assert st["launches"] > 0 and st["kernel_ns"] > 0
    assert st["algo_bytes"] >= 1.5 * rep.decoded_bytes  # >= bf16 written + sign/mantissa read
    with pytest.raises(OutOfRangeError):
        runner.ctx.set_stage_buffers(1)
    with pytest.raises(OutOfRangeError):
        runner.ctx.set_stage_buffers(17)


def test_lean_gemm_tiles_bit_identical(X):
    """The lean GEMM tiles (one stage fewer, co-resident with decoder CTAs) change the
    pipeline depth only: results are bit-identical to the full tiles."""
    import subprocess
    import sys

    code = (
        "import numpy as np, paper_2604_02715_b200 as X\n"
        "spec = X.ModelSpec(3, 8, 256, 512); fwd = X.ForwardSpec(96, 2, 4)\n"
        "c = X.generate_synthetic_model(spec, 4)\n"
        "b = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]\n"
        "h = X.StorageHierarchy(c, None, X.plan_placement(spec, b), b)\n"
        "r = X.StreamedRunner(spec, h, fwd, host_codec=True, ring_experts=4).run(2, acts=X.initial_activations(spec, fwd, 4))\n"
        "import sys; sys.stdout.buffer.write(np.ascontiguousarray(r.final_activations).tobytes())\n")
    outs = []
    for lean in ("0", "1"):
        env = dict(__import__("os").environ, XPGB_COSCHED=lean)
        root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
        outs.append(subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, check=True,
                                   timeout=300, cwd=root).stdout)
    assert len(outs[0]) > 0 and outs[0] == outs[1]
