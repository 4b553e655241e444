"""FX4 device-tier records (fx4.cuh): lossless round trips on the GPU, exact record sizes, and
paged stacks on an FX4 device tier -- decoded into the ring or read in place by the
decode-into-GEMM kernel -- byte-identical to the resident model."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def X():
    import paper_2604_02715_b200 as X

    return X


def _roundtrip(words: np.ndarray):
    import torch

    from paper_2604_02715_b200._lib import call, lib

    n = words.size
    raw = torch.from_numpy(words.view(np.int16).copy()).cuda()
    scratch = torch.empty(int(lib().xpgb_fx4_scratch_bytes(n)), dtype=torch.uint8, device="cuda")
    base, esc, nbytes = C.c_int32(), C.c_uint64(), C.c_uint64()
    s = torch.cuda.current_stream().cuda_stream
    call("xpgb_fx4_measure", C.c_void_p(raw.data_ptr()), C.c_uint64(n), C.c_void_p(scratch.data_ptr()),
         C.byref(base), C.byref(esc), C.byref(nbytes), C.c_void_p(s))
    rec = torch.full((int(nbytes.value),), 0xAB, dtype=torch.uint8, device="cuda")
    call("xpgb_fx4_encode", C.c_void_p(raw.data_ptr()), C.c_uint64(n), base.value, C.c_void_p(scratch.data_ptr()),
         C.c_void_p(rec.data_ptr()), C.c_void_p(s))
    out = torch.empty_like(raw)
    call("xpgb_fx4_decode", C.c_void_p(rec.data_ptr()), C.c_uint64(n), base.value, C.c_void_p(out.data_ptr()),
         C.c_void_p(s))
    torch.cuda.synchronize()
    return out.cpu().numpy().view(np.uint16), base.value, esc.value, nbytes.value


def test_fx4_roundtrip_gaussian_weights():
    rng = np.random.default_rng(1)
    n = 1 << 20
    w = (rng.standard_normal(n, dtype=np.float32) * 0.02).view(np.uint32)
    words = ((w + 0x7FFF + ((w >> 16) & 1)) >> 16).astype(np.uint16)  # RNE to bf16
    out, base, esc, nbytes = _roundtrip(words)
    assert np.array_equal(out, words)
    ex = (words >> 7) & 0xFF
    assert esc == int(((ex < base) | (ex > base + 14)).sum())
    assert esc < n // 1000  # a 15-wide window covers N(0, 0.02) almost entirely
    assert nbytes <= n * 1.52 + 8192  # ~12.1 bits per value


def test_fx4_roundtrip_every_bf16_pattern_and_escapes():
    # all 65,536 bf16 patterns (NaN, Inf, subnormals, both signs): most exponents escape
    words = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    rng = np.random.default_rng(5)
    words = np.concatenate([words, rng.permutation(words)])
    out, base, esc, _ = _roundtrip(words)
    assert np.array_equal(out, words)
    assert esc > words.size // 2


def test_fx4_roundtrip_top_exponents():
    """Exponents crowded at the top of the range: the base stops at 240 so base + 15 (an escape's
    code) never carries into the next byte of the decoders' four-codes-at-once add."""
    rng = np.random.default_rng(9)
    n = 1 << 16
    ex = rng.integers(236, 256, n).astype(np.uint32)
    words = ((rng.integers(0, 2, n).astype(np.uint32) << 15) | (ex << 7) | rng.integers(0, 128, n).astype(np.uint32))
    words = words.astype(np.uint16)
    out, base, esc, _ = _roundtrip(words)
    assert base <= 240
    assert np.array_equal(out, words)


@pytest.mark.parametrize("fused", [True, False])
@pytest.mark.parametrize("T,host_codec", [(16, False), (40, True), (100, True)])
def test_fx4_device_tier_stack_equals_resident(X, fused, T, host_codec):
    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(T, 2, 7)
    container = X.generate_synthetic_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 50),
                X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 50)]
    hier = X.StorageHierarchy(container, None, X.plan_placement(spec, backends, alpha=0.5 if host_codec else 1.0),
                              backends)
    x = np.random.default_rng(T).standard_normal((T, spec.hidden_dim), dtype=np.float32)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=host_codec, fused_decode=fused, device_format="fx4")
    rep = runner.run(2, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert np.asarray(rep.final_activations).tobytes() == np.asarray(base).tobytes()
    assert runner.ctx.hbm_bytes()["device_tier"] > 0


def test_fx4_full_shape_fused_equals_resident(X):
    import torch

    from paper_2604_02715_b200.exponent_codec import CompressedModel

    spec = X.ModelSpec(2, 8, 4096, 14336)
    T = 256
    fwd = X.ForwardSpec(T, 2, 7)
    container = X.generate_fast_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 50),
                X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 50)]
    hier = X.StorageHierarchy(container, CompressedModel.from_container(container),
                              X.plan_placement(spec, backends, alpha=1.0), backends)
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((T, 4096), dtype=np.float32)).cuda()
    runner = X.StreamedRunner(spec, hier, fwd, fused_decode=True, device_format="fx4")
    rep = runner.run(2, acts=x.clone())
    assert rep.page_fault is None and rep.violations == [] and rep.decoded_bytes == 0
    paged = rep.final_activations.cpu().numpy()
    del runner
    torch.cuda.empty_cache()
    model = X.ResidentModel(spec, container, max_tokens=T)
    y, _ = model.run(2, fwd, x.clone())
    assert paged.tobytes() == y.cpu().numpy().tobytes()


def test_host_staging_released_when_no_host_tier(X):
    """A plan that leaves no expert on the host tier gives the staging ring and the chunk index
    back (xpgb_set_host_staging); streaming a host record without them fails loudly."""
    from paper_2604_02715_b200.budget import fx4_expert_bytes, plan_tiers
    from paper_2604_02715_b200.errors import XpgError

    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(16, 2, 7)
    container = X.generate_synthetic_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    hier = X.StorageHierarchy(container, None, X.plan_placement(spec, backends), backends)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=True)
    overhead = runner.ctx.hbm_bytes()["staging"]
    assert overhead > 0
    L, N = spec.experts_per_layer, spec.num_layers
    ceb = runner.device_tier_bytes(L) / (N * L) * 1.002
    plan = plan_tiers(N, L, spec.expert_bytes, ceb, 0.95 * spec.total_bytes, overhead_bytes=overhead,
                      fx4_ceb=fx4_expert_bytes(spec.hidden_dim, spec.intermediate_dim) * 1.002,
                      units_per_expert=spec.intermediate_dim // 128)
    assert plan.host_experts == 0
    runner.apply_plan(plan)
    assert runner.ctx.hbm_bytes()["staging"] == 0
    x = X.initial_activations(spec, fwd, 7)
    rep = runner.run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    assert np.asarray(rep.final_activations).tobytes() == np.asarray(base).tobytes()
    # experts back on the host tier need the staging ring: refused while it is released
    runner.set_device_mask(np.zeros((N, L), dtype=bool))
    runner.ctx.set_pinned(np.zeros((N, L), dtype=np.uint8))
    with pytest.raises(XpgError):
        runner.ctx.set_host_staging(False)


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("T,host_codec", [(16, False), (40, True), (100, True)])
def test_mixed_device_tier_stack_equals_resident(X, mode, T, host_codec):
    """Per-tensor formats (xpgb_set_device_formats): FX4 and Huffman records side by side on the
    device tier -- gate/up and down of one expert may differ -- decoded into the ring (mode 0),
    all read in place (1), or FX4 in place and Huffman into the ring (2): byte-identical."""
    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(T, 2, 7)
    container = X.generate_synthetic_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 50),
                X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 50)]
    hier = X.StorageHierarchy(container, None, X.plan_placement(spec, backends, alpha=0.75 if host_codec else 1.0),
                              backends)
    x = np.random.default_rng(T).standard_normal((T, spec.hidden_dim), dtype=np.float32)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=host_codec)
    fmts = np.random.default_rng(T + mode).random((spec.num_layers, spec.experts_per_layer, 2)) < 0.5
    runner.ctx.set_device_formats(fmts)
    runner.ctx.set_fused_decode(mode)
    rep = runner.run(2, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert np.asarray(rep.final_activations).tobytes() == np.asarray(base).tobytes()
    # both formats staged: bigger than all-Huffman, smaller than all-FX4
    mixed = runner.ctx.hbm_bytes()["device_tier"]
    runner.ctx.set_device_format("huffman")
    huff = runner.ctx.hbm_bytes()["device_tier"]
    runner.ctx.set_device_format("fx4")
    assert huff < mixed < runner.ctx.hbm_bytes()["device_tier"]
    rep = runner.run(2, acts=x.copy())
    assert np.asarray(rep.final_activations).tobytes() == np.asarray(base).tobytes()


def test_mixed_plan_full_shape_equals_resident(X):
    """The planner's mixed device tier (budget.plan_tiers) applied to two Mixtral-shaped layers at
    T = 256: every expert on the device tier, FX4 in place beside Huffman into the ring, no host
    record streamed, byte-identical to the resident model."""
    import torch

    from paper_2604_02715_b200.budget import fx4_expert_bytes, plan_tiers
    from paper_2604_02715_b200.exponent_codec import CompressedModel

    spec = X.ModelSpec(2, 8, 4096, 14336)
    T = 256
    fwd = X.ForwardSpec(T, 2, 7)
    container = X.generate_fast_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 50)]
    hier = X.StorageHierarchy(container, CompressedModel.from_container(container),
                              X.plan_placement(spec, backends), backends)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=True)
    N, L, eb = 2, 8, spec.expert_bytes
    ceb = runner.device_tier_bytes(L) / (N * L) * 1.002
    fx = fx4_expert_bytes(4096, 14336) * 1.002
    budget = (N * L * ceb + 2 * eb + 5 * (fx - ceb)) * 1.001  # room for 5 FX4 conversions
    plan = plan_tiers(N, L, eb, ceb, budget, fx4_ceb=fx, device_format="mixed", units_per_expert=112)
    assert plan.device_format == "mixed" and plan.host_experts == 0 and 0 < plan.fx4_experts < N * L
    runner.apply_plan(plan)
    assert runner.ctx.hbm_bytes()["staging"] == 0
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((T, 4096), dtype=np.float32)).cuda()
    rep = runner.run(2, acts=x.clone(), profile=True)
    assert rep.page_fault is None and rep.violations == [] and rep.h2d_bytes == 0
    assert runner.ctx.fused_stats()["launches"] > 0 and rep.decoded_bytes > 0
    paged = rep.final_activations.cpu().numpy()
    del runner
    torch.cuda.empty_cache()
    model = X.ResidentModel(spec, container, max_tokens=T)
    y, _ = model.run(2, fwd, x.clone())
    assert paged.tobytes() == y.cpu().numpy().tobytes()


def test_device_formats_rejects_bad_entries(X):
    """xpgb_set_device_formats: entries other than 0 / 1 fail loudly, the tier is left as it was."""
    from paper_2604_02715_b200.errors import XpgError

    spec = X.ModelSpec(2, 4, 256, 512)
    fwd = X.ForwardSpec(8, 2, 7)
    container = X.generate_synthetic_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 50),
                X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 50)]
    hier = X.StorageHierarchy(container, None, X.plan_placement(spec, backends, alpha=1.0), backends)
    runner = X.StreamedRunner(spec, hier, fwd)
    before = runner.ctx.hbm_bytes()["device_tier"]
    bad = np.zeros((spec.num_layers, spec.experts_per_layer, 2), dtype=np.uint8)
    bad[1, 2, 0] = 2
    with pytest.raises(XpgError):
        runner.ctx.set_device_formats(bad)
    assert runner.ctx.hbm_bytes()["device_tier"] == before
    x = X.initial_activations(spec, fwd, 7)
    rep = runner.run(1, acts=x.copy())
    base = X.resident_baseline(1, spec, container, fwd, acts=x.copy())
    assert rep.page_fault is None and np.asarray(rep.final_activations).tobytes() == np.asarray(base).tobytes()


@pytest.mark.parametrize("fused", [True, False])
def test_single_activation_plane_mode(X, fused):
    """xpgb_set_activation_planes(1): the decode-sized GEMMs multiply the bf16 hi plane only.
    Streamed (FX4 device tier, read in place or decoded into the ring) == resident in that mode,
    byte for byte; against the two-plane result it stays well inside the 1e-2 tolerance."""
    import torch

    spec = X.ModelSpec(2, 8, 256, 512)
    T = 40
    fwd = X.ForwardSpec(T, 2, 7)
    container = X.generate_synthetic_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 50),
                X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 50)]
    hier = X.StorageHierarchy(container, None, X.plan_placement(spec, backends, alpha=1.0), backends)
    # one pass over the 2-layer stack (deep synthetic stacks overflow by design)
    x = torch.from_numpy(np.random.default_rng(11).standard_normal((T, spec.hidden_dim), dtype=np.float32)).cuda()
    model = X.ResidentModel(spec, container, max_tokens=T)
    y2, _ = model.run(1, fwd, x.clone())
    y2 = y2.cpu().numpy()
    model.ctx.set_activation_planes(1)
    y1, _ = model.run(1, fwd, x.clone())
    y1 = y1.cpu().numpy()
    del model
    runner = X.StreamedRunner(spec, hier, fwd, fused_decode=fused, device_format="fx4")
    runner.ctx.set_activation_planes(1)
    rep = runner.run(1, acts=x.clone())
    assert rep.page_fault is None and rep.violations == []
    assert rep.final_activations.cpu().numpy().tobytes() == y1.tobytes()
    assert np.isfinite(y1).all() and np.isfinite(y2).all()
    rel = float(np.linalg.norm(y1 - y2) / np.linalg.norm(y2))
    assert 0.0 < rel < 1e-2
