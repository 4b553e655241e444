"""Host-side logic of the B200 package (no GPU): geometry, ids, placement, ordering."""

import numpy as np
import pytest

import paper_2604_02715_b200 as X
from paper_2604_02715_b200.errors import STATUS_CLASSES, raise_for_status
from oracle import xpg_oracle as O

TINY = X.ModelSpec(2, 2, 4, 8)


def test_sigma_and_sizes():
    assert TINY.sigma_gate_up == 2 * 4 * 16 == 128
    assert TINY.sigma_down == 2 * 8 * 4 == 64
    assert TINY.layer_bytes == 2 * (128 + 64)
    assert TINY.total_bytes == 768
    assert TINY.tensor_shape(X.TensorKind.GATE_UP) == (16, 4)
    assert TINY.tensor_shape(X.TensorKind.DOWN) == (4, 8)


def test_spec_validation():
    for bad in [(1, 2, 4, 8), (2, 0, 4, 8), (2, 2, 0, 8)]:
        with pytest.raises(X.OutOfRangeError):
            X.ModelSpec(*bad)


def test_tensor_offsets_match_oracle_and_tile_payload():
    spec = X.ModelSpec(3, 5, 16, 24)
    spans = []
    for tid in X.iter_tensor_ids(spec):
        off = X.tensor_offset(tid, spec)
        assert off == O.tensor_offset(3, 5, 16, 24, tid.layer, tid.expert, int(tid.kind))
        spans.append((off, off + spec.sigma(tid.kind)))
    spans.sort()
    assert spans[0][0] == 0 and spans[-1][1] == spec.total_bytes
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    with pytest.raises(X.OutOfRangeError):
        X.tensor_offset(X.ExpertTensorId(4, 1, X.TensorKind.GATE_UP), spec)


def test_generator_bit_identical_to_reference(golden):
    _, meta = golden
    for key, digest in meta["cases"].items():
        if key.startswith("gen_"):
            _, N, L, H, F, seed = key.split("_")
            c = X.generate_synthetic_model(X.ModelSpec(int(N), int(L), int(H), int(F)), int(seed),
                                           chunk_values=1000)
            import hashlib

            assert hashlib.sha256(c.payload).hexdigest() == digest, key


@pytest.mark.parametrize("total,seg_draws,threads", [(1, 1 << 10, 4), (4097, 1 << 10, 3), (1_000_003, 1 << 12, 8),
                                                      (300_000, 1 << 8, 2), (2_500_000, 1 << 16, 5)])
def test_parallel_generator_splices_to_one_shot_stream(total, seg_draws, threads):
    """The segment-parallel decode of the PCG64 normal stream (geometry._fill_normal_bf16)
    equals the reference's one-shot draw (model.py:205-214), across hundreds of splices,
    tiny segments and an output split over two arrays (routed + shared payload)."""
    from paper_2604_02715_b200.geometry import SYNTH_STD, _fill_normal_bf16, float32_to_bf16

    want = float32_to_bf16(np.random.default_rng(11).standard_normal(total, dtype=np.float32) * SYNTH_STD)
    a = np.zeros(total // 3, np.uint16)
    b = np.zeros(total - total // 3, np.uint16)
    _fill_normal_bf16(11, [a, b], threads, seg_draws)
    np.testing.assert_array_equal(np.concatenate([a, b]), want)


def test_container_roundtrip_and_errors():
    c = X.generate_synthetic_model(TINY, 5)
    raw = c.to_bytes()
    again = X.WeightContainer.from_bytes(raw)
    assert again.spec == TINY and again.payload == c.payload
    rebuilt = b"".join(c.tensor_bytes(t) for t in X.iter_tensor_ids(TINY))
    assert rebuilt == c.payload
    with pytest.raises(X.ContainerFormatError):
        X.WeightContainer.from_bytes(b"NOPE" + raw[4:])
    with pytest.raises(X.ContainerFormatError):
        X.WeightContainer.from_bytes(raw[:-1])


def test_bf16_conversions(golden):
    arrays, _ = golden
    np.testing.assert_array_equal(X.float32_to_bf16(arrays["bf16_in"]), arrays["bf16_out"])
    assert X.float32_to_bf16(np.array([1.0], np.float32))[0] == 0x3F80


@pytest.mark.parametrize("i,n,want", [(2, 48, 48), (3, 48, 1), (5, 48, 3), (1, 8, 7), (2, 8, 8), (1, 2, 1), (2, 2, 2)])
def test_target_layer(i, n, want):
    assert X.target_layer(i, n) == want == O.target_layer(i, n)


def test_target_layer_range():
    with pytest.raises(X.OutOfRangeError):
        X.target_layer(3, 2)
    with pytest.raises(X.OutOfRangeError):
        X.target_layer(1, 1)


def test_vaddr():
    spec = X.ModelSpec(4, 3, 8, 16)
    space = X.AddressSpace.for_spec(spec)
    assert X.page_vaddr(X.ExpertTensorId(1, 1, X.TensorKind.GATE_UP), space) == space.base_gate_up
    last = X.ExpertTensorId(4, 3, X.TensorKind.DOWN)
    assert X.page_vaddr(last, space) == space.base_down + space.extent(X.TensorKind.DOWN) - spec.sigma_down
    assert space.base_gate_up + space.extent(X.TensorKind.GATE_UP) <= space.base_down
    sp2 = X.AddressSpace(X.ModelSpec(4, 8, 5, 5), 0, 10**9)
    assert X.page_vaddr(X.ExpertTensorId(2, 3, X.TensorKind.GATE_UP), sp2) == 10 * sp2.spec.sigma_gate_up


def test_placement_matches_reference(golden):
    arrays, meta = golden
    n = 0
    for key, case in meta["cases"].items():
        if not key.startswith("place_"):
            continue
        spec = X.ModelSpec(*case["spec"])
        backends = [X.Backend(b[0], X.BackendKind(b[1]), b[2], b[3]) for b in case["backends"]]
        plan = X.plan_placement(spec, backends, alpha=case["alpha"])
        tab = np.zeros((spec.num_layers, spec.experts_per_layer, 2), dtype=np.int32)
        for tid, bid in plan.assignment.items():
            tab[tid.layer - 1, tid.expert - 1, int(tid.kind) - 1] = bid
        np.testing.assert_array_equal(tab, arrays[key], err_msg=key)
        for bid, frac in case["fractions"].items():
            assert plan.fractions[int(bid)] == pytest.approx(frac)
        assert X.estimate_load(plan, backends, spec).tau_load == pytest.approx(case["tau_load"])
        n += 1
    assert n == 12


def test_placement_errors():
    with pytest.raises(X.OutOfRangeError):
        X.plan_placement(TINY, [])
    b = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 1e9, 10)]
    with pytest.raises(X.CapacityExceededError):
        X.plan_placement(TINY, b)
    with pytest.raises(X.OutOfRangeError):
        X.Backend(1, X.BackendKind.HOST_OFFLOAD, 0, 1)


def test_validate_ordering_constructed_logs():
    R = X.OrderingRecord
    war = [R(0, "load-done", 1, 1, 1), R(1, "load-done", 1, 1, 2), R(2, "compute-start", 1, 1),
           R(3, "recycle", 1, 3, 1, 1, 1), R(4, "compute-done", 1, 1)]
    v = X.validate_ordering(war)
    assert len(v) == 1 and v[0].startswith("WAR")
    raw = [R(0, "compute-start", 1, 1), R(1, "load-done", 1, 1, 1), R(2, "load-done", 1, 1, 2)]
    v = X.validate_ordering(raw)
    assert len(v) == 2 and all(s.startswith("RAW") for s in v)


def test_status_codes_map_onto_reference_errors():
    assert STATUS_CLASSES[4] is X.DoubleMapError and STATUS_CLASSES[7] is X.PageFaultError
    with pytest.raises(X.PoolExhaustedError):
        raise_for_status(5, "x")
    raise_for_status(0, "")


def test_storage_fetch_host_dest():
    c = X.generate_synthetic_model(TINY, 3)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 1e9, 1 << 40)]
    h = X.StorageHierarchy(c, None, X.plan_placement(TINY, backends), backends)
    tid = X.ExpertTensorId(2, 1, X.TensorKind.DOWN)
    dest = bytearray(TINY.sigma_down)
    h.fetch(tid, memoryview(dest))
    assert bytes(dest) == c.tensor_bytes(tid)
    with pytest.raises(X.BackendMissError):
        h.fetch(tid, memoryview(bytearray(3)))
    assert h.backend_map().sum() == 0


def test_shared_experts_continue_the_generator_stream():
    """Routed payload unchanged by shared experts; shared words = the stream continued."""
    import numpy as np

    import paper_2604_02715_b200 as X
    from oracle import xpg_oracle as O

    spec = X.ModelSpec(2, 3, 16, 32)
    plain = X.generate_synthetic_model(spec, 9, pin=False)
    c = X.generate_synthetic_model(spec, 9, pin=False, shared_experts=2, chunk_values=100)
    assert np.array_equal(plain.words, c.words)
    n_routed, n_shared = plain.words.size, c.shared.words.size
    stream = O.f32_to_bf16(np.random.default_rng(9).standard_normal(n_routed + n_shared, dtype=np.float32)
                           * O.WEIGHT_STD)
    assert np.array_equal(stream[n_routed:], c.shared.words)
    assert c.shared.tensor_f32(2, 2, X.TensorKind.DOWN).shape == (16, 32)


def test_open_container_mmap_ingest(tmp_path):
    """XPGW ingest by mmap (no read copy): same words/tensors as the generated container,
    and the reference's header checks."""
    import numpy as np
    import pytest

    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200.errors import ContainerFormatError

    spec = X.ModelSpec(2, 3, 16, 32)
    c = X.generate_synthetic_model(spec, 4, pin=False)
    path = tmp_path / "m.xpgw"
    c.write(path)
    o = X.open_container(path, register=False)
    assert o.spec == spec and np.array_equal(o.words, c.words)
    tid = X.ExpertTensorId(2, 3, X.TensorKind.DOWN)
    assert o.tensor_bytes(tid) == c.tensor_bytes(tid)
    raw = path.read_bytes()
    bad = tmp_path / "bad.xpgw"
    bad.write_bytes(b"XPGX" + raw[4:])
    with pytest.raises(ContainerFormatError):
        X.open_container(bad, register=False)
    bad.write_bytes(raw[:-2])
    with pytest.raises(ContainerFormatError):
        X.open_container(bad, register=False)


def test_cli_generate_compress_match_reference_bytes(tmp_path):
    """`python -m paper_2604_02715_b200 generate/compress` write the reference's XPGW/XPGC
    bytes (sha256 pinned to tests/golden from the reference itself)."""
    import hashlib
    import json
    import os

    from paper_2604_02715_b200.__main__ import main
    from paper_2604_02715_b200.exponent_codec import CompressedModel

    meta = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden_v1.json")))["cases"]
    xpgw, xpgc = tmp_path / "m.xpgw", tmp_path / "m.xpgc"
    assert main(["generate", str(xpgw), "--model", "2,3,64,96", "--seed", "11"]) == 0
    payload = xpgw.read_bytes()[40:]
    assert hashlib.sha256(payload).hexdigest() == meta["gen_2_3_64_96_11"]
    assert main(["generate", str(xpgw), "--model", "2,3,64,96"]) == 1  # exists, no --force
    assert main(["generate", str(xpgw), "--model", "3,2,32,64", "--seed", "4", "--force"]) == 0
    assert main(["compress", str(xpgw), str(xpgc)]) == 0
    assert hashlib.sha256(xpgc.read_bytes()).hexdigest() == meta["xpgc_3_2_32_64_4"]["sha256"]
    # XPGC ingest is host-only (bit counts from the index scan) and round-trips its bytes
    assert CompressedModel.read(xpgc).to_bytes() == xpgc.read_bytes()


def test_residency_plan_spends_the_budget():
    """budget.plan_residency: within budget, link-bound budgets buy compressed device-tier
    experts (1.5x more experts per byte than pinning), large budgets pin experts, masks are
    disjoint and every ring window mixes device- and host-tier experts."""
    import numpy as np

    from paper_2604_02715_b200.budget import plan_residency

    eb = 352321536
    ceb = 0.662 * eb
    total = 64 * eb
    prev = None
    for b in (0.1, 0.25, 0.5, 0.8, 1.0):
        pl = plan_residency(8, 8, eb, ceb, b * total)
        assert pl.hbm_bytes <= b * total + 1
        assert not (pl.device_mask & pl.pinned_mask).any()
        if prev is not None:
            assert pl.est_step_s <= prev + 1e-12  # more budget never slower
        prev = pl.est_step_s
    pl = plan_residency(8, 8, eb, ceb, 0.25 * total)  # link-bound: one window in flight, ring of 1
    assert pl.pinned_experts == 0 and pl.device_experts == 22 and pl.ring == 1 and pl.depth == 1
    pl = plan_residency(8, 8, eb, ceb, 0.25 * total, depth=2)  # one 352 MB expert per window: ring of 2
    assert pl.pinned_experts == 0 and pl.device_experts == 21 and pl.ring == 2
    assert plan_residency(8, 8, eb, ceb, 0.65 * total).depth == 2  # decode-bound: double-buffered
    pl = plan_residency(8, 8, eb, ceb, 0.25 * total, window=2, depth=2)
    assert pl.pinned_experts == 0 and pl.device_experts == 18 and pl.ring == 4
    w = pl.ring // 2
    for l in range(8):  # windows of 2 experts: a device expert never shares a window with another
        for j in range(0, 8, w):
            assert pl.device_mask[l, j:j + w].sum() <= 1
    assert plan_residency(8, 8, eb, ceb, 1.0 * total).pinned_experts == 64


def test_residency_plan_narrows_windows_for_small_budgets():
    """Tiny experts: windows sized for min_window_bytes would not fit a 25% budget; the planner
    narrows the window until the ring fits (the tiny bench config)."""
    from paper_2604_02715_b200.budget import plan_residency

    eb = 786432
    pl = plan_residency(4, 8, eb, 0.68 * eb, 0.25 * 32 * eb * 0.998)
    assert 0 < pl.ring < 8 and pl.hbm_bytes <= 0.25 * 32 * eb


def test_residency_plan_spaces_host_experts_and_picks_depth():
    """Host-tier experts are spaced over the layers (not bunched at the ends), and the ring
    keeps one window in flight only while the plan is clearly link-bound."""
    import numpy as np

    from paper_2604_02715_b200.budget import _spaced, plan_residency

    assert _spaced(3, 8) == [0, 1, 0, 0, 1, 0, 1, 0] and _spaced(10, 8) == [1, 1, 2, 1, 1, 1, 2, 1]
    assert sum(_spaced(13, 7)) == 13 and max(_spaced(13, 7)) - min(_spaced(13, 7)) <= 1
    eb = 352321536
    ceb = 0.6655 * 1.012 * eb
    pl = plan_residency(8, 8, eb, ceb, 0.7 * 64 * eb, overhead_bytes=0.7e9)
    host = (~(pl.device_mask | pl.pinned_mask)).sum(axis=1)
    gaps = np.diff(np.flatnonzero(host))
    assert host.sum() >= 2 and gaps.min() >= 2  # never in adjacent layers at this budget
    # once every streamed expert fits on the device tier the staging overhead is not charged,
    # and a few host records no longer pay while the SMs are the bottleneck
    assert (~(plan_residency(8, 8, eb, ceb, 0.8 * 64 * eb).device_mask |
              plan_residency(8, 8, eb, ceb, 0.8 * 64 * eb).pinned_mask)).sum() == 0
    assert plan_residency(8, 8, eb, ceb, 0.25 * 64 * eb).depth == 1
    assert plan_residency(8, 8, eb, ceb, 0.8 * 64 * eb).depth == 2


def test_tier_plan_mixed_device_tier_between_the_formats():
    """budget.plan_tiers: between the budget that holds every streamed expert in Huffman records
    and the one that holds them all in FX4, the mixed plan keeps every expert on the device tier
    (no host record crosses the link), spends the budget on FX4 conversions, and stays within it."""
    import numpy as np

    from paper_2604_02715_b200.budget import fx4_expert_bytes, plan_tiers

    H, F, N, L = 4096, 14336, 32, 8
    eb = 3 * H * F * 2
    ceb, fx = 0.6655 * 1.012 * eb, fx4_expert_bytes(H, F)
    seen = []
    prev = None
    for b in (0.65, 0.7, 0.72, 0.75, 0.78, 0.8):
        pl = plan_tiers(N, L, eb, ceb, b * N * L * eb, fx4_ceb=fx, overhead_bytes=0.8e9, units_per_expert=F // 128)
        assert pl.hbm_bytes <= b * N * L * eb + 1
        if prev is not None:
            assert pl.est_step_s <= prev + 1e-12
        prev = pl.est_step_s
        seen.append(pl.device_format)
        if pl.device_format == "mixed":
            assert pl.host_experts == 0 and pl.link_bytes == 0 and pl.fused == 2
            assert 0 < pl.fx4_experts < pl.device_experts
            assert not (pl.fx4_mask & ~pl.device_mask).any()
            # every layer's Huffman experts come first (ring windows), its FX4 experts after them
            # (one wide decode-into-GEMM window); counts balanced over the layers
            huff = pl.device_mask & ~pl.fx4_mask
            for l in range(N):
                h = int(huff[l].sum())
                assert huff[l, :h].all() and not huff[l, h:].any()
            assert huff.sum(axis=1).max() - huff.sum(axis=1).min() <= 1
    assert "mixed" in seen and seen[-1] == "fx4"
    pl = plan_tiers(N, L, eb, ceb, 0.72 * N * L * eb, fx4_ceb=fx, device_format="mixed", units_per_expert=F // 128)
    assert pl.device_format == "mixed"


def test_fused_plans_pin_whole_layers():
    """Decode-into-GEMM plans pin whole layers (a layer's pinned experts would otherwise run in a
    second, mostly idle GEMM launch beside its FX4 launch), spaced over the stack."""
    from paper_2604_02715_b200.budget import fx4_expert_bytes, plan_tiers

    H, F, N, L = 4096, 14336, 8, 8
    eb = 3 * H * F * 2
    ceb, fx = 0.6655 * 1.012 * eb, fx4_expert_bytes(H, F)
    for b in (0.8, 0.85, 0.9, 0.95):
        pl = plan_tiers(N, L, eb, ceb, b * N * L * eb, fx4_ceb=fx, units_per_expert=F // 128)
        assert pl.hbm_bytes <= b * N * L * eb + 1
        if pl.fused is True:
            per_layer = pl.pinned_mask.sum(axis=1)
            assert set(per_layer.tolist()) <= {0, L}
    pl = plan_tiers(N, L, eb, ceb, 0.9 * N * L * eb, fx4_ceb=fx, units_per_expert=F // 128)
    assert pl.device_format == "fx4" and pl.pinned_experts > 0
    pinned_layers = [l for l in range(N) if pl.pinned_mask[l].all()]
    assert len(pinned_layers) < 2 or min(b - a for a, b in zip(pinned_layers, pinned_layers[1:])) >= 2
