"""PagedTensor semantics of the device-backed PageTable (mirrors reference test_paging.py)."""

import random
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def X():
    import paper_2604_02715_b200 as X

    return X


def tid(X, layer, expert, kind=1):
    return X.ExpertTensorId(layer, expert, X.TensorKind(kind))


def test_pool_capacity_and_exhaustion(X):
    table = X.PageTable(X.ModelSpec(4, 2, 8, 8))
    blocks = [table.map_page(tid(X, ly, e)) for ly in (1, 2) for e in (1, 2)]
    assert sorted(b.block_id for b in blocks) == [1, 2, 3, 4]
    with pytest.raises(X.PoolExhaustedError):
        table.map_page(tid(X, 3, 1))
    table.map_page(tid(X, 3, 1, 2))  # the other kind's pool is independent


def test_double_map_and_not_mapped(X):
    table = X.PageTable(X.ModelSpec(4, 3, 8, 16))
    table.map_page(tid(X, 1, 1))
    with pytest.raises(X.DoubleMapError):
        table.map_page(tid(X, 1, 1))
    with pytest.raises(X.NotMappedError):
        table.unmap_page(tid(X, 2, 1))
    with pytest.raises(X.NotMappedError):
        table.unmap_page(tid(X, 1, 1))  # still loading
    with pytest.raises(X.OutOfRangeError):
        table.map_page(tid(X, 5, 1))


def test_lifecycle_lowest_block_reuse_and_faults(X):
    table = X.PageTable(X.ModelSpec(4, 3, 8, 16))
    b = table.map_page(tid(X, 1, 1))
    assert table.page_state(tid(X, 1, 1)) == X.PageState.LOADING
    with pytest.raises(X.PageFaultError):
        table.read_page(tid(X, 1, 1))
    view = table.loading_view(tid(X, 1, 1))
    payload = np.arange(view.numel(), dtype=np.uint8)
    import torch

    view.copy_(torch.from_numpy(payload))
    table.mark_resident(tid(X, 1, 1))
    assert table.read_page(tid(X, 1, 1)) == payload.tobytes()
    with pytest.raises(X.PageFaultError):
        table.loading_view(tid(X, 1, 1))
    table.unmap_page(tid(X, 1, 1))
    assert table.page_state(tid(X, 1, 1)) == X.PageState.UNMAPPED
    again = table.map_page(tid(X, 2, 1))
    assert again.block_id == b.block_id == 1
    table.check_consistency()


def test_random_ops_against_shadow_model(X):
    spec = X.ModelSpec(4, 3, 8, 16)
    trace = []
    table = X.PageTable(spec, trace=trace)
    rng = random.Random(3)
    ids = list(X.iter_tensor_ids(spec))
    state = {t: "unmapped" for t in ids}
    for _ in range(1500):
        t = rng.choice(ids)
        op = rng.choice(["map", "res", "unmap"])
        try:
            if op == "map":
                table.map_page(t)
                assert state[t] == "unmapped"
                state[t] = "loading"
            elif op == "res":
                table.mark_resident(t)
                assert state[t] == "loading"
                state[t] = "resident"
            else:
                table.unmap_page(t)
                assert state[t] == "resident"
                state[t] = "unmapped"
        except X.DoubleMapError:
            assert state[t] != "unmapped"
        except X.PoolExhaustedError:
            kind_bound = sum(1 for u, s in state.items() if u.kind == t.kind and s != "unmapped")
            assert kind_bound == 2 * spec.experts_per_layer
        except X.NotMappedError:
            assert (op == "res" and state[t] != "loading") or (op == "unmap" and state[t] != "resident")
        assert table.page_state(t).value == state[t]
    table.check_consistency()
    pat = re.compile(r"^event=(map|unmap|state) layer=\d+ expert=\d+ kind=[12] block=\d+ t=\d+( state=\w+)?$")
    assert trace and all(pat.match(line) for line in trace)


def test_fetch_into_loading_view_is_exact(X):
    spec = X.ModelSpec(2, 2, 16, 32)
    c = X.generate_synthetic_model(spec, 9)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 1e9, 1 << 40)]
    h = X.StorageHierarchy(c, None, X.plan_placement(spec, backends), backends)
    table = X.PageTable(spec)
    for t in X.iter_tensor_ids(spec):
        if t.layer == 1:
            table.map_page(t)
            h.fetch(t, table.loading_view(t))
            table.mark_resident(t)
            assert table.read_page(t) == c.tensor_bytes(t)


def test_layer_forward_through_page_table_faults_on_unmapped(X):
    spec = X.ModelSpec(2, 2, 16, 32)
    table = X.PageTable(spec)
    with pytest.raises(X.PageFaultError):
        X.layer_forward(table, spec, X.ForwardSpec(2, 2, 1), 1, np.ones((2, 16), np.float32))


@pytest.mark.parametrize("ring,pinned,host_codec,S,depth", [
    (2, None, False, 0, 2), (4, None, True, 0, 2), (6, None, False, 1, 2), (4, 3, True, 0, 2), (2, 5, False, 1, 2),
    (16, None, False, 0, 2), (3, None, True, 0, 3), (6, 2, False, 1, 3), (4, None, True, 0, 4), (16, None, False, 0, 3),
    (5, 6, True, 0, 5), (2, None, True, 0, 1), (1, None, False, 1, 1), (3, 4, True, 0, 1)])
def test_sub_layer_ring_windows_stay_exact(ring, pinned, host_codec, S, depth):
    """Budgets below two layers: the ring holds `ring` blocks per kind and each layer streams
    in windows of ring/depth experts, `depth` windows in flight; results stay bit-identical to
    the resident model, the log replays clean window by window and the arena never exceeds the
    ring (+ pinned)."""
    import paper_2604_02715_b200 as X

    spec = X.ModelSpec(3, 8, 128, 256)
    fwd = X.ForwardSpec(24, 2, 3)
    c = X.generate_synthetic_model(spec, 3, shared_experts=S)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    hier = X.StorageHierarchy(c, None, X.plan_placement(spec, backends), backends)
    x = X.initial_activations(spec, fwd, 3)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=host_codec, pinned=pinned, ring_experts=ring,
                              ring_depth=depth)
    rep = runner.run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, c, fwd, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    assert rep.final_activations.tobytes() == base.tobytes()
    p = pinned or 0
    streamed = spec.experts_per_layer - p
    ring_used = min(ring // depth * depth, depth * streamed)
    gs = max(1, ring_used // depth)
    windows = max(1, -(-streamed // gs))
    sizes = [min(gs, streamed - i * gs) for i in range(windows)] * (2 * spec.num_layers)
    in_flight = max(sum(sizes[i:i + depth]) for i in range(len(sizes)))  # window g recycles g - depth
    assert rep.arena_peak_bytes == in_flight * spec.expert_bytes + p * spec.num_layers * spec.expert_bytes
    assert in_flight <= ring_used
    starts = [r for r in rep.records if r.event == "compute-start"]
    assert len(starts) == 2 * spec.num_layers * windows
    if windows > 1:
        assert max(r.group for r in starts) == windows - 1
        assert any(r.event == "recycle" and r.target_group is not None for r in rep.records)


def test_sub_layer_ring_sabotage_faults():
    import paper_2604_02715_b200 as X

    spec = X.ModelSpec(3, 6, 64, 128)
    c = X.generate_synthetic_model(spec, 2)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    hier = X.StorageHierarchy(c, None, X.plan_placement(spec, backends), backends, lambda tid: 0.02)
    runner = X.StreamedRunner(spec, hier, X.ForwardSpec(8, 2, 1), sabotage_skip_raw=(1, 2), ring_experts=2)
    rep = runner.run(1)
    assert rep.page_fault is not None
    assert any(v.startswith("RAW") for v in rep.violations)


def test_ring_experts_argument_checks():
    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200.errors import OutOfRangeError

    spec = X.ModelSpec(2, 4, 64, 128)
    ctx = X.PageTable(spec).ctx
    with pytest.raises(OutOfRangeError):
        ctx.set_ring_experts(1)
    ctx.set_ring_experts(-1)
    for bad in (0, 7):
        with pytest.raises(OutOfRangeError):
            ctx.set_ring_depth(bad)
    ctx.set_ring_depth(3)
    with pytest.raises(OutOfRangeError):
        ctx.set_ring_experts(2)   # fewer blocks than windows in flight
    ctx.set_ring_experts(3)
    with pytest.raises(OutOfRangeError):
        ctx.set_ring_depth(4)


def test_ring_resize_keeps_pinned_experts():
    """set_ring_experts after set_pinned keeps the pinned experts resident (regression: the
    arena rebuild used to clear the mask it was reading)."""
    import paper_2604_02715_b200 as X

    spec = X.ModelSpec(3, 6, 64, 128)
    c = X.generate_synthetic_model(spec, 2)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    hier = X.StorageHierarchy(c, None, X.plan_placement(spec, backends), backends)
    fwd = X.ForwardSpec(8, 2, 1)
    runner = X.StreamedRunner(spec, hier, fwd, pinned=2)
    runner.ctx.set_ring_experts(2)
    x = X.initial_activations(spec, fwd, 1)
    rep = runner.run(1, acts=x.copy())
    assert rep.h2d_bytes == spec.num_layers * (spec.experts_per_layer - 2) * spec.expert_bytes
    assert rep.final_activations.tobytes() == X.resident_baseline(1, spec, c, fwd, acts=x.copy()).tobytes()
