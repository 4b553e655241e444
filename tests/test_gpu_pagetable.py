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
