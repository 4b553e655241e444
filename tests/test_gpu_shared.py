"""Shared (always-on) experts, DeepSeek-V3 style: every token passes through each shared
expert after its routed experts, weight 1.0.  Absent from the reference (SURVEY §8(c):
parity unpinned) -- the oracle restatement is ``oracle.xpg_oracle.layer_forward(...,
shared=SharedPool)``.  Needs a B200."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-2


@pytest.fixture(scope="module")
def X():
    import paper_2604_02715_b200 as X

    return X


@pytest.fixture(scope="module")
def O():
    from oracle import xpg_oracle as O

    return O


@pytest.mark.parametrize("L,k,S,T", [(8, 2, 1, 16), (16, 4, 2, 77), (32, 8, 1, 300), (4, 8, 1, 33)])
def test_layer_forward_with_shared_vs_oracle(X, O, L, k, S, T):
    spec = X.ModelSpec(2, L, 128, 256)
    c = X.generate_synthetic_model(spec, 3, shared_experts=S)
    pool = O.WordPool(2, L, 128, 256, c.words)
    sp = O.SharedPool(2, S, 128, 256, c.shared.words)
    x = np.random.default_rng(T).standard_normal((T, 128), dtype=np.float32)
    fwd = X.ForwardSpec(T, k, 5)
    for layer in (1, 2):
        y = X.layer_forward(c.tensor_f32, spec, fwd, layer, x)
        want = O.layer_forward(pool, layer, x, k, 5, shared=sp)
        assert O.rel_l2(y, want) <= TOL
        # the shared expert contributes: without it the result is far off
        assert O.rel_l2(y, O.layer_forward(pool, layer, x, k, 5)) > 10 * TOL


@pytest.mark.parametrize("host_codec,pinned", [(False, None), (True, None), (False, 3)])
def test_streamed_with_shared_equals_resident(X, host_codec, pinned):
    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(48, 2, 7)
    c = X.generate_synthetic_model(spec, 7, shared_experts=1)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    hier = X.StorageHierarchy(c, None, X.plan_placement(spec, backends), backends)
    x = X.initial_activations(spec, fwd, 7)
    rep = X.StreamedRunner(spec, hier, fwd, host_codec=host_codec, pinned=pinned).run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, c, fwd, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    assert rep.final_activations.tobytes() == base.tobytes()
    assert rep.arena_peak_bytes == 2 * (spec.experts_per_layer - (pinned or 0)) * spec.expert_bytes + \
        (pinned or 0) * spec.num_layers * spec.expert_bytes


def test_shared_hbm_footprint_and_removal(X):
    spec = X.ModelSpec(2, 4, 64, 128)
    c = X.generate_synthetic_model(spec, 1, shared_experts=2)
    model = X.ResidentModel(spec, c)
    ring = model.ctx.hbm_bytes()["ring"]
    assert ring == spec.total_bytes + c.shared.total_bytes
    x = np.random.default_rng(0).standard_normal((8, 64), dtype=np.float32)
    fwd = X.ForwardSpec(8, 2, 1)
    with_shared = model.forward(1, x, fwd)
    model.ctx.set_shared(None)
    assert model.ctx.hbm_bytes()["ring"] == spec.total_bytes
    plain = model.forward(1, x, fwd)
    from oracle import xpg_oracle as O

    pool = O.WordPool(2, 4, 64, 128, c.words)
    assert O.rel_l2(plain, O.layer_forward(pool, 1, x, 2, 1)) <= TOL
    assert not np.array_equal(plain, with_shared)


def test_expert_shards_with_shared_sum_to_full_layer(X, O):
    """One expert-parallel rank's slice on one device (expert_shard + shared_tokens): the
    shards' partial layer outputs add up to the full layer (shared experts applied once)."""
    from paper_2604_02715_b200.expert_parallel import shard_payload

    spec = X.ModelSpec(2, 8, 128, 256)
    c = X.generate_synthetic_model(spec, 4, shared_experts=1)
    T, fwd = 40, X.ForwardSpec(40, 2, 6)
    x = np.random.default_rng(1).standard_normal((T, 128), dtype=np.float32)
    full = X.ResidentModel(spec, c, max_tokens=T).forward(1, x, fwd)
    parts = []
    for first, count, sh in ((0, 3, (0, T)), (3, 5, (0, 0))):
        shard = X.WeightContainer._adopt(X.ModelSpec(2, count, 128, 256), shard_payload(c, first, count))
        shard.shared = c.shared
        m = X.ResidentModel(spec, shard, max_tokens=T, expert_shard=(first, count), shared_tokens=sh)
        parts.append(m.forward(1, x, fwd))
    assert O.rel_l2(parts[0] + parts[1], full) <= 1e-5
    # paged shard run of the same slice equals its resident twin
    shard = X.WeightContainer._adopt(X.ModelSpec(2, 5, 128, 256), shard_payload(c, 3, 5))
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    hier = X.StorageHierarchy(shard, None, X.plan_placement(shard.spec, backends), backends)
    rep = X.StreamedRunner(spec, hier, fwd, host_codec=True, expert_shard=(3, 5)).run(1, acts=x.copy())
    twin, _ = X.ResidentModel(spec, shard, max_tokens=T, expert_shard=(3, 5)).run(1, fwd, x.copy())
    assert rep.violations == [] and rep.page_fault is None
    assert rep.final_activations.tobytes() == np.asarray(twin).tobytes()
