"""CTA-pair (cta_group::2) grouped GEMM used for prefill-sized expert groups.  Needs a B200.

XPGB_PAIR_GEMM=1 forces the pair kernel at any size (ragged 256-row token tiles,
experts with fewer rows than a tile), =0 forces the 1-CTA kernel."""

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


@pytest.mark.parametrize("L,k,T,S", [(8, 2, 600, 0), (4, 2, 1000, 1), (16, 4, 333, 0), (3, 3, 2, 0)])
def test_pair_gemm_layer_vs_oracle(X, O, monkeypatch, L, k, T, S):
    monkeypatch.setenv("XPGB_PAIR_GEMM", "1")
    spec = X.ModelSpec(2, L, 256, 512)
    c = X.generate_synthetic_model(spec, 4, shared_experts=S)
    pool = O.WordPool(2, L, 256, 512, c.words)
    sp = O.SharedPool(2, S, 256, 512, c.shared.words) if S else None
    x = np.random.default_rng(T).standard_normal((T, 256), dtype=np.float32)
    fwd = X.ForwardSpec(T, k, 2)
    model = X.ResidentModel(spec, c, max_tokens=T)
    for layer in (1, 2):
        y = model.forward(layer, x, fwd)
        assert O.rel_l2(y, O.layer_forward(pool, layer, x, k, 2, shared=sp)) <= TOL


def test_pair_gemm_streamed_equals_resident(X, monkeypatch):
    monkeypatch.setenv("XPGB_PAIR_GEMM", "1")
    spec = X.ModelSpec(3, 8, 256, 512)
    fwd = X.ForwardSpec(700, 2, 5)
    c = X.generate_synthetic_model(spec, 5)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    hier = X.StorageHierarchy(c, None, X.plan_placement(spec, backends), backends)
    x = X.initial_activations(spec, fwd, 5)
    rep = X.StreamedRunner(spec, hier, fwd, host_codec=True, ring_experts=4).run(2, acts=x.copy())
    base = X.resident_baseline(2, spec, c, fwd, acts=x.copy())
    assert rep.violations == [] and rep.page_fault is None
    assert rep.final_activations.tobytes() == base.tobytes()


def test_pair_gemm_auto_at_prefill_size_matches_one_cta(X, O, monkeypatch):
    """Mixtral-width layer at a prefill size: the auto path (pair) against the 1-CTA path."""
    spec = X.ModelSpec(2, 8, 4096, 1024)
    c = X.generate_fast_model(spec, 3)
    T = 4096
    x = np.random.default_rng(1).standard_normal((T, 4096), dtype=np.float32)
    fwd = X.ForwardSpec(T, 2, 3)
    monkeypatch.setenv("XPGB_PAIR_GEMM", "0")
    y1 = X.ResidentModel(spec, c, max_tokens=T).forward(1, x, fwd)
    monkeypatch.delenv("XPGB_PAIR_GEMM")
    model = X.ResidentModel(spec, c, max_tokens=T)
    y2 = model.forward(1, x, fwd)
    assert O.rel_l2(y2, y1) <= 1e-3
    prof = model.ctx.profile_layer(1, *[__import__("torch").from_numpy(a).cuda() for a in (x, x.copy())], T, 2, 3,
                                   reps=1)
    assert prof["gate_up_ns"] > 0
