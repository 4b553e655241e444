"""Float parity at the Qwen3-30B-A3B layer shape (BASELINE configs[2]: 128 experts, top-8,
hidden 2048, ffn 768) against the oracle's ``layer_forward`` (reference
pipeline.py:192-208), on the reference generator's weights (model.py:205-214; a 5-layer
prefix of the 48-layer model).  Needs a B200.

1-CTA decode GEMMs at T = 1/16/256, CTA-pair GEMMs at T = 4096 (256 rows per expert), the
bench's paged tiering at 25%, and the SURVEY §8(c)(3) short stack (5 layers; the reference
stack underflows at layer 6).
"""
import numpy as np
import pytest

from fullshape_common import check, fresh_rows, paged_runner

pytestmark = pytest.mark.gpu
CFG = "qwen3"
N, L, H, F, K, SEED = 5, 128, 2048, 768, 8, 7


@pytest.fixture(scope="module")
def X():
    import paper_2604_02715_b200 as X

    return X


@pytest.fixture(scope="module")
def O():
    from oracle import xpg_oracle as O

    return O


@pytest.fixture(scope="module")
def model(X, O):
    spec = X.ModelSpec(N, L, H, F)
    c = X.generate_synthetic_model(spec, SEED)
    pool = O.WordPool(N, L, H, F, c.words)
    yield spec, c, pool, X.ResidentModel(spec, c, max_tokens=4096)


@pytest.mark.parametrize("T", [1, 16, 256])
@pytest.mark.parametrize("layer", [1, 3])
def test_layer_vs_oracle_decode(X, O, model, T, layer):
    spec, _, pool, res = model
    x = fresh_rows(T, H, 100 * layer + T)
    y = res.forward(layer, x, X.ForwardSpec(T, K, SEED))
    check(O, CFG, f"layer{layer}_T{T}", y, O.layer_forward(pool, layer, x, K, SEED), path="1-CTA swap-AB")


@pytest.mark.parametrize("force", ["auto", "0"])
def test_layer_vs_oracle_prefill_pair(X, O, model, monkeypatch, force):
    spec, _, pool, res = model
    if force != "auto":
        monkeypatch.setenv("XPGB_PAIR_GEMM", force)
    T = 4096
    x = fresh_rows(T, H, 11)
    y = res.forward(1, x, X.ForwardSpec(T, K, SEED))
    check(O, CFG, f"layer1_T{T}_{'pair' if force == 'auto' else '1cta'}", y, O.layer_forward(pool, 1, x, K, SEED),
          path="CTA-pair" if force == "auto" else "1-CTA")


def test_short_stack_teacher_forced_and_free(X, O, model):
    spec, _, pool, res = model
    T = 16
    fwd = X.ForwardSpec(T, K, SEED)
    a = fresh_rows(T, H, 5)
    g = a.copy()
    for layer in range(1, N + 1):
        want = O.layer_forward(pool, layer, a, K, SEED)
        check(O, CFG, f"stack_teacher_layer{layer}_T{T}", res.forward(layer, a, fwd), want)
        g = res.forward(layer, g, fwd)
        a = want
    check(O, CFG, f"stack_free_{N}layers_T{T}", g, a)


def test_paged_bench_tiering_vs_oracle(X, O, model):
    import torch

    spec, c, pool, res = model
    T = 256
    fwd = X.ForwardSpec(T, K, SEED)
    runner, plan = paged_runner(X, spec, c, fwd)
    assert plan.device_experts > 0
    x = fresh_rows(T, H, 77)
    rep = runner.run(1, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    assert rep.decoded_bytes > 0 and rep.h2d_bytes > 0
    paged = rep.final_activations
    del runner
    torch.cuda.empty_cache()
    check(O, CFG, f"paged25_stack_{N}layers_T{T}", paged, O.resident_stack(pool, x, K, SEED), budget=0.25)
    y, _ = res.run(1, fwd, x.copy())
    assert np.asarray(paged).tobytes() == np.asarray(y).tobytes()
