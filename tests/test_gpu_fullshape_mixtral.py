"""Float parity at the Mixtral-8x7B layer shape (BASELINE configs[1]: 8 experts, top-2,
hidden 4096, ffn 14336) against the oracle's ``layer_forward`` (reference
pipeline.py:192-208), on the reference generator's weights (model.py:205-214; the 6-layer
model is a bit-exact prefix of the 8-layer one).  Needs a B200.

Covers the paths the bench runs: the 1-CTA swap-AB decode GEMMs (T = 1/16/256, split-K
down projection), the CTA-pair GEMMs (T = 1024: 256 rows per expert), and the paged
tiering of the bench (budget planner at 25%: one-expert sub-layer ring, compressed device
tier, exponent-Huffman host tier), plus the SURVEY §8(c)(3) short stack (6 layers; the
reference stack overflows at layer 8).
"""
import numpy as np
import pytest

from fullshape_common import TOL, check, fresh_rows, paged_runner

pytestmark = pytest.mark.gpu
CFG = "mixtral"
N, L, H, F, K, SEED = 6, 8, 4096, 14336, 2, 7


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
    yield spec, c, pool, X.ResidentModel(spec, c, max_tokens=1024)


@pytest.mark.parametrize("T", [1, 16, 256])
@pytest.mark.parametrize("layer", [1, 2])
def test_layer_vs_oracle_decode(X, O, model, T, layer):
    spec, _, pool, res = model
    x = fresh_rows(T, H, 100 * layer + T)
    y = res.forward(layer, x, X.ForwardSpec(T, K, SEED))
    check(O, CFG, f"layer{layer}_T{T}", y, O.layer_forward(pool, layer, x, K, SEED), path="1-CTA swap-AB")


@pytest.mark.parametrize("force", ["auto", "0"])
def test_layer_vs_oracle_prefill_pair(X, O, model, monkeypatch, force):
    """T = 1024: 256 rows per expert, the CTA-pair kernel (auto); =0 forces the 1-CTA kernel."""
    spec, _, pool, res = model
    if force != "auto":
        monkeypatch.setenv("XPGB_PAIR_GEMM", force)
    T = 1024
    x = fresh_rows(T, H, 9)
    y = res.forward(1, x, X.ForwardSpec(T, K, SEED))
    check(O, CFG, f"layer1_T{T}_{'pair' if force == 'auto' else '1cta'}", y, O.layer_forward(pool, 1, x, K, SEED),
          path="CTA-pair" if force == "auto" else "1-CTA")


def test_short_stack_teacher_forced_and_free(X, O, model):
    """Every layer of the 6-layer stack on the oracle's own input (per-layer error), then
    the free-running GPU stack against the oracle stack."""
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
    """The bench's paged tiering at 25% over the 6-layer stack (T = 256): equal to the
    oracle stack within tolerance and byte-identical to the resident GPU stack."""
    import torch

    spec, c, pool, res = model
    T = 256
    fwd = X.ForwardSpec(T, K, SEED)
    runner, plan = paged_runner(X, spec, c, fwd)
    assert plan.device_experts > 0  # the compressed device tier is exercised
    x = fresh_rows(T, H, 77)
    rep = runner.run(1, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    assert rep.decoded_bytes > 0 and rep.h2d_bytes > 0
    paged = rep.final_activations
    del runner
    torch.cuda.empty_cache()
    want = O.resident_stack(pool, x, K, SEED)
    check(O, CFG, f"paged25_stack_{N}layers_T{T}", paged, want, budget=0.25)
    y, _ = res.run(1, fwd, x.copy())
    assert np.asarray(paged).tobytes() == np.asarray(y).tobytes()
