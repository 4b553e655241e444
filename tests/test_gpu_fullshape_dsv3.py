"""Float parity at the DeepSeek-V3 layer shape (BASELINE configs[3]: 256 routed experts +
1 shared, top-8, hidden 7168, ffn 2048) for the slice one GPU runs in 8-way expert
parallelism: rank 0's experts 1..32 of every layer routed over all 256, plus the shared
expert on the rank's own tokens.  Needs a B200.

Weights: the reference generator's stream (model.py:205-214) in the shard's layout, so
layer 1 of the shard is bit-identical to the reference model's experts 1..32 of layer 1;
layers 2..7 continue the same stream (the reference model's layer 2 starts 22.5 GB later).
The shared expert is ours (absent from the reference: parity unpinned) and is
checked against the oracle restatement ``layer_forward_shard(..., shared=...)``.

1-CTA GEMMs at 1/16/256 tokens per rank (8/128/2048 routed), CTA-pair GEMMs at 1024 per
rank (256 rows per expert), the bench's paged tiering at 25% and the 7-layer short stack
(the reference stack underflows at layer 8).
"""
import numpy as np
import pytest

from fullshape_common import check, fresh_rows, paged_runner

pytestmark = pytest.mark.gpu
CFG = "dsv3_rank0_of_ep8"
N, L, H, F, K, SEED, G = 7, 256, 7168, 2048, 8, 7, 8
SHARD = (0, 32)


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
    cspec = X.ModelSpec(N, SHARD[1], H, F)
    c = X.generate_synthetic_model(cspec, SEED, shared_experts=1)
    pool = O.WordPool(N, SHARD[1], H, F, c.words)
    sp = O.SharedPool(N, 1, H, F, c.shared.words)
    yield spec, c, pool, sp


def _resident(X, spec, c, t_rank):
    return X.ResidentModel(spec, c, max_tokens=G * t_rank, expert_shard=SHARD, shared_tokens=(0, t_rank))


def _want(O, pool, sp, layer, x, t_rank):
    return O.layer_forward_shard(pool, layer, x, K, SEED, L, SHARD[0], shared=sp, shared_rows=(0, t_rank))


@pytest.mark.parametrize("t_rank", [1, 16, 256, 1024])
def test_layer1_vs_oracle(X, O, model, t_rank):
    spec, c, pool, sp = model
    res = _resident(X, spec, c, t_rank)
    x = fresh_rows(G * t_rank, H, t_rank)
    y = res.forward(1, x, X.ForwardSpec(G * t_rank, K, SEED))
    check(O, CFG, f"layer1_Trank{t_rank}", y, _want(O, pool, sp, 1, x, t_rank),
          path="CTA-pair" if t_rank >= 1024 else "1-CTA swap-AB")


def test_short_stack_teacher_forced_and_free(X, O, model):
    spec, c, pool, sp = model
    t_rank = 16
    res = _resident(X, spec, c, t_rank)
    fwd = X.ForwardSpec(G * t_rank, K, SEED)
    a = fresh_rows(G * t_rank, H, 5)
    g = a.copy()
    for layer in range(1, N + 1):
        want = _want(O, pool, sp, layer, a, t_rank)
        check(O, CFG, f"stack_teacher_layer{layer}_Trank{t_rank}", res.forward(layer, a, fwd), want)
        g = res.forward(layer, g, fwd)
        a = want
    check(O, CFG, f"stack_free_{N}layers_Trank{t_rank}", g, a)


def test_paged_bench_tiering_vs_oracle(X, O, model):
    """Over the first NP layers: with the weight-1 shared expert, the rank slice's 7-layer
    stack overflows float32 at 256 tokens per rank (the reference stack itself would)."""
    import torch

    from paper_2604_02715_b200.geometry import SharedExperts, WeightContainer

    spec7, c7, pool, sp = model
    NP = 4
    spec = X.ModelSpec(NP, L, H, F)
    cspec = X.ModelSpec(NP, SHARD[1], H, F)
    c = WeightContainer._adopt(cspec, c7.pinned[:cspec.total_bytes])  # layer-major: a prefix view
    c.shared = SharedExperts(cspec, 1, c7.shared.pinned[:NP * cspec.expert_bytes])
    t_rank = 256
    fwd = X.ForwardSpec(G * t_rank, K, SEED)
    runner, plan = paged_runner(X, spec, c, fwd, expert_shard=SHARD, shared_tokens=(0, t_rank))
    assert plan.device_experts > 0
    x = fresh_rows(G * t_rank, H, 77)
    rep = runner.run(1, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    assert rep.decoded_bytes > 0 and rep.h2d_bytes > 0
    paged = rep.final_activations
    del runner
    torch.cuda.empty_cache()
    a = x.copy()
    for layer in range(1, NP + 1):
        a = _want(O, pool, sp, layer, a, t_rank)
    check(O, CFG, f"paged25_stack_{NP}layers_Trank{t_rank}", paged, a, budget=0.25)
    y, _ = _resident(X, spec, c, t_rank).run(1, fwd, x.copy())
    assert np.asarray(paged).tobytes() == np.asarray(y).tobytes()
