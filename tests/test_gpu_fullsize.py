"""Full-size, size-independent parity: the bench's own shapes (Mixtral-8x7B experts, the
DSv3 rank slice) with the bench's own tiering (budget planner at 25%: sub-layer ring,
compressed device tier, exponent-Huffman host tier), cut to two layers.  The paged stack
must be byte-identical to the fully-resident stack on the same kernels, with a clean
ordering log -- the property the small-shape oracle tests pin, checked at 5.6 GB."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _run(X, spec, cspec, T, k, run_kw, shared=0):
    import torch

    from paper_2604_02715_b200.budget import plan_residency
    from paper_2604_02715_b200.exponent_codec import CompressedModel

    G = 1 if not run_kw else spec.experts_per_layer // cspec.experts_per_layer
    fwd = X.ForwardSpec(T * G, k, 7)
    container = X.generate_fast_model(cspec, 7, shared_experts=shared)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 55e9, 1 << 50)]
    hier = X.StorageHierarchy(container, CompressedModel.from_container(container),
                              X.plan_placement(cspec, backends), backends)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=True, **run_kw)
    L = cspec.experts_per_layer
    ceb = runner.device_tier_bytes(L) / (spec.num_layers * L) * 1.002
    sb = container.shared.total_bytes if container.shared is not None else 0
    plan = plan_residency(spec.num_layers, L, spec.expert_bytes, ceb, 0.25 * (cspec.total_bytes + sb),
                          shared_bytes=sb)
    runner.apply_plan(plan)
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((T * G, spec.hidden_dim), dtype=np.float32)).cuda()
    rep = runner.run(2, acts=x.clone())
    assert rep.page_fault is None and rep.violations == []
    assert rep.decoded_bytes > 0 and rep.h2d_bytes > 0
    paged = rep.final_activations.cpu().numpy() if hasattr(rep.final_activations, "cpu") else rep.final_activations
    del runner
    torch.cuda.empty_cache()
    model = X.ResidentModel(spec, container, max_tokens=T * G, **run_kw)
    y, _ = model.run(2, fwd, x.clone())
    resident = y.cpu().numpy() if hasattr(y, "cpu") else y
    assert paged.tobytes() == resident.tobytes()


def test_mixtral_shape_two_layers_paged_equals_resident():
    import paper_2604_02715_b200 as X

    spec = X.ModelSpec(2, 8, 4096, 14336)
    _run(X, spec, spec, 256, 2, {})


def test_dsv3_rank_slice_two_layers_paged_equals_resident():
    import paper_2604_02715_b200 as X

    spec = X.ModelSpec(2, 256, 7168, 2048)
    cspec = X.ModelSpec(2, 32, 7168, 2048)
    _run(X, spec, cspec, 256, 8, {"expert_shard": (0, 32), "shared_tokens": (0, 256)}, shared=1)
