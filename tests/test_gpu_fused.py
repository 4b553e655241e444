"""Decode-into-GEMM (k_moe_gemm_dec): device-tier experts read in place by the grouped GEMM
must give results byte-identical to decoding them into the ring first and to the fully
resident model, with the same page-table/ordering behaviour (clean log, no fault)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def X():
    import paper_2604_02715_b200 as X

    return X


def _hier(X, container, alpha):
    backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 50),
                X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 50)]
    return X.StorageHierarchy(container, None, X.plan_placement(container.spec, backends, alpha=alpha), backends)


def _run(X, spec, hier, fwd, x, fused, **kw):
    runner = X.StreamedRunner(spec, hier, fwd, fused_decode=fused, **kw)
    rep = runner.run(2, acts=x.copy())
    assert rep.page_fault is None and rep.violations == []
    out = rep.final_activations
    out = out.cpu().numpy() if hasattr(out, "cpu") else out
    return out, rep


@pytest.mark.parametrize("T", [1, 16, 40, 100])
@pytest.mark.parametrize("alpha,host_codec", [(1.0, False), (0.5, True)])
def test_fused_equals_unfused_and_resident(X, T, alpha, host_codec):
    spec = X.ModelSpec(4, 8, 256, 512)
    fwd = X.ForwardSpec(T, 2, 7)
    container = X.generate_synthetic_model(spec, 7)
    hier = _hier(X, container, alpha)
    x = np.random.default_rng(T).standard_normal((T, spec.hidden_dim), dtype=np.float32)
    fz, rf = _run(X, spec, hier, fwd, x, True, host_codec=host_codec)
    uf, ru = _run(X, spec, hier, fwd, x, False, host_codec=host_codec)
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert fz.tobytes() == uf.tobytes() == np.asarray(base).tobytes()
    # the fused run expanded no device-tier expert into the ring
    assert rf.decoded_bytes < ru.decoded_bytes
    if alpha == 1.0:
        assert rf.decoded_bytes == 0


def test_fused_with_sub_layer_ring_and_mixed_windows(X):
    """The bench's tiering: device-tier experts spread over the windows of a sub-layer ring,
    the rest streamed as compressed host records: windows mix fused and ring experts."""
    spec = X.ModelSpec(3, 12, 256, 512)
    fwd = X.ForwardSpec(40, 3, 5)
    container = X.generate_synthetic_model(spec, 5)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    hier = X.StorageHierarchy(container, None, X.plan_placement(spec, backends), backends)
    mask = np.zeros((3, 12), dtype=bool)
    mask[:, [0, 4, 5, 9]] = True
    x = X.initial_activations(spec, fwd, 5)
    outs = []
    for fused in (True, False):
        runner = X.StreamedRunner(spec, hier, fwd, host_codec=True, ring_experts=6, fused_decode=fused)
        runner.set_device_mask(mask)
        rep = runner.run(2, acts=x.copy())
        assert rep.violations == [] and rep.page_fault is None
        outs.append(np.asarray(rep.final_activations).tobytes())
    base = X.resident_baseline(2, spec, container, fwd, acts=x.copy())
    assert outs[0] == outs[1] == np.asarray(base).tobytes()


def test_fused_sabotage_still_faults(X):
    """A device-tier expert read in place is still behind the page table: compute that skips
    its RAW wait on a window faults exactly as with ring blocks (paging.py:228-237)."""
    spec = X.ModelSpec(4, 2, 256, 512)
    container = X.generate_synthetic_model(spec, 2)
    hier = _hier(X, container, 1.0)
    hier.delay_fn = lambda tid: 0.03 if tid.layer == 3 else 0.0
    runner = X.StreamedRunner(spec, hier, X.ForwardSpec(3, 2, 5), sabotage_skip_raw=(1, 3), fused_decode=True)
    rep = runner.run(2)
    assert rep.page_fault is not None
    assert any(v.startswith("RAW") for v in rep.violations)


@pytest.mark.parametrize("shape,T", [("mixtral", 256), ("mixtral", 16), ("qwen3", 256)])
def test_fused_full_shape_equals_resident(X, shape, T):
    """Bench shapes cut to two layers, every expert on the device tier: the decode-into-GEMM
    stack is byte-identical to the resident stack on the same weights."""
    import torch

    from paper_2604_02715_b200.exponent_codec import CompressedModel

    N, L, H, F, k = {"mixtral": (2, 8, 4096, 14336, 2), "qwen3": (2, 128, 2048, 768, 8)}[shape]
    spec = X.ModelSpec(N, L, H, F)
    fwd = X.ForwardSpec(T, k, 7)
    container = X.generate_fast_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 50),
                X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 50)]
    hier = X.StorageHierarchy(container, CompressedModel.from_container(container),
                              X.plan_placement(spec, backends, alpha=1.0), backends)
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((T, H), dtype=np.float32)).cuda()
    runner = X.StreamedRunner(spec, hier, fwd, fused_decode=True)
    rep = runner.run(2, acts=x.clone())
    assert rep.page_fault is None and rep.violations == [] and rep.decoded_bytes == 0
    paged = rep.final_activations.cpu().numpy()
    del runner
    torch.cuda.empty_cache()
    model = X.ResidentModel(spec, container, max_tokens=T)
    y, _ = model.run(2, fwd, x.clone())
    assert paged.tobytes() == y.cpu().numpy().tobytes()
