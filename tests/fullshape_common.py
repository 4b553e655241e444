"""Helpers for the full-shape parity tests (tests/test_gpu_fullshape_*.py).

Weights come from the reference generator (``generate_synthetic_model`` is bit-identical
to xpg model.py:205-214, parallel decode of the same PCG64 stream), inputs are fresh
N(0,1) rows, and every GPU output is compared with the oracle's ``layer_forward``
restatement (reference pipeline.py:192-208) by relative L2 -- never elementwise (deep
synthetic stacks under/overflow by design).  Each measured rel-L2 is
appended to $XPGB_PARITY_LOG (JSON lines) when set, which is where DESIGN.md's per-config
table comes from.
"""
from __future__ import annotations

import json
import os

import numpy as np

TOL = 1e-2  # north star: layer outputs within rel err <= 1e-2, stated per config


def log(config: str, case: str, rel: float, **extra) -> None:
    path = os.environ.get("XPGB_PARITY_LOG")
    if path:
        os.makedirs(os.path.dirname(path) or ".", exist_ok=True)
        with open(path, "a") as fh:
            fh.write(json.dumps({"config": config, "case": case, "rel_l2": rel, **extra}) + "\n")


def fresh_rows(T: int, H: int, seed: int) -> np.ndarray:
    """initial_activations-style float32 N(0,1) rows (pipeline.py:211-213)."""
    return np.random.default_rng(seed ^ 0xA5A5A5).standard_normal((T, H), dtype=np.float32)


def check(O, config: str, case: str, got, want, tol: float = TOL, **extra) -> float:
    got = got.cpu().numpy() if hasattr(got, "cpu") else np.asarray(got)
    assert np.isfinite(want).all(), f"{config} {case}: oracle output not finite (stack too deep)"
    rel = O.rel_l2(got, want)
    log(config, case, rel, **extra)
    assert rel <= tol, f"{config} {case}: rel-L2 {rel:.3e} > {tol}"
    return rel


def paged_runner(X, spec, container, fwd, budget: float = 0.25, **run_kw):
    """The bench's tiering (bench.py): the budget planner's sub-layer ring, compressed device
    tier and exponent-Huffman host tier at ``budget`` of the expert bytes."""
    from paper_2604_02715_b200.budget import plan_residency
    from paper_2604_02715_b200.exponent_codec import CompressedModel

    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 55e9, 1 << 50)]
    cspec = container.spec
    hier = X.StorageHierarchy(container, CompressedModel.from_container(container),
                              X.plan_placement(cspec, backends), backends)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=True, **run_kw)
    L = cspec.experts_per_layer
    ceb = runner.device_tier_bytes(L) / (cspec.num_layers * L) * 1.002
    sb = container.shared.total_bytes if container.shared is not None else 0
    plan = plan_residency(cspec.num_layers, L, cspec.expert_bytes, ceb, budget * (cspec.total_bytes + sb),
                          shared_bytes=sb, overhead_bytes=runner.ctx.hbm_bytes()["staging"])
    runner.apply_plan(plan)
    return runner, plan
