"""Live residency planner on a BASELINE config: one JSON line per decode (or prefill) step.

    python tools/live_planner.py [--config mixtral] [--tokens 256] [--budget-experts 3] [--steps 40]

The HBM budget for the device tier is the compressed size of ``--budget-experts``
experts per layer (beside the 2-layer ring); the controller starts at m = 1 and
moves by the reference's dead-zone rule on measured tau_comp / tau_load.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import CONFIGS, SEED  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--budget-experts", type=int, default=3)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--cooldown", type=int, default=2)
    args = ap.parse_args()
    import torch

    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200 import residency as R
    from paper_2604_02715_b200.exponent_codec import CompressedModel

    cfg = dict(CONFIGS[args.config])
    T = args.tokens or cfg["T"]
    spec = X.ModelSpec(cfg["N"], cfg["L"], cfg["H"], cfg["F"])
    fwd = X.ForwardSpec(T, cfg["k"], SEED)
    t0 = time.time()
    c = X.generate_fast_model(spec, SEED)
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 55e9, 1 << 50)]
    hier = X.StorageHierarchy(c, CompressedModel.from_container(c), X.plan_placement(spec, backends), backends)
    runner = X.StreamedRunner(spec, hier, fwd, host_codec=True)
    x = torch.from_numpy(X.initial_activations(spec, fwd, SEED)).cuda()
    b_dev, b_host = R.calibrate_bandwidths(runner, x)
    budget = runner.device_tier_bytes(spec.experts_per_layer) * (args.budget_experts + 0.5) / spec.experts_per_layer
    print(json.dumps({"setup_s": time.time() - t0, "config": args.config, "T": T, "b_dev_GBps": b_dev / 1e9,
                      "b_host_GBps": b_host / 1e9, "device_tier_budget_bytes": budget}), flush=True)
    ctl = R.LiveResidencyController(runner, R.PlannerState(spec.experts_per_layer, 1, cooldown=args.cooldown),
                                    budget, b_dev, b_host)
    for _ in range(args.steps):
        s = ctl.step(x)
        print(json.dumps({"it": s.iteration, "m_layers": s.m_layers, "tau_comp_ms": s.tau_comp * 1e3,
                          "tau_load_ms": s.tau_load * 1e3, "rho": s.rho, "step_ms": s.step_seconds * 1e3,
                          "tok_s": s.tokens_per_second, "migration_bytes": s.migration_bytes,
                          "adjusted": s.adjusted}), flush=True)


if __name__ == "__main__":
    main()
