"""Dump golden vectors of the reference simulator (xpg simulate.py / planner.py closed loop)
for tests/test_simulate_cpu.py.  Run in a container that has the reference:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_sim_golden.py

Writes tests/golden/sim_golden.json (small: a few configs x tens of iterations)."""
import json
import os

from xpg import planner, simulate
from xpg.model import ModelSpec

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "sim_golden.json")


def cfg(spec, **kw):
    base = dict(b_dev=400e9, b_host=25e9, tau_comp_theory=0.02, batch_size=16, context_start=512,
                max_new_tokens=60, kv_bytes_per_token=1 << 20, non_expert_bytes=1 << 30,
                swap_bandwidth=20e9, compression_ratio=0.66)
    base.update(kw)
    window = 2 * spec.experts_per_layer * spec.expert_bytes
    base.setdefault("c_gpu", int(window + base["non_expert_bytes"] + 0.3 * spec.total_bytes))
    return simulate.SimConfig(spec=spec, **base)


def main():
    cases = []
    specs = {"tiny": ModelSpec(4, 8, 256, 512), "mixtral": ModelSpec(8, 8, 4096, 14336),
             "qwen3_8": ModelSpec(8, 128, 2048, 768)}
    for name, spec in specs.items():
        for kw in ({}, {"tau_comp_theory": 0.2, "b_host": 55e9}, {"kv_bytes_per_token": 64 << 20,
                                                                   "max_new_tokens": 30}):
            c = cfg(spec, **kw)
            grid = [m / spec.experts_per_layer for m in range(1, spec.experts_per_layer + 1, max(1, spec.experts_per_layer // 8))]
            samples = simulate.simulate_decode(c, 0.25)
            st = planner.PlannerState(experts_per_layer=spec.experts_per_layer,
                                      device_experts=max(1, spec.experts_per_layer // 4), cooldown=5)
            loop_samples, trace = planner.run_control_loop(c, st)
            cases.append({
                "spec": [spec.num_layers, spec.experts_per_layer, spec.hidden_dim, spec.intermediate_dim],
                "config": {k: getattr(c, k) for k in ("b_dev", "b_host", "tau_comp_theory", "batch_size",
                                                         "context_start", "max_new_tokens", "kv_bytes_per_token",
                                                         "c_gpu", "non_expert_bytes", "swap_bandwidth",
                                                         "compression_ratio")},
                "knee": simulate.knee_alpha(c),
                "sweep": simulate.sweep_alpha(c, grid),
                "fixed_alpha_samples": [[s.iteration, s.kv_bytes, s.alpha, s.tau_load, s.tau_comp_actual,
                                         s.iteration_time, s.throughput, s.rho, s.kv_overflow] for s in samples],
                "loop_trace": [[r.iteration, r.rho, r.alpha, r.c_kv, r.c_exp, r.throughput, r.adjusted]
                               for r in trace],
            })
    with open(OUT, "w") as fh:
        json.dump({"source": "xpg 0.1.0 simulate.py / planner.py", "cases": cases}, fh)
    print("wrote", OUT, len(cases), "cases")


if __name__ == "__main__":
    main()
