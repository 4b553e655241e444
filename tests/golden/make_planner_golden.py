"""Dump planner decisions and landscape traces from the reference ``xpg.planner``
(run in the dev container, where /root/reference exists; the output is committed).

    python tests/golden/make_planner_golden.py   ->  tests/golden/planner_v1.json
"""

from __future__ import annotations

import itertools
import json
import math
import os
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

RHOS = [0.0, 0.5, 0.8999, 0.9, 0.95, 1.0, 1.0000001, 1.5, "inf"]
BUDGETS = [None, (3.5e9, 0.0, 8e9), (10e9, 6e9, 8e9), (1e9, 0.0, 0.0)]


def estimator(kind):
    if kind == "none":
        return None
    if kind == "steep":
        return lambda a: 0.2 + 2.0 * a  # >= 1 only for alpha >= 0.4
    return lambda a: 5.0  # always compute-bound


def main():
    sys.path.insert(0, REF)
    from xpg import planner as P

    cases = []
    for L, theta, step, est, bud in itertools.product((4, 8), (0.9, 1.0), (1, 2), ("none", "steep", "flat"),
                                                      BUDGETS):
        for m in range(1, L + 1):
            for rho in RHOS:
                r = math.inf if rho == "inf" else rho
                st = P.PlannerState(experts_per_layer=L, device_experts=m, theta=theta, step_experts=step)
                b = P.MemoryBudget(float("inf"), 0.0, 0.0) if bud is None else P.MemoryBudget(*bud)
                out = P.plan_step(st, r, b, estimator(est))
                cases.append({"L": L, "m": m, "theta": theta, "step": step, "est": est, "budget": bud,
                              "rho": rho, "out_m": out.device_experts})
    loops = []
    curves = {"knee": [None] + [8.0 - 0.9 * m for m in range(1, 9)],
              "flat": [None] + [2.0] * 8,
              "cliff": [None] + [10.0, 9.0, 8.0, 1.0, 0.9, 0.8, 0.7, 0.6]}
    for name, curve in curves.items():
        for noise, seed, cooldown, m0 in ((0.0, 0, 3, 1), (0.2, 7, 5, 4), (0.5, 3, 2, 8)):
            st = P.PlannerState(experts_per_layer=8, device_experts=m0, cooldown=cooldown)
            res = P.run_landscape_loop(curve, 4.0, st, 60, noise_amplitude=noise, seed=seed)
            loops.append({"curve": name, "tau_by_m": curve, "noise": noise, "seed": seed, "cooldown": cooldown,
                          "m0": m0, "alphas": list(res.alphas), "adjustments": [list(a) for a in res.adjustments],
                          "reversals": res.reversals, "final_m": res.final_m})
    with open(os.path.join(HERE, "planner_v1.json"), "w") as fh:
        json.dump({"reference": "xpg 0.1.0 planner.py", "plan_step": cases, "landscape": loops}, fh)
    print(len(cases), "plan_step cases,", len(loops), "landscape loops")


if __name__ == "__main__":
    main()
