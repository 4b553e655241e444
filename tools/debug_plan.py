"""Per-window load/compute spans of one planned decode step (debugging the budget planner)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_02715_b200 as X  # noqa: E402
from paper_2604_02715_b200.budget import plan_residency  # noqa: E402
from paper_2604_02715_b200.exponent_codec import CompressedModel  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 0.8
spec = X.ModelSpec(8, 8, 4096, 14336)
fwd = X.ForwardSpec(256, 2, 7)
c = X.generate_fast_model(spec, 7)
backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 55e9, 1 << 50)]
hier = X.StorageHierarchy(c, CompressedModel.from_container(c), X.plan_placement(spec, backends), backends)
runner = X.StreamedRunner(spec, hier, fwd, host_codec=True)
ceb = runner.device_tier_bytes(8) / 64 * 1.002
plan = plan_residency(8, 8, spec.expert_bytes, ceb, budget * spec.total_bytes)
runner.apply_plan(plan)
print("ring", plan.ring, "device", plan.device_mask.astype(int).tolist()[0], "pinned", plan.pinned_mask.astype(int).tolist()[0])
x = torch.from_numpy(X.initial_activations(spec, fwd, 7)).cuda()
runner.run(2, acts=x)
rep = runner.run(2, acts=x)
print("elapsed ms", rep.elapsed_seconds * 1e3, "h2d GB", rep.h2d_bytes / 1e9, "decoded GB", rep.decoded_bytes / 1e9)
last = max(r.iteration for r in rep.records)
t0 = min(r.wall for r in rep.records if r.iteration == last)
rows = {}
for r in rep.records:
    if r.iteration != last:
        continue
    key = (r.layer, r.group)
    rows.setdefault(key, {})[(r.event, r.kind)] = round((r.wall - t0) * 1e3, 2)
print("layer win | ls1 ls2 | ld1 ld2 | cs cd   (ms from the iteration's first record)")
for (layer, g), d in sorted(rows.items()):
    get = lambda e, k: d.get((e, k), "-")
    print(layer, g, "|", get("load-start", 1), get("load-start", 2), "|", get("load-done", 1), get("load-done", 2),
          "|", get("compute-start", None), get("compute-done", None))
