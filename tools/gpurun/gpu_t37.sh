#!/bin/bash
O=gpurun_out/t37; mkdir -p $O
for v in "" 1; do
  XPGB_FLAT_PRIORITY=$v timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.25,0.5,0.65,0.8,0.9 > $O/sweep_flat$v.jsonl 2> $O/sweep_flat$v.err; echo "flat=$v rc=$?"
  python - $v <<'PY'
import json,sys
for l in open(f"gpurun_out/t37/sweep_flat{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1), round(d['hbm_footprint'],3))
PY
done
XPGB_LOG=1 timeout 300 python tools/debug_plan.py 0.65 > $O/plan_0.65.txt 2>&1
