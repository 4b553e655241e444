#!/bin/bash
O=gpurun_out/t38; mkdir -p $O
for v in prio flat; do
  if [ $v = flat ]; then export XPGB_FLAT_PRIORITY=1; fi
  timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.25,0.5,0.65,0.8,0.9 > $O/sweep_$v.jsonl 2> $O/sweep_$v.err; echo "$v rc=$?"
  python - $v <<'PY'
import json,sys
for l in open(f"gpurun_out/t38/sweep_{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1), round(d['hbm_footprint'],3))
PY
done
unset XPGB_FLAT_PRIORITY
XPGB_LOG=1 timeout 300 python tools/debug_plan.py 0.8 > $O/plan_0.8.txt 2>&1
