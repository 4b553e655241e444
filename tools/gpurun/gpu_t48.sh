#!/bin/bash
O=gpurun_out/t48; mkdir -p $O
run() {
  timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.5,0.65,0.8,0.9 "${@:2}" > $O/sweep_$1.jsonl 2> $O/sweep_$1.err; echo "$1 rc=$?"
  python - $1 <<'PY'
import json,sys
for l in open(f"gpurun_out/t48/sweep_{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], d['ring_experts'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1), round(d['hbm_footprint'],3))
PY
}
run s4 --stage-bufs 4
XPGB_DEC_BPS=3 run bps3
XPGB_DEC_BPS=2 run bps2
