#!/bin/bash
O=gpurun_out/t57; mkdir -p $O
run() {
  timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.25,0.65,0.8,0.9 > $O/sweep_$1.jsonl 2> $O/sweep_$1.err; echo "$1 rc=$?"
  python - $1 <<'PY'
import json,sys
for l in open(f"gpurun_out/t57/sweep_{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1), 'resident', round(d['resident_tok_s']))
PY
}
run base
XPGB_COSCHED=1 XPGB_DEC_BPS=3 run lean_b3
XPGB_COSCHED=1 XPGB_DEC_BPS=2 run lean_b2
XPGB_COSCHED=1 run lean_b5
