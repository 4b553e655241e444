#!/bin/bash
O=gpurun_out/t56; mkdir -p $O
for c in qwen3 dsv3; do
  timeout 1500 python tools/sweep.py budget --config $c --steps 3 > $O/sweep_$c.jsonl 2> $O/sweep_$c.err; echo "$c rc=$?"; tail -2 $O/sweep_$c.err
  python - $c <<'PY'
import json,sys
for l in open(f"gpurun_out/t56/sweep_{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], d['ring_experts'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1), round(d['hbm_fraction'],3), round(d['fraction_of_resident'],3))
PY
done
