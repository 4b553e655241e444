#!/bin/bash
O=gpurun_out/t78; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_codec.py tests/test_gpu_residency.py -q -x > $O/pt.log 2>&1; tail -1 $O/pt.log
for c in mixtral dsv3 qwen3; do timeout 900 python tools/sweep.py budget --config $c --steps 3 --budgets 0.25,0.5,0.65,0.8,0.9 > $O/sweep_$c.jsonl 2> $O/sweep_$c.err; echo "$c rc=$?"; python - $c <<'PY'
import json,sys
for l in open(f"gpurun_out/t78/sweep_{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], d['ring_experts'], d['ring_depth'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1))
PY
done
