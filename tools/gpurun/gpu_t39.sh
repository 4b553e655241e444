#!/bin/bash
O=gpurun_out/t39; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pagetable.py tests/test_gpu_parity.py tests/test_gpu_residency.py -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head -8
run() { # name, args
  timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.5,0.65,0.8,0.9 "${@:2}" > $O/sweep_$1.jsonl 2> $O/sweep_$1.err; echo "$1 rc=$?"
  python - $1 <<'PY'
import json,sys
for l in open(f"gpurun_out/t39/sweep_{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], d['ring_experts'], d['ring_depth'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1), round(d['hbm_footprint'],3))
PY
}
run d3w1 --depth 3 --window 1
run d4w1 --depth 4 --window 1
run d3w2 --depth 3 --window 2
run d3w1s4 --depth 3 --window 1 --stage-bufs 4
