#!/bin/bash
O=gpurun_out/t67; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_pagetable.py -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head -8
run() {
  timeout 900 python tools/sweep.py budget --config $2 --steps 3 --budgets 0.1,0.25,0.5,0.65,0.8 "${@:3}" > $O/sweep_$1.jsonl 2> $O/sweep_$1.err; echo "$1 rc=$?"
  python - $1 <<'PY'
import json,sys
for l in open(f"gpurun_out/t67/sweep_{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], d['ring_experts'], d['ring_depth'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1), round(d['hbm_fraction'],3))
PY
}
run mix_d1 mixtral --depth 1
run ds_d1 dsv3 --depth 1
run qw_d1 qwen3 --depth 1
