#!/bin/bash
O=gpurun_out/t75; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log; grep -E "FAILED" $O/pytest.log | head -8
for c in mixtral qwen3 dsv3; do timeout 900 python bench.py --config $c --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
python -c "
import json; d=json.load(open('$O/bench_$c.json')); r=d['roofline']; c=d['config']; print(round(d['value'],1), round(d['e2e']['value'],1), c['expert_hbm_budget'], c['ring_blocks_per_kind'], c['device_tier_experts_per_layer'], round(d['page_in']['achieved_gbps'],1)); print(round(r['achieved'],1), round(r['frac'],3), 'gemm', round(r['gemm']['frac'],3))"; done
for c in mixtral qwen3 dsv3; do timeout 900 python tools/sweep.py budget --config $c --steps 3 --budgets 0.5,0.65,0.8 > $O/sweep_$c.jsonl 2> $O/sweep_$c.err; echo "$c rc=$?"; python - $c <<'PY'
import json,sys
for l in open(f"gpurun_out/t75/sweep_{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], d['ring_experts'], d['ring_depth'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1))
PY
done
