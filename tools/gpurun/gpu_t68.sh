#!/bin/bash
O=gpurun_out/t68; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log; grep -E "FAILED" $O/pytest.log | head -8
timeout 600 python bench.py --config mixtral --steps 5 > $O/bench_mixtral.json 2> $O/bench_mixtral.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/bench_mixtral.json')); r=d['roofline']; c=d['config']; print(round(d['value'],1), round(d['e2e']['value'],1), c['expert_hbm_budget'], c['ring_blocks_per_kind'], c['device_tier_experts_per_layer']); print(round(r['achieved'],1), round(r['frac'],3), 'gemm', round(r['gemm']['frac'],3))"
for c in mixtral qwen3 dsv3; do timeout 1200 python tools/sweep.py budget --config $c --steps 3 > $O/sweep_$c.jsonl 2> $O/sweep_$c.err; echo "$c rc=$?"; python - $c <<'PY'
import json,sys
for l in open(f"gpurun_out/t68/sweep_{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], d['ring_experts'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1), round(d['fraction_of_resident'],3))
PY
done
