#!/bin/bash
O=gpurun_out/t33; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_codec.py -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -5
for c in mixtral qwen3 dsv3; do timeout 900 python bench.py --config $c --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
python - <<'PY'
import json
for f in ("mixtral","qwen3","dsv3"):
    try:
        d=json.load(open(f"gpurun_out/t33/bench_{f}.json")); c=d['config']
        print(f, round(d['value'],1), round(d['e2e']['value'],1), round(d['page_in']['frac'],3), c['expert_hbm_budget'], c['ring_blocks_per_kind'], c['device_tier_experts_per_layer'], c['pinned_experts_per_layer'])
    except Exception as e: print(f, "ERR", e)
PY
timeout 1500 python tools/sweep.py budget --config mixtral --steps 3 > $O/sweep_budget_mixtral.jsonl 2> $O/sweep.err; echo "sweep rc=$?"
cut -c1-330 $O/sweep_budget_mixtral.jsonl
