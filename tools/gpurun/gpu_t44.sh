#!/bin/bash
O=gpurun_out/t44; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in qwen3 dsv3; do timeout 900 python bench.py --config $c --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
python - <<'PY'
import json
for f in ("qwen3","dsv3"):
    try:
        d=json.load(open(f"gpurun_out/t44/bench_{f}.json")); c=d['config']
        print(f, round(d['value'],1), round(d['e2e']['value'],1), c['expert_hbm_budget'], c['ring_blocks_per_kind'], c['device_tier_experts_per_layer'], c['pinned_experts_per_layer'])
    except Exception as e: print(f, "ERR", e)
PY
timeout 900 python tools/sweep.py budget --config mixtral --steps 3 > $O/sweep_budget_mixtral.jsonl 2> $O/sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/t44/sweep_budget_mixtral.jsonl"):
    d=json.loads(l); print(d['budget'], d['ring_experts'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1), round(d['hbm_footprint'],3), round(d['fraction_of_resident'],3))
PY
