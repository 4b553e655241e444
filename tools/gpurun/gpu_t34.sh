#!/bin/bash
O=gpurun_out/t34; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head -8
timeout 600 python bench.py --config mixtral --steps 5 > $O/bench_mixtral.json 2> $O/bench_mixtral.err; echo "bench rc=$?"
timeout 600 python bench.py --config mixtral --ep --steps 3 > $O/bench_ep.json 2> $O/bench_ep.err; echo "bench ep rc=$?"; tail -3 $O/bench_ep.err
python - <<'PY'
import json
for f in ("mixtral","ep"):
    try:
        d=json.load(open(f"gpurun_out/t34/bench_{f}.json")); c=d['config']
        print(f, round(d['value'],1), round(d['e2e']['value'],1), c.get('expert_hbm_budget'), c.get('ring_blocks_per_kind'), c.get('device_tier_experts_per_layer'), c.get('pinned_experts_per_layer'))
    except Exception as e: print(f, "ERR", e)
PY
timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.25,0.5,0.65,0.8,0.9 > $O/sweep_budget_mixtral.jsonl 2> $O/sweep.err; echo "sweep rc=$?"
python - <<'PY'
import json
for l in open("gpurun_out/t34/sweep_budget_mixtral.jsonl"):
    d=json.loads(l); print(d['budget'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1))
PY
