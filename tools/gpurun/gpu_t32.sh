#!/bin/bash
O=gpurun_out/t32; mkdir -p $O
for c in mixtral qwen3 dsv3; do timeout 900 python bench.py --config $c --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
python - <<'PY'
import json
for f in ("mixtral","qwen3","dsv3"):
    try:
        d=json.load(open(f"gpurun_out/t32/bench_{f}.json")); c=d['config']
        print(f, round(d['value'],1), round(d['e2e']['value'],1), round(d['page_in']['frac'],3), round(d['exposed_xfer_pct'],1), c['expert_hbm_budget'], c['expert_hbm_footprint'], c['ring_blocks_per_kind'], c['device_tier_experts_per_layer'], d.get('paged_over_resident'), round(d['roofline']['frac'],3))
    except Exception as e: print(f, "ERR", e)
PY
tail -3 $O/bench_mixtral.err
