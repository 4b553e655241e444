#!/bin/bash
O=gpurun_out/t72; mkdir -p $O
for c in qwen3 dsv3; do timeout 900 python bench.py --config $c --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
python -c "
import json; d=json.load(open('$O/bench_$c.json')); r=d['roofline']; c=d['config']; print(round(d['value'],1), round(d['e2e']['value'],1), c['expert_hbm_budget'], c['ring_blocks_per_kind'], c['device_tier_experts_per_layer'], c['pinned_experts_per_layer'], round(d['page_in']['achieved_gbps'],1), d['resident'].get('tok_s'), d.get('raw_host_tier',{}).get('tok_s')); print(round(r['achieved'],1), round(r['frac'],3), 'gemm', round(r['gemm']['frac'],3), d['cpu_baseline']['value'])"; done
