#!/bin/bash
O=gpurun_out/t83; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log; grep -E "FAILED" $O/pytest.log | head -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 10 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/bench.json')); r=d['roofline']; c=d['config']; print(round(d['value'],1), round(d['e2e']['value'],1), c['expert_hbm_budget'], c['ring_blocks_per_kind'], c['device_tier_experts_per_layer'], d['clocks']); print(round(r['achieved'],1), round(r['frac'],3), 'gemm', round(r['gemm']['frac'],3), d['cpu_baseline'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-resident > $O/bench_under_ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_list.py $O/launches.csv "ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-resident (default bench: Mixtral decode T=256, 25% budget, planner tiering: ring of 1 expert at depth 1 + device tier); xpgb kernels only; cold-cache serialised launch times (compare shares, not absolutes)" > $O/launches.json; python -c "
import json; d=json.load(open('$O/launches.json')); print({k:(v['launches'], round(v['share'],3)) for k,v in list(d['kernels'].items())[:5]})"
