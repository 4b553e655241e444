#!/bin/bash
O=gpurun_out/t49; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head -8
timeout 600 python bench.py --config mixtral --steps 5 > $O/bench_mixtral.json 2> $O/bench_mixtral.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/bench_mixtral.json')); r=d['roofline']; print(round(d['value'],1), round(d['e2e']['value'],1)); print({k:r[k] for k in ('kernel','achieved','frac','avg_launch_us','launches_per_step','kernel_time_per_step_ms','step_ms')}); print('gemm', round(r['gemm']['frac'],3))"
timeout 600 python bench.py --config mixtral --ep --steps 3 > $O/bench_ep.json 2> $O/bench_ep.err; echo "bench ep rc=$?"; tail -2 $O/bench_ep.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-resident > $O/bench_under_ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_list.py $O/launches.csv "ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-resident (default bench: Mixtral decode T=256, 25% budget, codec tiers); xpgb kernels only; cold-cache serialised launch times (compare shares, not absolutes)" > $O/launches.json; head -c 900 $O/launches.json
