#!/bin/bash
O=gpurun_out/t92; mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-resident > $O/bench_under_ncu.log 2>&1; echo "ncu rc=$?"
python tools/launch_list.py $O/launches.csv "ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-resident (default bench: Mixtral decode T=256, 25% budget, planner tiering: ring of 1 expert at depth 1 + device tier, 4-symbol decoder); xpgb kernels only; cold-cache serialised launch times (compare shares, not absolutes)" > $O/launches.json; python -c "
import json; d=json.load(open('$O/launches.json')); print({k:(v['launches'], round(v['share'],3)) for k,v in list(d['kernels'].items())[:6]})"
