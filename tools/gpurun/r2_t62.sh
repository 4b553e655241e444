#!/bin/bash
# round 2 final-3: validation of the final tree -- GPU suite, smoke, default bench, reference arm,
# 80% bench, launch list of the default bench
O=gpurun_out/r2_t62; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_all.log 2>&1; echo "all gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/pytest_all.log | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"
for b in 0.75 0.8 0.9; do timeout 900 python bench.py --budget $b --steps 10 --warmup 3 > $O/bench_$b.json 2> $O/bench_$b.err; echo "bench $b rc=$?"; done
for f in bench_default bench bench_0.75 bench_0.8 bench_0.9; do python -c "
import json; d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value']), 'e2e', round(d['e2e']['value']), d['config']['device_tier_format'], r['kernel'][:16], round(r['frac'],3), d.get('paged_over_resident'), d['clocks'])"; done
python -c "
import json; d=json.loads(open('$O/bench_ref.json').read().strip().splitlines()[-1]); print('ref', d['value'], d.get('cpu_baseline'))"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-resident --no-cpu-baseline > $O/bench_under_ncu.log 2>&1; echo "ncu launches rc=$?"
