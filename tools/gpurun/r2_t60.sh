#!/bin/bash
# round 2: one C call per served iteration -- GPU suite, e2e at 25% / 80%
O=gpurun_out/r2_t60; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_all.log 2>&1; echo "all gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/pytest_all.log | tail -6
for b in 0.25 0.8; do timeout 900 python bench.py --budget $b --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$b.json 2> $O/bench_$b.err; echo "bench $b rc=$?"; python -c "
import json; d=json.loads(open('$O/bench_$b.json').read().strip().splitlines()[-1]); r=d['roofline']
print($b, round(d['value']), 'e2e', round(d['e2e']['value']), d['config']['device_tier_format'], round(r['frac'],3), r.get('traffic'), d.get('paged_over_resident'))"; done
