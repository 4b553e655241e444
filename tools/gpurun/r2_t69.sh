#!/bin/bash
# round 2 last: full GPU suite, smoke and the default bench on the final tree
O=gpurun_out/r2_t69; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_all.log 2>&1; echo "all gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/pytest_all.log | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
timeout 900 python bench.py --budget 0.8 --steps 10 --warmup 3 > $O/bench_0.8.json 2> $O/bench_0.8.err; echo "bench 0.8 rc=$?"
for f in bench_default bench_0.8; do python -c "
import json; d=json.loads(open('$O/$f.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', round(d['value']), 'e2e', round(d['e2e']['value']), d['config']['device_tier_format'], r['kernel'][:16], round(r['frac'],3), r.get('traffic'), d.get('paged_over_resident'), d['gpu_launches'], d['clocks'])"; done
