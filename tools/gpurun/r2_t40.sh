#!/bin/bash
# round 2: does the timed run's per-launch event profiling cost throughput? (A/B, Mixtral)
O=gpurun_out/r2_t40; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for b in 0.7 0.8 0.25; do for np in "" "--no-timed-profile"; do for rep in 1 2; do
  timeout 600 python bench.py --budget $b --steps 10 --warmup 3 --no-cpu-baseline --no-resident $np > $O/b_${b}_${np}_$rep.json 2> $O/b.err
  python -c "
import json; d=json.loads(open('$O/b_${b}_${np}_$rep.json').read().strip().splitlines()[-1]); c=d['config']
print($b, '$np', $rep, round(d['value']), round(d['ms_per_step'],2), c['device_tier_format'], round(d['exposed_xfer_pct'],1))" 2>/dev/null || tail -3 $O/b.err
done; done; done
