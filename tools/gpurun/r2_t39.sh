#!/bin/bash
# round 2: format A/B at the 70-80% budgets (Mixtral, T = 256) to calibrate the planner's mixed model
O=gpurun_out/r2_t39; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for b in 0.72 0.75 0.78 0.8; do for f in huffman mixed fx4; do
  timeout 600 python bench.py --budget $b --device-format $f --steps 10 --warmup 3 --no-cpu-baseline --no-resident > $O/bench_${b}_$f.json 2> $O/bench_${b}_$f.err; rc=$?
  python -c "
import json; d=json.loads(open('$O/bench_${b}_$f.json').read().strip().splitlines()[-1]); c=d['config']
print($b, '$f', round(d['value']), round(d['ms_per_step'],2), c['device_tier_format'], c['fx4_experts_per_layer'], c['device_tier_experts_per_layer'], c['pinned_experts_per_layer'], c['ring_blocks_per_kind'], c['expert_hbm_footprint'], round(d['exposed_xfer_pct'],1))" 2>/dev/null || { echo "$b $f rc=$rc"; tail -2 $O/bench_${b}_$f.err; }
done; done
