#!/bin/bash
# round 2: Qwen3 at its full 48 layers, final tree
O=gpurun_out/r2_t71; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for b in 0.25 0.8; do timeout 1500 python bench.py --config qwen3 --layers 48 --budget $b --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_qwen3_48_$b.json 2> $O/bench_qwen3_48_$b.err; echo "qwen3-48 $b rc=$?"; python -c "
import json; d=json.loads(open('$O/bench_qwen3_48_$b.json').read().strip().splitlines()[-1]); r=d['roofline']
print($b, round(d['value']), 'e2e', round(d['e2e']['value']), d['config']['workload'][:50], d['config']['device_tier_format'], d['config']['expert_hbm_footprint'], d.get('paged_over_resident'), round(r['frac'],3))"; tail -1 $O/bench_qwen3_48_$b.err; done
