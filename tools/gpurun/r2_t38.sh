#!/bin/bash
# round 2: mixed (per-tensor FX4 + Huffman) device tier -- parity, then Mixtral 0.70-0.78 sweep
O=gpurun_out/r2_t38; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py tests/test_gpu_hazards.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/pytest.log
for b in 0.7 0.72 0.75 0.78; do timeout 900 python bench.py --budget $b --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_$b.json 2> $O/bench_$b.err; echo "mixtral $b rc=$?"; python -c "
import json; d=json.loads(open('$O/bench_$b.json').read().strip().splitlines()[-1]); c=d['config']
print(d['value'], d['e2e']['value'], c['device_tier_format'], c['fx4_experts_per_layer'], c['device_tier_experts_per_layer'], c['pinned_experts_per_layer'], c['expert_hbm_footprint'], d.get('paged_over_resident'), d['exposed_xfer_pct'])"; tail -2 $O/bench_$b.err; done
