#!/bin/bash
# round 2: planner fix (all-device plans place every streamed expert) -- plan tests, Qwen3 x 48 and Mixtral at 80%
O=gpurun_out/r2_t72; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fx4.py tests/test_gpu_residency.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for spec in "--config qwen3 --layers 48" "--config mixtral"; do
  timeout 1500 python bench.py $spec --budget 0.8 --steps 5 --warmup 3 --no-cpu-baseline > $O/b.json 2> $O/b.err; echo "$spec rc=$?"; python -c "
import json; d=json.loads(open('$O/b.json').read().strip().splitlines()[-1]); c=d['config']
print('$spec', round(d['value']), 'e2e', round(d['e2e']['value']), c['device_tier_format'], 'footprint', c['expert_hbm_footprint'], 'pinned', c['pinned_experts_per_layer'], d.get('paged_over_resident'))"; cp $O/b.json "$O/b_$(echo $spec | tr ' -' '__').json"; done
