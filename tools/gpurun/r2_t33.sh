#!/bin/bash
# round 2: bench lines at 25% (default) and 80% (FX4 in place) for the three configs
O=gpurun_out/r2_t33; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_fx4.py -q > $O/pytest.log 2>&1; echo "tests rc=$?"; tail -1 $O/pytest.log
timeout 900 python bench.py --budget 0.8 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench80.json 2> $O/bench80.err; echo "bench80 rc=$?"; python -c "
import json; d=json.loads(open('$O/bench80.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['e2e']['value'], d['config']['device_tier_format'], d['config']['expert_hbm_footprint'], r['kernel'][:40], round(r['achieved']), round(r['frac'],3), d.get('paged_over_resident'))"
for cfg in qwen3 dsv3; do timeout 900 python bench.py --config $cfg --budget 0.8 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench80_$cfg.json 2> $O/bench80_$cfg.err; echo "bench80 $cfg rc=$?"; python -c "
import json; d=json.loads(open('$O/bench80_$cfg.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['e2e']['value'], d['config']['device_tier_format'], d['config']['expert_hbm_footprint'], r['kernel'][:40], round(r['achieved']), round(r['frac'],3), d.get('paged_over_resident'))"; done
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['e2e']['value'], d['config']['device_tier_format'], d['config']['expert_hbm_footprint'], r['kernel'][:40], round(r['achieved']), round(r['frac'],3), d.get('paged_over_resident'))"
