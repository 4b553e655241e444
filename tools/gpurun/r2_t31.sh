#!/bin/bash
# round 2: host staging released by all-device plans; sweeps; bench at 80%
O=gpurun_out/r2_t31; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_codec.py -q > $O/pytest.log 2>&1; echo "tests rc=$?"; tail -3 $O/pytest.log
timeout 1500 python tools/sweep.py budget --config mixtral --budgets 0.65,0.75,0.8,0.9 > $O/sweep_mixtral.jsonl 2> $O/sweep_mixtral.err; echo "sweep mixtral rc=$?"
for cfg in dsv3 qwen3; do timeout 1500 python tools/sweep.py budget --config $cfg --budgets 0.75,0.8,0.9 > $O/sweep_$cfg.jsonl 2> $O/sweep_$cfg.err; echo "sweep $cfg rc=$?"; done
for cfg in mixtral dsv3 qwen3; do python -c "
import json
for l in open('$O/sweep_$cfg.jsonl'):
  d=json.loads(l); print('$cfg', d['budget'], d['device_format'], d['device_tier_per_layer'], d['pinned_per_layer'], d['ring_experts'], round(d['hbm_footprint'],3), round(d['tok_s']), 'planned', round(d['planned_tok_s'] or 0), 'res', round(d['resident_tok_s']))"; tail -2 $O/sweep_$cfg.err; done
timeout 900 python bench.py --budget 0.8 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench80.json 2> $O/bench80.err; echo "bench80 rc=$?"; head -c 400 $O/bench80.json; echo
