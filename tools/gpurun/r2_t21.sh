#!/bin/bash
# round 2: FX4 (fixed selector) correctness; planner-chosen device-tier format over the budget sweep
O=gpurun_out/r2_t21; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py -q > $O/pytest_fx4.log 2>&1; echo "fx4+fused tests rc=$?"; tail -4 $O/pytest_fx4.log
timeout 1500 python tools/sweep.py budget --config mixtral --budgets 0.25,0.5,0.65,0.8,0.9 > $O/sweep_auto.jsonl 2> $O/sweep_auto.err; echo "sweep rc=$?"
python -c "
import json
for l in open('$O/sweep_auto.jsonl'):
  d=json.loads(l); print(d['budget'], d['device_format'], d['fused_decode'], d['device_tier_per_layer'], d['pinned_per_layer'], round(d['hbm_footprint'],3), round(d['tok_s']), 'planned', round(d['planned_tok_s'] or 0), 'res', round(d['resident_tok_s']))"
tail -3 $O/sweep_auto.err
timeout 900 python bench.py --budget 0.8 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench80.json 2> $O/bench80.err; echo "bench80 rc=$?"; head -c 1800 $O/bench80.json; tail -2 $O/bench80.err
