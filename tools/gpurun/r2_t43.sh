#!/bin/bash
# round 2: budget sweeps with the mixed device tier in the planner (no event profiling)
O=gpurun_out/r2_t43; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1800 python tools/sweep.py budget --config mixtral --steps 5 --warmup 2 --budgets 0.1,0.25,0.5,0.65,0.7,0.72,0.75,0.78,0.8,0.9 > $O/sweep_mixtral.jsonl 2> $O/sweep_mixtral.err; echo "sweep mixtral rc=$?"
for cfg in qwen3 dsv3; do timeout 1800 python tools/sweep.py budget --config $cfg --steps 5 --warmup 2 --budgets 0.25,0.5,0.65,0.7,0.75,0.8,0.9 > $O/sweep_$cfg.jsonl 2> $O/sweep_$cfg.err; echo "sweep $cfg rc=$?"; done
for cfg in mixtral qwen3 dsv3; do python -c "
import json
for l in open('$O/sweep_$cfg.jsonl'):
  d=json.loads(l); print('$cfg', d['budget'], d['device_format'], d['fx4_per_layer'], d['device_tier_per_layer'], d['pinned_per_layer'], d['ring_experts'], round(d['hbm_footprint'],3), round(d['tok_s']), 'planned', round(d['planned_tok_s'] or 0), 'res', round(d['resident_tok_s']), round(d['fraction_of_resident'],3))"; tail -2 $O/sweep_$cfg.err; done
