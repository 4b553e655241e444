#!/bin/bash
# round 2 final-2: full GPU suite on the final tree, sweeps under the recalibrated planner, bench lines
O=gpurun_out/r2_t59; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_all.log 2>&1; echo "all gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/pytest_all.log | tail -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 2400 python tools/sweep.py budget --config mixtral --steps 5 --warmup 2 --budgets 0.1,0.25,0.5,0.65,0.7,0.72,0.75,0.78,0.8,0.85,0.9,0.95 > $O/sweep_mixtral.jsonl 2> $O/sweep_mixtral.err; echo "sweep mixtral rc=$?"
for cfg in qwen3 dsv3; do timeout 1800 python tools/sweep.py budget --config $cfg --steps 5 --warmup 2 --budgets 0.25,0.5,0.7,0.75,0.8,0.9 > $O/sweep_$cfg.jsonl 2> $O/sweep_$cfg.err; echo "sweep $cfg rc=$?"; done
for cfg in mixtral qwen3 dsv3; do python -c "
import json
for l in open('$O/sweep_$cfg.jsonl'):
  d=json.loads(l); print('$cfg', d['budget'], d['device_format'], d['fx4_per_layer'], d['device_tier_per_layer'], d['pinned_per_layer'], d['ring_experts'], round(d['hbm_footprint'],3), round(d['tok_s']), 'planned', round(d['planned_tok_s'] or 0), 'res', round(d['resident_tok_s']))"; done
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; head -c 300 $O/bench.json; echo
for b in 0.75 0.8 0.9; do timeout 900 python bench.py --budget $b --steps 10 --warmup 3 > $O/bench_$b.json 2> $O/bench_$b.err; echo "bench $b rc=$?"; python -c "
import json; d=json.loads(open('$O/bench_$b.json').read().strip().splitlines()[-1]); r=d['roofline']
print($b, round(d['value']), 'e2e', round(d['e2e']['value']), d['config']['device_tier_format'], round(r['frac'],3), d.get('paged_over_resident'))"; done
