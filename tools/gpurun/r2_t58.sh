#!/bin/bash
# round 2: compute-sanitizer on every tier incl. the TMEM-A FX4 kernel, the gate/up -> down overlap and the mixed tier
O=gpurun_out/r2_t58; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 600 python tools/sanitize_run.py > $O/plain.log 2>&1; echo "plain rc=$?"; cat $O/plain.log | tail -10
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_run.py > $O/sanitize_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok$|MISMATCH" $O/sanitize_$tool.log | tail -14
done
timeout 900 python -m paper_2604_02715_b200 calibrate --model 8,8,4096,14336 --tokens 256 --top-k 2 --out $O/calib_mixtral.json > $O/calib.log 2>&1; echo "calibrate rc=$?"; cat $O/calib_mixtral.json
timeout 1500 python tools/sweep.py budget --config mixtral --budgets 0.1,0.25,0.5,0.65,0.8,0.9 > $O/sweep_mixtral.jsonl 2> $O/sweep_mixtral.err; echo "sweep mixtral rc=$?"
for cfg in dsv3 qwen3; do timeout 1500 python tools/sweep.py budget --config $cfg --budgets 0.8,0.9 > $O/sweep_$cfg.jsonl 2> $O/sweep_$cfg.err; echo "sweep $cfg rc=$?"; done
for cfg in mixtral dsv3 qwen3; do python -c "
import json
for l in open('$O/sweep_$cfg.jsonl'):
  d=json.loads(l); print('$cfg', d['budget'], d['device_format'], d['device_tier_per_layer'], d['pinned_per_layer'], d['ring_experts'], round(d['hbm_footprint'],3), round(d['tok_s']), 'planned', round(d['planned_tok_s'] or 0), 'res', round(d['resident_tok_s']))"; done
timeout 900 python bench.py --gpus 2 --oversubscribe --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_gpus2.json 2> $O/bench_gpus2.err; echo "bench --gpus 2 rc=$?"; head -c 900 $O/bench_gpus2.json; echo; tail -3 $O/bench_gpus2.err
