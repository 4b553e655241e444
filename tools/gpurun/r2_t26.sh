#!/bin/bash
# round 2: full GPU suite; budget sweeps with the planner's format choice (3 configs); bench 25% / 80%; ncu fused FX4
O=gpurun_out/r2_t26; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_all.log 2>&1; echo "all gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/pytest_all.log | tail -6
for cfg in mixtral qwen3 dsv3; do
  timeout 1500 python tools/sweep.py budget --config $cfg --budgets 0.25,0.5,0.65,0.8,0.9 > $O/sweep_$cfg.jsonl 2> $O/sweep_$cfg.err; echo "sweep $cfg rc=$?"
  python -c "
import json
for l in open('$O/sweep_$cfg.jsonl'):
  d=json.loads(l); print('$cfg', d['budget'], d['device_format'], d['device_tier_per_layer'], d['pinned_per_layer'], round(d['hbm_footprint'],3), round(d['tok_s']), 'planned', round(d['planned_tok_s'] or 0), 'res', round(d['resident_tok_s']))"
done
timeout 900 python bench.py --budget 0.8 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench80.json 2> $O/bench80.err; echo "bench80 rc=$?"; head -c 700 $O/bench80.json; echo
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; head -c 700 $O/bench.json; echo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm_dec -s 2 -c 2 -o $O/fused_fx4 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --steps 1 --modes 1 --device-format fx4 > $O/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
