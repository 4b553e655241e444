#!/bin/bash
# round 2: fused experts map without ring blocks (virtual pages); all-device plans with tiny rings
O=gpurun_out/r2_t32; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -x > $O/pytest_all.log 2>&1; echo "all gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/pytest_all.log | tail -6
timeout 600 python tools/sanitize_run.py > $O/plain.log 2>&1; echo "sanitize-run plain rc=$?"; grep -c "ok$" $O/plain.log
timeout 1500 python tools/sweep.py budget --config mixtral --budgets 0.75,0.8,0.9 > $O/sweep_mixtral.jsonl 2> $O/sweep_mixtral.err; echo "sweep mixtral rc=$?"
for cfg in dsv3 qwen3; do timeout 1500 python tools/sweep.py budget --config $cfg --budgets 0.75,0.8,0.9 > $O/sweep_$cfg.jsonl 2> $O/sweep_$cfg.err; echo "sweep $cfg rc=$?"; done
for cfg in mixtral dsv3 qwen3; do python -c "
import json
for l in open('$O/sweep_$cfg.jsonl'):
  d=json.loads(l); print('$cfg', d['budget'], d['device_format'], d['device_tier_per_layer'], d['pinned_per_layer'], d['ring_experts'], round(d['hbm_footprint'],3), round(d['tok_s']), 'planned', round(d['planned_tok_s'] or 0), 'res', round(d['resident_tok_s']))"; tail -2 $O/sweep_$cfg.err; done
