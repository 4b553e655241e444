#!/bin/bash
# round 2: gate/up -> down overlap for the regular grouped GEMMs too -- full GPU suite, then A/B
O=gpurun_out/r2_t53; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > $O/pytest_all.log 2>&1; echo "all gpu tests rc=$?"; tail -3 $O/pytest_all.log
for ov in 1 0 1 0; do XPGB_FUSED_OVERLAP=$ov timeout 300 python tools/resident_time.py >> $O/resident.jsonl 2>> $O/rt.err; done; cat $O/resident.jsonl; tail -2 $O/rt.err
for ov in 1 0; do XPGB_FUSED_OVERLAP=$ov timeout 300 python tools/resident_time.py --config qwen3 >> $O/resident_q.jsonl 2>> $O/rt.err; done; cat $O/resident_q.jsonl
for ov in 1 0; do
  for b in 0.25 0.9; do
  XPGB_FUSED_OVERLAP=$ov timeout 900 python bench.py --budget $b --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}_$ov.json 2> $O/b.err
  python -c "
import json; d=json.loads(open('$O/b${b}_$ov.json').read().strip().splitlines()[-1]); g=d['roofline'].get('gemm') or {}
print('overlap=$ov $b', round(d['value']), round(d['ms_per_step'],3), 'resident', round(d['resident']['tok_s']), round(d['resident']['ms_per_step'],3), 'gu frac', round(g.get('frac',0),3))" 2>/dev/null || tail -3 $O/b.err
  done
done
