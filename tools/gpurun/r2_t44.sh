#!/bin/bash
# round 2: programmatic dependent launch for the grouped GEMMs -> GPU suite, then PDL on/off A/B
O=gpurun_out/r2_t44; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_all.log 2>&1; echo "all gpu tests rc=$?"; tail -3 $O/pytest_all.log
for pdl in 1 0; do
  XPGB_PDL=$pdl timeout 900 python bench.py --budget 0.25 --steps 10 --warmup 3 --no-cpu-baseline > $O/b25_$pdl.json 2> $O/b.err
  python -c "
import json; d=json.loads(open('$O/b25_$pdl.json').read().strip().splitlines()[-1]); g=d['roofline'].get('gemm') or {}
print('pdl=$pdl 0.25', round(d['value']), 'resident', round(d['resident']['tok_s']), round(d['resident']['ms_per_step'],3), 'gu', round(g.get('frac',0),3), round(g.get('avg_launch_us',0),1), 'dn', round(g.get('down',{}).get('frac',0),3), round(g.get('down',{}).get('avg_launch_us',0),1))" 2>/dev/null || tail -3 $O/b.err
  for b in 0.8 0.75; do
  XPGB_PDL=$pdl timeout 900 python bench.py --budget $b --steps 10 --warmup 3 --no-cpu-baseline --no-resident > $O/b${b}_$pdl.json 2> $O/b.err
  python -c "
import json; d=json.loads(open('$O/b${b}_$pdl.json').read().strip().splitlines()[-1])
print('pdl=$pdl $b', round(d['value']), d['config']['device_tier_format'], round(d['ms_per_step'],3))" 2>/dev/null || tail -3 $O/b.err
  done
done
