#!/bin/bash
# round 2: FX4 decode-into-GEMM -- MMA/decoder handoffs spinning vs backing off (profile_fused, 2 layers)
O=gpurun_out/r2_t45; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for rep in 1 2; do for spin in 0 1; do
  XPGB_FX_SPIN=$spin timeout 600 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --steps 5 --modes 1 --device-format fx4 > $O/pf_${spin}_$rep.jsonl 2> $O/pf.err
  echo "spin=$spin rep=$rep"; tail -2 $O/pf_${spin}_$rep.jsonl | cut -c1-400
done; done
for spin in 0 1; do
  XPGB_FX_SPIN=$spin timeout 900 python bench.py --budget 0.8 --steps 10 --warmup 3 --no-cpu-baseline --no-resident > $O/b80_$spin.json 2> $O/b.err
  python -c "
import json; d=json.loads(open('$O/b80_$spin.json').read().strip().splitlines()[-1]); r=d['roofline']
print('spin=$spin 0.8', round(d['value']), round(d['ms_per_step'],3), r['kernel'][:16], round(r['frac'],3), round(r['avg_launch_us'],1))" 2>/dev/null || tail -3 $O/b.err
done
for pdl in 1 0 1 0; do XPGB_PDL=$pdl timeout 300 python tools/resident_time.py >> $O/resident_pdl.jsonl 2>> $O/rt.err; done; cat $O/resident_pdl.jsonl; tail -2 $O/rt.err
