#!/bin/bash
# round 2: mixed device tier at 75%: window layout (spread / grouped) x fused grid cap (SMs left to the decoder)
O=gpurun_out/r2_t41; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for b in 0.75 0.72; do for lay in spread grouped; do for cap in 0 120 96; do
  XPGB_MIXED_LAYOUT=$lay XPGB_FUSED_SMS=$cap timeout 600 python bench.py --budget $b --device-format mixed --steps 10 --warmup 3 --no-cpu-baseline --no-resident > $O/b_${b}_${lay}_$cap.json 2> $O/b.err
  python -c "
import json; d=json.loads(open('$O/b_${b}_${lay}_$cap.json').read().strip().splitlines()[-1]); c=d['config']
print($b, '$lay', $cap, round(d['value']), round(d['ms_per_step'],2), c['fx4_experts_per_layer'], round(d['exposed_xfer_pct'],1))" 2>/dev/null || tail -3 $O/b.err
done; done; done
