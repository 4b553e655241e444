#!/bin/bash
# round 2: single-launch slot-table updates for load-free windows, sampled profiling -> full gpu suite,
# then the mixed-tier layout / fused-grid A/B at 72% and 75%
O=gpurun_out/r2_t42; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_all.log 2>&1; echo "all gpu tests rc=$?"; tail -3 $O/pytest_all.log
for b in 0.75 0.72; do for lay in spread grouped; do for cap in 0 112; do
  XPGB_MIXED_LAYOUT=$lay XPGB_FUSED_SMS=$cap timeout 600 python bench.py --budget $b --device-format mixed --steps 10 --warmup 3 --no-cpu-baseline --no-resident > $O/b_${b}_${lay}_$cap.json 2> $O/b.err
  python -c "
import json; d=json.loads(open('$O/b_${b}_${lay}_$cap.json').read().strip().splitlines()[-1]); c=d['config']; r=d['roofline']
print($b, '$lay', $cap, round(d['value']), round(d['ms_per_step'],2), c['fx4_experts_per_layer'], round(d['exposed_xfer_pct'],1), d['gpu_launches'], r.get('kernel','')[:20], round(r['frac'],3))" 2>/dev/null || tail -3 $O/b.err
done; done; done
for b in 0.25 0.7 0.8; do
  timeout 600 python bench.py --budget $b --steps 10 --warmup 3 --no-cpu-baseline --no-resident > $O/b_$b.json 2> $O/b.err
  python -c "
import json; d=json.loads(open('$O/b_$b.json').read().strip().splitlines()[-1]); c=d['config']; r=d['roofline']
print($b, round(d['value']), round(d['ms_per_step'],2), c['device_tier_format'], round(d['exposed_xfer_pct'],1), d['gpu_launches'], r.get('kernel','')[:20], round(r['frac'],3), r.get('launches_per_step'))" 2>/dev/null || tail -3 $O/b.err
done
