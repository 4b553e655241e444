#!/bin/bash
# round 2: fused gate/up -> down overlap (PDL + per-group unit counters) -- parity x3, then A/B
O=gpurun_out/r2_t52; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for r in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py -x -q > $O/pytest_$r.log 2>&1; echo "pytest $r rc=$?"; tail -2 $O/pytest_$r.log; done
timeout 600 python -m pytest tests/test_gpu_hazards.py tests/test_gpu_budget*.py -x -q > $O/pytest_h.log 2>&1; echo "hazards rc=$?"; tail -2 $O/pytest_h.log
run() { env "$@" timeout 600 python tools/profile_fused.py --config $C --layers 4 --tokens 256 --steps 10 --modes 1,0 --device-format fx4 --no-profile 2> $O/pf.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'bit_identical' in d: print('$C $*', d); continue
    print('$C $*', 'fused', d['fused'], round(d['ms_per_step'],3))"; tail -2 $O/pf.err; }
for C in mixtral qwen3 dsv3; do
C=$C run XPGB_FUSED_OVERLAP=1
C=$C run XPGB_FUSED_OVERLAP=0
done
for ov in 1 0; do
  XPGB_FUSED_OVERLAP=$ov timeout 900 python bench.py --budget 0.8 --steps 10 --warmup 3 --no-cpu-baseline --no-resident > $O/b80_$ov.json 2> $O/b.err
  python -c "
import json; d=json.loads(open('$O/b80_$ov.json').read().strip().splitlines()[-1])
print('overlap=$ov 0.8', round(d['value']), round(d['ms_per_step'],3), d['config']['device_tier_format'])" 2>/dev/null || tail -3 $O/b.err
done
