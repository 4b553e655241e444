#!/bin/bash
# round 2: FX4 TMEM decoder, compressed reads pipelined one stage ahead of the TMEM stores -- parity x2, timing
O=gpurun_out/r2_t64; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for r in 1 2; do timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py tests/test_gpu_hazards.py -x -q > $O/pytest_$r.log 2>&1; echo "pytest $r rc=$?"; tail -2 $O/pytest_$r.log; done
run() { env "$@" timeout 600 python tools/profile_fused.py --config $C --layers 2 --tokens 256 --steps 5 --modes 1 --device-format fx4 2> $O/pf.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); k=d.get('kernels',{})
    print('$C $*', round(d['ms_per_step'],3), 'gu_us', round(k.get('gate_up_ns',0)/1e3,1), 'dn_us', round(k.get('down_ns',0)/1e3,1))"; tail -2 $O/pf.err; }
for C in mixtral qwen3 dsv3; do C=$C run X=1; done
C=mixtral run X=1
timeout 900 python bench.py --budget 0.8 --steps 10 --warmup 3 --no-cpu-baseline --no-resident > $O/b80.json 2> $O/b.err; python -c "
import json; d=json.loads(open('$O/b80.json').read().strip().splitlines()[-1]); r=d['roofline']
print('0.8', round(d['value']), round(d['ms_per_step'],3), round(r['frac'],3))" 2>/dev/null || tail -3 $O/b.err
