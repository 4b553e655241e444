#!/bin/bash
# round 2: FX4 TMEM decoder with up to 4 decoded A stages (BN <= 80) -- parity, timing
O=gpurun_out/r2_t68; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py tests/test_gpu_hazards.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log; grep -E "^E " $O/pytest.log | head -3
run() { env "$@" timeout 600 python tools/profile_fused.py --config $C --layers 2 --tokens 256 --steps 5 --modes 1 --device-format fx4 2> $O/pf.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); k=d.get('kernels',{})
    print('$C $*', round(d['ms_per_step'],3), 'gu_us', round(k.get('gate_up_ns',0)/1e3,1), 'dn_us', round(k.get('down_ns',0)/1e3,1))"; tail -2 $O/pf.err; }
C=mixtral run XPGB_BN_DEC=96
C=mixtral run XPGB_BN_DEC=80
C=mixtral run XPGB_BN_DEC=64
C=qwen3 run X=1
C=dsv3 run X=1
