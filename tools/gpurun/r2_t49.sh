#!/bin/bash
# round 2: compressed-stage depth with the A tiles in TMEM (4 / 6 / up-to-8 stages)
O=gpurun_out/r2_t49; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
run() { env "$@" timeout 600 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --steps 5 --modes 1 --device-format fx4 2> $O/pf.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); k=d.get('kernels',{})
    print('$*', round(d['ms_per_step'],3), 'gu_us', round(k.get('gate_up_ns',0)/1e3,1), 'dn_us', round(k.get('down_ns',0)/1e3,1))"; tail -2 $O/pf.err; }
for r in 1 2; do
run X=cst6
run XPGB_LIB_PATH=tools/micro/ab/cst4/libxpgb.so
run XPGB_LIB_PATH=tools/micro/ab/cst8/libxpgb.so
done
