#!/bin/bash
# round 2: what bounds the FX4 decode-into-GEMM kernel? decode math off (timing only) / token-tile width
O=gpurun_out/r2_t47; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
run() { env "$@" timeout 600 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --steps 5 --modes 1 --device-format fx4 2> $O/pf.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); k=d.get('kernels',{})
    print('$*', round(d['ms_per_step'],3), 'gu_us', round(k.get('gate_up_ns',0)/1e3,1), 'dn_us', round(k.get('down_ns',0)/1e3,1))"; }
run X=0
run XPGB_FX_NODEC=1
run XPGB_BN_DEC=80
run XPGB_BN_DEC=128
run XPGB_BN_DEC=64
run XPGB_BN_DEC=48
run XPGB_FX_NODEC=1 XPGB_BN_DEC=48
run X=0
