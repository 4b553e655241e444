#!/bin/bash
# round 2: 16 decoder warps x single activation plane (the two near-equal limits together)
O=gpurun_out/r2_t70; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
XPGB_FX_WARPS=16 timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py -x -q > $O/pytest16.log 2>&1; echo "pytest16 rc=$?"; tail -2 $O/pytest16.log
run() { env "$@" timeout 600 python tools/profile_fused.py --config $C --layers 2 --tokens 256 --steps 5 --modes 1 --device-format fx4 $A 2> $O/pf.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); k=d.get('kernels',{})
    print('$C $* $A', round(d['ms_per_step'],3), 'gu_us', round(k.get('gate_up_ns',0)/1e3,1), 'dn_us', round(k.get('down_ns',0)/1e3,1))"; tail -2 $O/pf.err; }
for C in mixtral qwen3; do for w in 8 16; do for A in "--act-planes 2" "--act-planes 1"; do C=$C A="$A" run XPGB_FX_WARPS=$w; done; done; done
