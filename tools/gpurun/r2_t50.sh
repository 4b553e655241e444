#!/bin/bash
# round 2: FX4 TMEM decoder with 4-op value pairs -- parity, then timing
O=gpurun_out/r2_t50; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
run() { env "$@" timeout 600 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --steps 5 --modes 1 --device-format fx4 2> $O/pf.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); k=d.get('kernels',{})
    print('$*', round(d['ms_per_step'],3), 'gu_us', round(k.get('gate_up_ns',0)/1e3,1), 'dn_us', round(k.get('down_ns',0)/1e3,1))"; tail -2 $O/pf.err; }
run X=1
run XPGB_FX_NODEC=1
run X=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm_dec -s 2 -c 2 -o $O/fused_fx4_tmem python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --steps 1 --modes 1 --device-format fx4 > $O/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
