#!/bin/bash
# round 2: FX4 decode-into-GEMM with the decoded A tiles in TMEM (FMT 2) -- parity, then A/B
O=gpurun_out/r2_t48; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py tests/test_gpu_hazards.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest.log
run() { env "$@" timeout 600 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --steps 5 --modes 0,1 --device-format fx4 2> $O/pf.err | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if 'bit_identical' in d: print('$*', d); continue
    k=d.get('kernels',{})
    print('$*', 'fused', d['fused'], round(d['ms_per_step'],3), 'gu_us', round(k.get('gate_up_ns',0)/1e3,1), 'dn_us', round(k.get('down_ns',0)/1e3,1))"; tail -3 $O/pf.err; }
run XPGB_FX_TMEM=1
run XPGB_FX_TMEM=0
run XPGB_FX_TMEM=1
for cfg in qwen3 dsv3; do env timeout 600 python tools/profile_fused.py --config $cfg --layers 2 --tokens 256 --steps 5 --modes 1 --device-format fx4 2>/dev/null | cut -c1-200; XPGB_FX_TMEM=0 timeout 600 python tools/profile_fused.py --config $cfg --layers 2 --tokens 256 --steps 5 --modes 1 --device-format fx4 2>/dev/null | cut -c1-200; done
