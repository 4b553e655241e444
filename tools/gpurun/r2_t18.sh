#!/bin/bash
# round 2: fused GEMM, sign/mantissa without register rotation
O=gpurun_out/r2_t18; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > $O/pytest_fused.log 2>&1; echo "fused tests rc=$?"; tail -2 $O/pytest_fused.log
timeout 900 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --modes 1 > $O/fused_mixtral.jsonl 2> $O/fused.err; echo "profile_fused rc=$?"; cut -c1-330 $O/fused_mixtral.jsonl; tail -3 $O/fused.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm_dec -s 2 -c 1 -o $O/fused python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --steps 1 --modes 1 > $O/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
