#!/bin/bash
# round 2: fused FX4 with 16 decoder warps (half-rows), 8-column epilogue loads
O=gpurun_out/r2_t29; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 600 python tools/debug_fused.py > $O/debug.jsonl 2> $O/debug.err; echo "rc=$?"; cut -c1-120 $O/debug.jsonl | head -4
timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py -q > $O/pytest_fx4.log 2>&1; echo "fx4+fused tests rc=$?"; tail -2 $O/pytest_fx4.log
timeout 900 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --device-format fx4 --modes 1 > $O/fused_fx4.jsonl 2> $O/fused_fx4.err; cut -c1-330 $O/fused_fx4.jsonl
for cfg in qwen3 dsv3; do timeout 900 python tools/profile_fused.py --config $cfg --layers 2 --tokens 256 --device-format fx4 --modes 1 > $O/fused_fx4_$cfg.jsonl 2>> $O/fused_fx4.err; cut -c1-260 $O/fused_fx4_$cfg.jsonl; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm_dec -s 2 -c 2 -o $O/fused_fx4 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --steps 1 --modes 1 --device-format fx4 > $O/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
