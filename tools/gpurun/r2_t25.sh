#!/bin/bash
O=gpurun_out/r2_t25; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 600 python tools/debug_fused.py > $O/debug.jsonl 2> $O/debug.err; echo "rc=$?"; cut -c1-150 $O/debug.jsonl | head -4; tail -3 $O/debug.err
timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py -q > $O/pytest_fx4.log 2>&1; echo "fx4+fused tests rc=$?"; tail -3 $O/pytest_fx4.log
timeout 900 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --device-format fx4 --modes 1 > $O/fused_fx4.jsonl 2> $O/fused_fx4.err; cut -c1-330 $O/fused_fx4.jsonl
