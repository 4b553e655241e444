#!/bin/bash
# round 2: hand-off timeline of the FX4 decode-into-GEMM kernel (trace build)
O=gpurun_out/r2_t65; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
XPGB_LIB_PATH=tools/micro/ab/trace/libxpgb.so timeout 600 python tools/fx_trace.py > $O/trace.txt 2> $O/trace.err; echo "trace rc=$?"; cat $O/trace.txt; tail -3 $O/trace.err
