#!/bin/bash
O=gpurun_out/r2_t24; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 600 python tools/debug_fused.py > $O/debug.jsonl 2> $O/debug.err; echo "rc=$?"; cat $O/debug.jsonl; tail -3 $O/debug.err
T=64 timeout 600 python tools/debug_fused.py > $O/debug64.jsonl 2>> $O/debug.err; cat $O/debug64.jsonl
