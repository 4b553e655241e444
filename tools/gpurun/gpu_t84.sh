#!/bin/bash
O=gpurun_out/t84; mkdir -p $O
XPGB_LIB_PATH=tools/micro/ab/sym4/libxpgb.so timeout 300 python -m pytest tests/test_gpu_codec.py -q -x > $O/pt.log 2>&1; tail -1 $O/pt.log
for r in 1 2 3; do for v in cur sym4; do
  if [ $v = cur ]; then unset XPGB_LIB_PATH; else export XPGB_LIB_PATH=tools/micro/ab/$v/libxpgb.so; fi
  for n in 117440512 14680064; do for ch in 256 128; do echo -n "$v n=$n ch=$ch "; timeout 120 python tools/profile_codec.py --values $n --chunk $ch --reps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['out_GBps'],1), d['exact'])"; done; done
done; done | tee $O/ab.txt
