#!/bin/bash
O=gpurun_out/t81; mkdir -p $O
XPGB_LIB_PATH=tools/micro/ab/group/libxpgb.so timeout 300 python -m pytest tests/test_gpu_codec.py -q -x 2>&1 | tail -1
for r in 1 2 3; do for v in cur group; do
  if [ $v = cur ]; then unset XPGB_LIB_PATH; else export XPGB_LIB_PATH=tools/micro/ab/$v/libxpgb.so; fi
  for n in 117440512 14680064; do echo -n "$v n=$n "; timeout 120 python tools/profile_codec.py --values $n --chunk 256 --reps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['out_GBps'],1), d['exact'])"; done
done; done | tee $O/ab.txt
