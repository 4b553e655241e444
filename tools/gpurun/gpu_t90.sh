#!/bin/bash
O=gpurun_out/t90; mkdir -p $O
XPGB_LIB_PATH=tools/micro/ab/b12/libxpgb.so timeout 300 python -m pytest tests/test_gpu_codec.py -q -x > $O/pt.log 2>&1; tail -1 $O/pt.log
for r in 1 2; do for v in cur b12; do
  if [ $v = cur ]; then unset XPGB_LIB_PATH; else export XPGB_LIB_PATH=tools/micro/ab/$v/libxpgb.so; fi
  for n in 117440512 14680064; do echo -n "$v n=$n "; timeout 120 python tools/profile_codec.py --values $n --chunk 256 --reps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['out_GBps'],1), d['exact'])"; done
  echo -n "$v sweep "; timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.65,0.8 2>/dev/null | python -c "
import json,sys
print(' '.join(str(round(json.loads(l)['tok_s'])) for l in sys.stdin))"
done; done | tee $O/ab.txt
