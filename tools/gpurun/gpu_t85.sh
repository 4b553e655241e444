#!/bin/bash
O=gpurun_out/t85; mkdir -p $O
for r in 1 2; do for v in sym4 pre4; do
  if [ $v = sym4 ]; then unset XPGB_LIB_PATH; else export XPGB_LIB_PATH=tools/micro/ab/$v/libxpgb.so; fi
  echo -n "$v "; timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.65,0.8,0.9 2>/dev/null | python -c "
import json,sys
print(' '.join(str(round(json.loads(l)['tok_s'])) for l in sys.stdin))"
done; done | tee $O/ab.txt
