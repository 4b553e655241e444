#!/bin/bash
O=gpurun_out/t86; mkdir -p $O
for r in 1 2; do for sb in 4 8; do
  echo -n "sb=$sb "; XPGB_STAGE_BUFS=$sb timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.5,0.65,0.8 2>/dev/null | python -c "
import json,sys
print(' '.join(str(round(json.loads(l)['tok_s'])) for l in sys.stdin))"
done; done | tee $O/ab.txt
