#!/bin/bash
O=gpurun_out/t88; mkdir -p $O
for r in 1 2; do for bd in 1100 1500 2000; do
  echo -n "b_dec=$bd "; timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.65,0.8,0.9 --b-dec $bd 2>/dev/null | python -c "
import json,sys
print(' '.join(str(round(json.loads(l)['tok_s'])) for l in sys.stdin))"
done; done | tee $O/ab.txt
