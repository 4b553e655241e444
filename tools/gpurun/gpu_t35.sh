#!/bin/bash
O=gpurun_out/t35; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_codec.py tests/test_gpu_residency.py -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head -8
for nb in 2 4 8; do
  XPGB_STAGE_BUFS=$nb timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.25,0.5,0.65,0.8 > $O/sweep_nb$nb.jsonl 2> $O/sweep_nb$nb.err; echo "nb=$nb rc=$?"
  python - $nb <<'PY'
import json,sys
for l in open(f"gpurun_out/t35/sweep_nb{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1), round(d['hbm_footprint'],3))
PY
done
