#!/bin/bash
O=gpurun_out/t17; mkdir -p $O
timeout 600 ncu --set full --clock-control none -k regex:k_moe_gemm -s 2 -c 2 -o $O/gemm_T16 python tools/profile_layer.py --config mixtral --tokens 16 --reps 1 > $O/ncu16.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_moe_gemm -s 2 -c 2 -o $O/gemm_T256 python tools/profile_layer.py --config mixtral --tokens 256 --reps 1 > $O/ncu256.log 2>&1
for sb in 33554432 67108864; do XPGB_STAGE_BYTES=$sb timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-resident > $O/bench_mixtral_sb$sb.json 2>/dev/null; XPGB_STAGE_BYTES=$sb timeout 600 python bench.py --config dsv3 --steps 3 --no-cpu-baseline --no-resident > $O/bench_dsv3_sb$sb.json 2>/dev/null; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/t17/bench_*.json")):
    try:
        d=json.load(open(f)); print(f.split('/')[-1], round(d['value'],1), round(d['page_in']['achieved_gbps'],2), round(d['page_in']['frac'],3))
    except Exception as e: print(f, e)
PY
