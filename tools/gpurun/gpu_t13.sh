#!/bin/bash
O=gpurun_out/t13; mkdir -p $O
for m in 0 1; do XPGB_PAIR_GEMM=$m timeout 300 python tools/profile_layer.py --config mixtral --sweep 256,512,1024,2048 > $O/mixtral_pair$m.jsonl 2>/dev/null; done
for m in 0 1; do XPGB_PAIR_GEMM=$m timeout 300 python tools/profile_layer.py --config qwen3 --sweep 1024,2048,4096 > $O/qwen3_pair$m.jsonl 2>/dev/null; done
for m in 0 1; do XPGB_PAIR_GEMM=$m timeout 300 python tools/profile_layer.py --config dsv3 --sweep 1024,2048,4096 > $O/dsv3_pair$m.jsonl 2>/dev/null; done
for bn in 64 128; do XPGB_BN=$bn timeout 300 python tools/profile_layer.py --config mixtral --sweep 128,256 > $O/mixtral_bn$bn.jsonl 2>/dev/null; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/t13/*.jsonl")):
    for l in open(f):
        d=json.loads(l); print(f.split('/')[-1], d["T"], "gu_us", round(d["gate_up_ns"]/1e3,1), "dn_us", round(d["down_ns"]/1e3,1), "GBps", round(d["gate_up_GBps"]), round(d["down_GBps"]))
PY
