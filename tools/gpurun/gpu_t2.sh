#!/bin/bash
O=gpurun_out/t2; mkdir -p $O
free -g > $O/box.txt; nproc >> $O/box.txt; nvidia-smi topo -m >> $O/box.txt 2>&1; numactl -H >> $O/box.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 600 python tools/profile_layer.py --config qwen3 --sweep 1,16,64,256,1024,4096,16384 > $O/layer_qwen3.jsonl 2> $O/layer_qwen3.err
timeout 600 python tools/profile_layer.py --config dsv3 --sweep 1,256,4096 > $O/layer_dsv3.jsonl 2> $O/layer_dsv3.err
timeout 600 python tools/profile_layer.py --config mixtral --sweep 1,256,16384 > $O/layer_mixtral.jsonl 2> $O/layer_mixtral.err
python - <<'PY'
import json
for f in ("qwen3","dsv3","mixtral"):
    for l in open(f"gpurun_out/t2/layer_{f}.jsonl"):
        d=json.loads(l); print(f, d["T"], "plan_us", round(d["plan_ns"]/1e3,1), "gu_us", round(d["gate_up_ns"]/1e3,1), "dn_us", round(d["down_ns"]/1e3,1))
PY
