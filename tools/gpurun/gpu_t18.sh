#!/bin/bash
O=gpurun_out/t18; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head
timeout 300 python tools/profile_layer.py --config mixtral --sweep 1,16,64,128,256 > $O/layer_mixtral.jsonl 2>/dev/null
timeout 300 python tools/profile_layer.py --config qwen3 --sweep 1,16,64,256,1024 > $O/layer_qwen3.jsonl 2>/dev/null
timeout 300 python tools/profile_layer.py --config dsv3 --sweep 256,2048 > $O/layer_dsv3.jsonl 2>/dev/null
python - <<'PY'
import json
for f in ("mixtral","qwen3","dsv3"):
    for l in open(f"gpurun_out/t18/layer_{f}.jsonl"):
        d=json.loads(l); print(f, d["T"], "gu_us", round(d["gate_up_ns"]/1e3,1), "dn_us", round(d["down_ns"]/1e3,1), "GBps", round(d["gate_up_GBps"]), round(d["down_GBps"]))
PY
for c in mixtral qwen3 dsv3; do timeout 600 python bench.py --config $c --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
python - <<'PY'
import json
for f in ("mixtral","qwen3","dsv3"):
    d=json.load(open(f"gpurun_out/t18/bench_{f}.json")); print(f, round(d['value'],1), round(d['e2e']['value'],1), d['resident'], round(d['page_in']['frac'],3), round(d['exposed_xfer_pct'],1), d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['down']['frac'],3), d['config']['expert_hbm_budget'])
PY
