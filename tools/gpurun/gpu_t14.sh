#!/bin/bash
O=gpurun_out/t14; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 300 python tools/profile_layer.py --config qwen3 --sweep 256,1024,2048 > $O/layer_qwen3.jsonl 2>/dev/null
timeout 300 python tools/profile_layer.py --config mixtral --sweep 256,512 > $O/layer_mixtral.jsonl 2>/dev/null
timeout 900 python bench.py --config dsv3 --steps 3 --warmup 3 > $O/bench_dsv3.json 2> $O/bench_dsv3.err; echo "dsv3 rc=$?"
timeout 900 python bench.py --prefill --tokens 65536 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_prefill64k.json 2> $O/bench_prefill64k.err; echo "prefill64k rc=$?"
python - <<'PY'
import json
for f in ("qwen3","mixtral"):
    for l in open(f"gpurun_out/t14/layer_{f}.jsonl"):
        d=json.loads(l); print(f, d["T"], "gu_us", round(d["gate_up_ns"]/1e3,1), "dn_us", round(d["down_ns"]/1e3,1))
for f in ("bench_dsv3","bench_prefill64k"):
    d=json.load(open(f"gpurun_out/t14/{f}.json")); print(f, d['value'], d['e2e']['value'], d['resident'], d['paged_over_resident'], d['page_in']['achieved_gbps'], d['exposed_xfer_pct'], d['roofline']['bound'], d['roofline']['frac'], d['roofline']['down']['frac'])
PY
