#!/bin/bash
O=gpurun_out/t19; mkdir -p $O
for c in mixtral qwen3 dsv3; do timeout 600 python bench.py --config $c --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --prefill --tokens 65536 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_prefill64k.json 2> $O/bench_prefill64k.err; echo "prefill rc=$?"
python - <<'PY'
import json
for f in ("mixtral","qwen3","dsv3","prefill64k"):
    d=json.load(open(f"gpurun_out/t19/bench_{f}.json")); print(f, round(d['value'],1), round(d['e2e']['value'],1), d['resident'], round(d['page_in']['frac'],3), round(d['exposed_xfer_pct'],1), d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['down']['frac'],3), d['config']['expert_hbm_budget'], d['config']['placement'][:60], d.get('paged_over_resident'))
PY
