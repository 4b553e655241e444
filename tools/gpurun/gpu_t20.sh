#!/bin/bash
O=gpurun_out/t20; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
for c in mixtral qwen3 dsv3; do timeout 600 python bench.py --config $c --steps 5 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --prefill --tokens 65536 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_prefill64k.json 2> $O/bench_prefill64k.err; echo "prefill rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "ref rc=$?"; cat $O/bench_reference.json | cut -c1-600
python - <<'PY'
import json
for f in ("mixtral","qwen3","dsv3","prefill64k"):
    d=json.load(open(f"gpurun_out/t20/bench_{f}.json")); print(f, round(d['value'],1), round(d['e2e']['value'],1), d['resident'], round(d['page_in']['frac'],3), round(d['exposed_xfer_pct'],1), d['roofline']['bound'], round(d['roofline']['frac'],3), round(d['roofline']['down']['frac'],3), d['config']['expert_hbm_budget'], d['config']['expert_hbm_footprint'], d['config']['placement'][:50], d.get('paged_over_resident'))
PY
