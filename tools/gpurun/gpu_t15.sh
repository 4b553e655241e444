#!/bin/bash
O=gpurun_out/t15; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 900 python bench.py --config dsv3 --steps 3 --warmup 3 > $O/bench_dsv3.json 2> $O/bench_dsv3.err; echo "dsv3 rc=$?"; grep "bench " $O/bench_dsv3.err
timeout 900 python bench.py --prefill --tokens 65536 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_prefill64k.json 2> $O/bench_prefill64k.err; echo "prefill64k rc=$?"; grep "bench " $O/bench_prefill64k.err
timeout 600 python bench.py --steps 5 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
for f in ("bench","bench_dsv3","bench_prefill64k"):
    try:
        d=json.load(open(f"gpurun_out/t15/{f}.json")); print(f, d['value'], d['e2e']['value'], d['resident'], d['paged_over_resident'], d['page_in']['achieved_gbps'], d['exposed_xfer_pct'], d['roofline']['bound'], d['roofline']['frac'], d['roofline']['down']['frac'])
    except Exception as e: print(f, "ERR", e)
PY
