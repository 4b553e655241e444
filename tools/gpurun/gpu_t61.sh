#!/bin/bash
O=gpurun_out/t61; mkdir -p $O
timeout 600 python bench.py --config mixtral --ep --steps 3 > $O/bench_ep.json 2> $O/bench_ep.err; echo "bench ep rc=$?"; tail -3 $O/bench_ep.err
python -c "
import json; d=json.load(open('$O/bench_ep.json')); print(round(d['value'],1), round(d['e2e']['value'],1), d['config'].get('parallelism'))"
timeout 600 python bench.py --config dsv3 --ep --steps 3 > $O/bench_ep_dsv3.json 2> $O/bench_ep_dsv3.err; echo "bench ep dsv3 rc=$?"; tail -3 $O/bench_ep_dsv3.err
python -c "
import json; d=json.load(open('$O/bench_ep_dsv3.json')); print(round(d['value'],1), round(d['e2e']['value'],1), d['config'].get('parallelism'))"
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log; grep -E "FAILED" $O/pytest.log | head -8
