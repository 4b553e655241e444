#!/bin/bash
O=gpurun_out/t80; mkdir -p $O
PYTHONPATH=. timeout 300 python tools/micro/dbg_resident.py 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log; grep -E "FAILED" $O/pytest.log | head -8
timeout 600 python bench.py --config dsv3 --prefill --tokens 4096 --steps 2 2>/dev/null | cut -c1-200
timeout 600 python bench.py --config dsv3 --steps 5 > $O/bench_dsv3.json 2>/dev/null; python -c "
import json; d=json.load(open('$O/bench_dsv3.json')); print(round(d['value'],1), round(d['e2e']['value'],1), d['resident'])"
