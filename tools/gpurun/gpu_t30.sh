#!/bin/bash
O=gpurun_out/t30; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k expert_parallel > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 600 python bench.py --ep --steps 3 --warmup 3 > $O/bench_ep.json 2> $O/bench_ep.err; echo "ep rc=$?"
python -c "import json; d=json.load(open('$O/bench_ep.json')); print(d['value'], d['page_in'], d['e2e'])"
