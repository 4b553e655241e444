#!/bin/bash
O=gpurun_out/t28; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/bench.json')); print(d['value'], d['e2e'], d['page_in']['frac'], d['exposed_xfer_pct'], d['roofline']['frac'], d['roofline']['traffic'], d['gpu_launches'], d['clocks'], d['cpu_baseline']['value'])"
