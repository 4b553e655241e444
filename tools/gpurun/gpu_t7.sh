#!/bin/bash
O=gpurun_out/t7; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_residency.py -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 900 python bench.py --prefill --tokens 32768 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_prefill32k.json 2> $O/bench_prefill32k.err; tail -2 $O/bench_prefill32k.err
timeout 900 python bench.py --prefill --tokens 32768 --steps 3 --warmup 3 --no-cpu-baseline --raw > $O/bench_prefill32k_raw.json 2> $O/bench_prefill32k_raw.err
python -c "
import json
for f in ['bench_prefill32k','bench_prefill32k_raw']:
    d=json.load(open('$O/'+f+'.json')); print(f, d['value'], d['resident'], d['paged_over_resident'], d['page_in']['achieved_gbps'], d['exposed_xfer_pct'], d['roofline']['bound'], d['roofline']['frac'])
"
