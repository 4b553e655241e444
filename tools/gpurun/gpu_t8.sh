#!/bin/bash
O=gpurun_out/t8; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; tail -2 $O/bench.err
timeout 900 python bench.py --prefill --tokens 32768 --steps 3 --warmup 3 > $O/bench_prefill32k.json 2> $O/bench_prefill32k.err
timeout 600 python tools/profile_layer.py --config mixtral --sweep 4096,16384,32768 > $O/layer_mixtral.jsonl 2> $O/layer.err
python -c "
import json
for f in ['bench','bench_prefill32k']:
    d=json.load(open('$O/'+f+'.json')); print(f, d['value'], d['e2e'], d['resident'], d['paged_over_resident'], d['page_in']['achieved_gbps'], d['exposed_xfer_pct'], d['roofline']['bound'], d['roofline']['frac'], d['roofline']['down'])
"
cut -c1-300 $O/layer_mixtral.jsonl
