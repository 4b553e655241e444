#!/bin/bash
O=gpurun_out/t62; mkdir -p $O
timeout 600 python bench.py --config mixtral --ep --steps 3 > $O/bench_ep.json 2> $O/bench_ep.err; echo "bench ep rc=$?"; tail -2 $O/bench_ep.err
python -c "
import json; d=json.load(open('$O/bench_ep.json')); print(round(d['value'],1), round(d['e2e']['value'],1), d['config'].get('parallelism')); r=d['roofline']; print(r.get('kernel'), r.get('achieved'), r.get('frac'))"
timeout 600 python bench.py --config mixtral --ep --transport nccl --steps 3 > $O/bench_ep_nccl.json 2> $O/bench_ep_nccl.err; echo "bench ep nccl rc=$?"
python -c "
import json; d=json.load(open('$O/bench_ep_nccl.json')); print(round(d['value'],1), round(d['e2e']['value'],1), d['config'].get('parallelism'))"
