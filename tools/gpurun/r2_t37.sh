#!/bin/bash
# round 2: prefill sanity with the new planner; Qwen3 at its full 48 layers
O=gpurun_out/r2_t37; mkdir -p $O
free -g > $O/free.txt; nproc >> $O/free.txt; cat $O/free.txt
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python bench.py --prefill --tokens 16384 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_prefill16k.json 2> $O/bench_prefill.err; echo "prefill rc=$?"; python -c "
import json; d=json.loads(open('$O/bench_prefill16k.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['value'], d['e2e']['value'], d['config']['device_tier_format'], d['config']['expert_hbm_footprint'], d.get('paged_over_resident'), d['exposed_xfer_pct'])"; tail -2 $O/bench_prefill.err
for b in 0.25 0.8; do timeout 1500 python bench.py --config qwen3 --layers 48 --budget $b --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_qwen3_48_$b.json 2> $O/bench_qwen3_48_$b.err; echo "qwen3-48 $b rc=$?"; python -c "
import json; d=json.loads(open('$O/bench_qwen3_48_$b.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['config']['workload'][:60], d['config']['device_tier_format'], d['config']['expert_hbm_footprint'], d.get('paged_over_resident'))"; tail -2 $O/bench_qwen3_48_$b.err; done
