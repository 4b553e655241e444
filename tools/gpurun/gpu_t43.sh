#!/bin/bash
O=gpurun_out/t43; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head -8
echo -n "dec "; timeout 120 python tools/profile_codec.py --reps 30 2>&1 | tail -1 | cut -c1-140
timeout 600 python bench.py --config mixtral --steps 5 > $O/bench_mixtral.json 2> $O/bench_mixtral.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('$O/bench_mixtral.json')); print(round(d['value'],1), round(d['e2e']['value'],1), d['roofline'])"
run() {
  timeout 900 python tools/sweep.py budget --config mixtral --steps 3 --budgets 0.25,0.5,0.65,0.8,0.9 "${@:2}" > $O/sweep_$1.jsonl 2> $O/sweep_$1.err; echo "$1 rc=$?"
  python - $1 <<'PY'
import json,sys
for l in open(f"gpurun_out/t43/sweep_{sys.argv[1]}.jsonl"):
    d=json.loads(l); print(d['budget'], d['ring_experts'], d['ring_depth'], d['pinned_per_layer'], d['device_tier_per_layer'], round(d['tok_s']), round(d['ms_per_step'],1), round(d['page_in_gbps'],1), round(d['hbm_footprint'],3))
PY
}
run d2
run d3w1s4 --depth 3 --window 1 --stage-bufs 4
run d4w1s4 --depth 4 --window 1 --stage-bufs 4
