#!/bin/bash
# round 2: opt-in single activation plane for the decode-sized GEMMs -- tests, timing
O=gpurun_out/r2_t66; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
for b in 0.8 0.25; do for ap in 1 2; do
  timeout 900 python bench.py --budget $b --act-planes $ap --steps 10 --warmup 3 --no-cpu-baseline > $O/b${b}_$ap.json 2> $O/b.err
  python -c "
import json; d=json.loads(open('$O/b${b}_$ap.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$b planes=$ap', round(d['value']), 'e2e', round(d['e2e']['value']), 'resident', round(d['resident']['tok_s']), round(r['frac'],3))" 2>/dev/null || tail -3 $O/b.err
done; done
