#!/bin/bash
O=gpurun_out/t9; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 300 python tools/profile_codec.py > $O/codec.json 2> $O/codec.err; cat $O/codec.json
timeout 300 python tools/profile_codec.py --values 3145728 > $O/codec_small.json 2>> $O/codec.err; cat $O/codec_small.json
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -1 $O/bench.err
timeout 900 python bench.py --prefill --tokens 32768 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_prefill32k.json 2> $O/bench_prefill32k.err; echo "prefill rc=$?"
python -c "
import json
for f in ['bench','bench_prefill32k']:
    d=json.load(open('$O/'+f+'.json')); print(f, d['value'], d['e2e']['value'], d['resident'], d['paged_over_resident'], d['page_in']['achieved_gbps'], d['exposed_xfer_pct'], d['roofline']['bound'], d['roofline']['frac'], d['roofline']['down']['frac'])
"
