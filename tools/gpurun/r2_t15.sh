#!/bin/bash
# round 2: decoder v7 with the next tile's stream prefetched and 4 merge loads in flight
O=gpurun_out/r2_t15; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
XPGB_DECODER=7 timeout 900 python -m pytest tests/test_gpu_codec.py -q -x > $O/pytest_codec7.log 2>&1; echo "codec tests (v7) rc=$?"; tail -2 $O/pytest_codec7.log
for d in 2 7 2 7; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 117440512 --chunk 256 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
for d in 2 7; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 14680064 --chunk 128 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
python -c "
import json
for l in open('$O/decoder_ab.jsonl'):
  d=json.loads(l); print(d['values'], d['chunk'], round(d['ms']*1e3,1), 'us', round(d['out_GBps']), round(d['algo_GBps']))"
XPGB_DECODER=7 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode7 -s 3 -c 1 -o $O/dec7 python tools/profile_codec.py --values 117440512 --chunk 256 --reps 5 > $O/ncu7.log 2>&1; echo "ncu7 rc=$?"
