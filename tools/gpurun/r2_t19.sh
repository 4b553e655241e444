#!/bin/bash
# round 2: decoder occupancy A/B (v2 vs 6 / 8 CTAs per SM); fused GEMM with direct sign/mantissa loads
O=gpurun_out/r2_t19; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for d in 2 8 9 2 8 9; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 117440512 --chunk 256 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
for d in 2 8 9; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 14680064 --chunk 128 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
python -c "
import json
for l in open('$O/decoder_ab.jsonl'):
  d=json.loads(l); print(d['values'], d['chunk'], d.get('exact'), round(d['ms']*1e3,1), 'us', round(d['out_GBps']), round(d['algo_GBps']))"
XPGB_DECODER=9 timeout 600 python -m pytest tests/test_gpu_codec.py -q -x > $O/pytest_codec9.log 2>&1; echo "codec v9 rc=$?"; tail -1 $O/pytest_codec9.log
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > $O/pytest_fused.log 2>&1; echo "fused tests rc=$?"; tail -1 $O/pytest_fused.log
timeout 900 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 > $O/fused_mixtral.jsonl 2> $O/fused.err; echo "profile_fused rc=$?"; cut -c1-300 $O/fused_mixtral.jsonl
