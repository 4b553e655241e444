#!/bin/bash
# round 2: decoder v2 correctness + standalone A/B, then the default bench
O=gpurun_out/r2_t04; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_codec.py tests/test_gpu_parity.py -q -x -m gpu > $O/pytest_codec.log 2>&1; echo "codec tests rc=$?"; tail -3 $O/pytest_codec.log
for d in 1 2 1 2; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 117440512 --chunk 256 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
for d in 1 2; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 14680064 --chunk 128 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
cat $O/decoder_ab.jsonl
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 3000 $O/bench.json; tail -5 $O/bench.err
