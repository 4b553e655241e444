#!/bin/bash
# round 2: tile-staged decoder v7 (bulk-copied stream, coalesced merge): exactness + A/B
O=gpurun_out/r2_t14; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
XPGB_DECODER=7 timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_fused.py -q -x > $O/pytest_codec7.log 2>&1; echo "codec tests (v7) rc=$?"; tail -3 $O/pytest_codec7.log
for d in 2 7 2 7; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 117440512 --chunk 256 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
for d in 2 7; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 14680064 --chunk 128 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
for d in 2 7; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 3145728 --chunk 128 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
python -c "
for l in open('$O/decoder_ab.jsonl'): print(l.strip()[:220])"; tail -3 $O/decoder_ab.err
XPGB_DECODER=7 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode7 -s 3 -c 1 -o $O/dec7 python tools/profile_codec.py --values 117440512 --chunk 256 --reps 5 > $O/ncu7.log 2>&1; echo "ncu7 rc=$?"
for d in 2 7; do XPGB_DECODER=$d timeout 900 python tools/sweep.py budget --config mixtral --budgets 0.25,0.8,0.9 > $O/sweep_dec$d.jsonl 2> $O/sweep_dec$d.err; echo "sweep dec=$d"; cut -c1-300 $O/sweep_dec$d.jsonl; done
XPGB_DECODER=7 timeout 900 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --modes 0 > $O/fused_mixtral_dec7.jsonl 2> $O/fused.err; cut -c1-300 $O/fused_mixtral_dec7.jsonl
