#!/bin/bash
# round 2: decode-into-GEMM correctness + first A/B (fused vs decode-into-ring)
O=gpurun_out/r2_t08; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x > $O/pytest_fused.log 2>&1; echo "fused tests rc=$?"; tail -15 $O/pytest_fused.log
timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > $O/pytest_rest.log 2>&1; echo "codec/parity tests rc=$?"; tail -5 $O/pytest_rest.log
for d in 2 3 2 3; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 117440512 --chunk 256 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
cat $O/decoder_ab.jsonl
for f in 1 0; do XPGB_FUSED=$f timeout 900 python tools/sweep.py budget --config mixtral --budgets 0.5,0.8,0.9 > $O/sweep_fused$f.jsonl 2> $O/sweep_fused$f.err; echo "sweep fused=$f rc=$?"; cat $O/sweep_fused$f.jsonl | cut -c1-400; done
XPGB_FUSED=1 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_fused.json 2> $O/bench_fused.err; echo "bench rc=$?"; head -c 600 $O/bench_fused.json; tail -3 $O/bench_fused.err
