#!/bin/bash
# round 2: decode-into-GEMM (128 regs) + 256-row down units: correctness, A/B sweeps, bench
O=gpurun_out/r2_t09; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_hazards.py -q -x > $O/pytest_fused.log 2>&1; echo "fused tests rc=$?"; tail -15 $O/pytest_fused.log
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_all.log 2>&1; echo "all gpu tests rc=$?"; tail -5 $O/pytest_all.log
timeout 300 python tools/profile_layer.py --config mixtral --sweep 1,16,64,256 > $O/layer_mixtral.jsonl 2>$O/layer.err; cat $O/layer_mixtral.jsonl | cut -c1-300
for f in 1 0; do XPGB_FUSED=$f timeout 900 python tools/sweep.py budget --config mixtral --budgets 0.25,0.5,0.8,0.9 > $O/sweep_fused$f.jsonl 2> $O/sweep_fused$f.err; echo "sweep fused=$f rc=$?"; cut -c1-330 $O/sweep_fused$f.jsonl; tail -2 $O/sweep_fused$f.err; done
XPGB_FUSED=1 XPGB_FUSED_WIN=1 timeout 900 python tools/sweep.py budget --config mixtral --budgets 0.8 > $O/sweep_fused_word.jsonl 2> $O/sweep_fused_word.err; echo "sweep word rc=$?"; cut -c1-330 $O/sweep_fused_word.jsonl
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; head -c 600 $O/bench.json; tail -3 $O/bench.err
