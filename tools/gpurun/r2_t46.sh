#!/bin/bash
# round 2 final: validation of the committed tree -- GPU suite, smoke, bench + reference arm, launch
# list, ncu captures (decoder, fused FX4, decode GEMMs, prefill pair GEMMs), 2-rank bench
O=gpurun_out/r2_t46; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }



timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"; head -c 400 $O/bench_default.json; echo
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; head -c 400 $O/bench.json; echo
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; head -c 300 $O/bench_ref.json; echo
for b in 0.75 0.8; do timeout 900 python bench.py --budget $b --steps 10 --warmup 3 > $O/bench_$b.json 2> $O/bench_$b.err; echo "bench $b rc=$?"; head -c 300 $O/bench_$b.json; echo; done
timeout 900 python bench.py --gpus 2 --oversubscribe --steps 5 --warmup 3 > $O/bench_2ranks.json 2> $O/bench_2ranks.err; echo "2-rank rc=$?"; head -c 300 $O/bench_2ranks.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-resident --no-cpu-baseline > $O/bench_under_ncu.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/launches_bench80.csv python bench.py --budget 0.8 --steps 2 --warmup 1 --no-resident --no-cpu-baseline > $O/bench80_under_ncu.log 2>&1; echo "ncu launches 80 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode2 -s 3 -c 1 -o $O/dec2 python tools/profile_codec.py --values 117440512 --chunk 256 --reps 5 > $O/ncu_dec2.log 2>&1; echo "ncu dec2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm_dec -s 2 -c 2 -o $O/fused_fx4 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --steps 1 --modes 1 --device-format fx4 > $O/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm -s 2 -c 2 -o $O/gemm_T256 python tools/profile_layer.py --config mixtral --tokens 256 --reps 1 > $O/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm_pair -s 2 -c 2 -o $O/pair_T16384 python tools/profile_layer.py --config mixtral --tokens 16384 --reps 1 > $O/ncu_pair.log 2>&1; echo "ncu pair rc=$?"
