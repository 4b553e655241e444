#!/bin/bash
O=gpurun_out/t21; mkdir -p $O
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm -s 2 -c 2 -o $O/gemm_T256 python tools/profile_layer.py --config mixtral --tokens 256 --reps 1 > $O/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode -s 1 -c 1 -o $O/exp_decode python tools/profile_codec.py --reps 1 > $O/ncu_dec.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_moe_gemm_pair -s 2 -c 2 -o $O/pair_T32768 python tools/profile_layer.py --config mixtral --tokens 32768 --reps 1 > $O/ncu_pair.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
ls -la $O
