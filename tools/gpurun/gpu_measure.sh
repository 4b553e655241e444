#!/bin/bash
# Measurement batch: kernel sweeps (decode + prefill sizes), budget/token sweeps, codec decoder, ncu captures.
O=gpurun_out/m1; mkdir -p $O
timeout 600 python tools/profile_layer.py --config mixtral --sweep 1,16,64,256,1024,4096,8192,16384 > $O/layer_mixtral.jsonl 2> $O/layer_mixtral.err
timeout 600 python tools/profile_layer.py --config qwen3 --sweep 1,16,64,256,1024,4096,16384 > $O/layer_qwen3.jsonl 2> $O/layer_qwen3.err
timeout 600 python tools/profile_layer.py --config dsv3 --sweep 1,16,64,256,1024,4096 > $O/layer_dsv3.jsonl 2> $O/layer_dsv3.err
timeout 300 python tools/profile_codec.py > $O/codec.json 2> $O/codec.err
timeout 900 python tools/sweep.py budget --config mixtral > $O/sweep_budget_mixtral.jsonl 2> $O/sweep_budget.err
timeout 900 python tools/sweep.py tokens --config qwen3 --list 1,4,16,64,256 > $O/sweep_tokens_qwen3.jsonl 2> $O/sweep_tokens.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm -s 2 -c 2 -o $O/gemm_T256 python tools/profile_layer.py --config mixtral --tokens 256 --reps 1 > $O/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm -s 2 -c 2 -o $O/gemm_T8192 python tools/profile_layer.py --config mixtral --tokens 8192 --reps 1 > $O/ncu_gemm2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode -s 1 -c 1 -o $O/exp_decode python tools/profile_codec.py --reps 1 > $O/ncu_dec.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
ls -la $O
