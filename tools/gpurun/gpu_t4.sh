#!/bin/bash
O=gpurun_out/t4; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 900 python tools/live_planner.py --config mixtral --steps 30 > $O/live_mixtral_decode.jsonl 2> $O/live1.err; tail -3 $O/live1.err
timeout 900 python tools/live_planner.py --config mixtral --tokens 32768 --budget-experts 6 --steps 30 > $O/live_mixtral_prefill32k.jsonl 2> $O/live2.err; tail -3 $O/live2.err
timeout 900 python bench.py --prefill --tokens 16384 --steps 3 --warmup 3 > $O/bench_prefill16k.json 2> $O/bench_prefill.err; tail -2 $O/bench_prefill.err
timeout 900 python bench.py --config dsv3 --steps 3 --warmup 3 > $O/bench_dsv3.json 2> $O/bench_dsv3.err
cut -c1-300 $O/live_mixtral_decode.jsonl | tail -5; cut -c1-300 $O/live_mixtral_prefill32k.jsonl | tail -8; cut -c1-1200 $O/bench_prefill16k.json
