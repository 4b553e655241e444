#!/bin/bash
O=gpurun_out/t3; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 900 python bench.py --config dsv3 --steps 3 --warmup 3 > $O/bench_dsv3.json 2> $O/bench_dsv3.err; tail -3 $O/bench_dsv3.err
timeout 600 python bench.py --config qwen3 --steps 5 > $O/bench_qwen3.json 2> $O/bench_qwen3.err; tail -2 $O/bench_qwen3.err
cat $O/bench_dsv3.json $O/bench_qwen3.json | cut -c1-1500
