#!/bin/bash
O=gpurun_out/t1; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -5 $O/pytest.log
timeout 600 python tools/profile_layer.py --config qwen3 --sweep 1,16,64,256,1024,4096,16384 > $O/layer_qwen3.jsonl 2> $O/layer_qwen3.err
timeout 600 python tools/profile_layer.py --config mixtral --sweep 256,4096,16384 > $O/layer_mixtral.jsonl 2> $O/layer_mixtral.err
timeout 900 python tools/sweep.py tokens --config qwen3 --list 1,16,256 > $O/sweep_tokens_qwen3.jsonl 2> $O/sweep_tokens.err
timeout 900 python tools/sweep.py tokens --config qwen3 --list 256 --raw > $O/sweep_tokens_qwen3_raw.jsonl 2>> $O/sweep_tokens.err
timeout 600 python bench.py --steps 5 > $O/bench.json 2> $O/bench.err
cat $O/*.jsonl $O/bench.json | cut -c1-400
