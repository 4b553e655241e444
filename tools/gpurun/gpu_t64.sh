#!/bin/bash
O=gpurun_out/t64; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -1 $O/pytest.log; grep -E "FAILED" $O/pytest.log | head -8
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; cut -c1-300 $O/bench_ref.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > $O/bench_torchrun.json 2> $O/bench_torchrun.err; echo "torchrun rc=$?"; cut -c1-200 $O/bench_torchrun.json
