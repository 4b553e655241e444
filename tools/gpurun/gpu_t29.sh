#!/bin/bash
O=gpurun_out/t29; mkdir -p $O
timeout 600 python bench.py --ep --steps 2 --warmup 3 > $O/bench_ep.json 2> $O/bench_ep.err; echo "ep rc=$?"; tail -3 $O/bench_ep.err
cut -c1-700 $O/bench_ep.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_torchrun.json 2> $O/bench_torchrun.err; echo "torchrun rc=$?"; tail -2 $O/bench_torchrun.err
cut -c1-300 $O/bench_torchrun.json
timeout 600 python bench.py --impl reference --steps 1 --warmup 1 --config dsv3 > $O/ref_dsv3.json 2> $O/ref_dsv3.err; echo "ref dsv3 rc=$?"; cut -c1-300 $O/ref_dsv3.json; tail -2 $O/ref_dsv3.err
