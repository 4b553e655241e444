#!/bin/bash
O=gpurun_out/t69; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_codec.py -q -x > gpurun_out/t69/pt.log 2>&1; tail -1 gpurun_out/t69/pt.log
for r in 1 2 3; do echo -n "chunk=256 "; timeout 120 python tools/profile_codec.py --chunk 256 --reps 30 2>&1 | tail -1 | cut -c1-110; done | tee $O/dec.txt
echo -n "small "; timeout 120 python tools/profile_codec.py --values 14680064 --chunk 256 --reps 30 2>&1 | tail -1 | cut -c1-110
