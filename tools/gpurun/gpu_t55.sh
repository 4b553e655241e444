#!/bin/bash
O=gpurun_out/t55; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_codec.py tests/test_gpu_residency.py -q -x 2>&1 | tail -2
for r in 1 2 3; do for ch in 256 128; do echo -n "chunk=$ch "; timeout 120 python tools/profile_codec.py --chunk $ch --reps 30 2>&1 | tail -1 | cut -c1-110; done; done | tee $O/dec.txt
echo -n "small "; timeout 120 python tools/profile_codec.py --values 14680064 --chunk 256 --reps 30 2>&1 | tail -1 | cut -c1-110
