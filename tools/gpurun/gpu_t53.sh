#!/bin/bash
O=gpurun_out/t53; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_codec.py tests/test_gpu_residency.py -q -x 2>&1 | tail -3
for v in 0 1 0; do for ch in 256 128; do echo -n "v1=$v chunk=$ch "; XPGB_DEC_V1=$v timeout 120 python tools/profile_codec.py --chunk $ch --reps 30 2>&1 | tail -1 | cut -c1-110; done; done | tee $O/dec.txt
for v in 0 1; do echo -n "small v1=$v "; XPGB_DEC_V1=$v timeout 120 python tools/profile_codec.py --values 14680064 --chunk 256 --reps 30 2>&1 | tail -1 | cut -c1-110; done | tee -a $O/dec.txt
