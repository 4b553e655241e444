#!/bin/bash
O=gpurun_out/t50; mkdir -p $O
for v in 0 1 2 3; do XPGB_DEC_VAR=$v timeout 300 python -m pytest tests/test_gpu_codec.py -q -x 2>&1 | tail -1; done
for v in 0 1 2 3 0; do echo -n "var=$v "; XPGB_DEC_VAR=$v timeout 120 python tools/profile_codec.py --chunk 256 --reps 30 2>&1 | tail -1 | cut -c1-110; done | tee $O/dec.txt
for v in 0 3; do echo -n "small var=$v "; XPGB_DEC_VAR=$v timeout 120 python tools/profile_codec.py --values 14680064 --chunk 256 --reps 30 2>&1 | tail -1 | cut -c1-110; done | tee -a $O/dec.txt
