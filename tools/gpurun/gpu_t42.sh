#!/bin/bash
O=gpurun_out/t42; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_codec.py -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log
for ch in 1024 512 256 128; do for bps in 5 8 16 64; do echo -n "chunk=$ch bps=$bps "; XPGB_DEC_BPS=$bps timeout 120 python tools/profile_codec.py --chunk $ch --reps 30 2>&1 | tail -1 | cut -c1-120; done; done | tee $O/dec.txt
for ch in 1024 256; do echo -n "small chunk=$ch "; timeout 120 python tools/profile_codec.py --values 14680064 --chunk $ch --reps 30 2>&1 | tail -1 | cut -c1-120; done | tee -a $O/dec.txt
