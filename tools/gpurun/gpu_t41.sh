#!/bin/bash
O=gpurun_out/t41; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_codec.py -q -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head -8
for ch in 1024 256; do echo -n "chunk=$ch "; timeout 120 python tools/profile_codec.py --chunk $ch --reps 30 2>&1 | tail -1; done | tee $O/dec.txt
echo -n "small "; timeout 120 python tools/profile_codec.py --values 14680064 --chunk 1024 --reps 30 2>&1 | tail -1
