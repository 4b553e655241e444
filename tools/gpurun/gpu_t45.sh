#!/bin/bash
O=gpurun_out/t45; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_codec.py -q -x > $O/pytest.log 2>&1; tail -1 $O/pytest.log; grep -E "^E |FAILED" $O/pytest.log | head -5
for ch in 256 128 512; do echo -n "chunk=$ch "; timeout 120 python tools/profile_codec.py --chunk $ch --reps 30 2>&1 | tail -1 | cut -c1-120; done | tee $O/dec.txt
echo -n "small chunk=256 "; timeout 120 python tools/profile_codec.py --values 14680064 --chunk 256 --reps 30 2>&1 | tail -1 | cut -c1-120
