#!/bin/bash
O=gpurun_out/t74; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_codec.py tests/test_gpu_residency.py -q -x > $O/pt.log 2>&1; tail -1 $O/pt.log; grep -E "^E " $O/pt.log | head
for n in 1024 3145728 14680064 117440512; do for ch in 128 256; do echo -n "n=$n chunk=$ch "; timeout 120 python tools/profile_codec.py --values $n --chunk $ch --reps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms']*1000,1),'us', round(d['out_GBps'],1),'GB/s', d['exact'])"; done; done | tee $O/dec.txt
