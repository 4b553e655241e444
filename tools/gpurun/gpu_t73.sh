#!/bin/bash
O=gpurun_out/t73; mkdir -p $O
for n in 3145728 14680064 117440512; do for ch in 64 128 256; do echo -n "n=$n chunk=$ch "; timeout 120 python tools/profile_codec.py --values $n --chunk $ch --reps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms']*1000,1),'us', round(d['out_GBps'],1),'GB/s')"; done; done | tee $O/dec.txt
