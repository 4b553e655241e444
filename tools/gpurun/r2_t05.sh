#!/bin/bash
# round 2: ncu full capture of decoder v2 and v1 (one 117M-value Mixtral gate/up tensor each)
O=gpurun_out/r2_t05; mkdir -p $O
XPGB_DECODER=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode2 -s 3 -c 1 -o $O/dec2 python tools/profile_codec.py --values 117440512 --chunk 256 --reps 5 > $O/ncu2.log 2>&1; echo "ncu2 rc=$?"
XPGB_DECODER=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode -s 3 -c 1 -o $O/dec1 python tools/profile_codec.py --values 117440512 --chunk 256 --reps 5 > $O/ncu1.log 2>&1; echo "ncu1 rc=$?"
ls -la $O
