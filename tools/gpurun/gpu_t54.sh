#!/bin/bash
O=gpurun_out/t54; mkdir -p $O
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode2 -s 1 -c 1 -o $O/dec_v2 python tools/profile_codec.py --chunk 256 --reps 1 > $O/ncu.log 2>&1
XPGB_DEC_V1=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode -s 1 -c 1 -o $O/dec_v1 python tools/profile_codec.py --chunk 256 --reps 1 > $O/ncu1.log 2>&1
ls $O
