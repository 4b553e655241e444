#!/bin/bash
O=gpurun_out/t89; mkdir -p $O
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode -s 1 -c 1 -o $O/dec_v7 python tools/profile_codec.py --chunk 256 --reps 1 > $O/ncu.log 2>&1
ls $O
