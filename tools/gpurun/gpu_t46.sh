#!/bin/bash
O=gpurun_out/t46; mkdir -p $O
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode -s 1 -c 1 -o $O/dec_v5 python tools/profile_codec.py --chunk 256 --reps 1 > $O/ncu.log 2>&1
tail -3 $O/ncu.log; ls $O
