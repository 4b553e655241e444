#!/bin/bash
O=gpurun_out/t40; mkdir -p $O
for ch in 1024 512 256; do for pf in 0 64 128 256; do
  echo -n "chunk=$ch pf=$pf "; XPGB_DEC_PF=$pf timeout 120 python tools/profile_codec.py --chunk $ch --reps 30 2>&1 | tail -1
done; done | tee $O/dec.txt
for pf in 0 128; do echo -n "small pf=$pf "; XPGB_DEC_PF=$pf timeout 120 python tools/profile_codec.py --values 4194304 --chunk 1024 --reps 30 2>&1 | tail -1; done | tee -a $O/dec.txt
