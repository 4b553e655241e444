#!/bin/bash
# round 2: full-shape float parity vs the oracle (Mixtral / Qwen3 / DSv3 rank slice)
O=gpurun_out/r2_t01; mkdir -p $O
nproc > $O/nproc.txt; free -g >> $O/nproc.txt
export XPGB_PARITY_LOG=$O/parity.jsonl
for f in qwen3 mixtral dsv3; do
  timeout 1500 python -m pytest tests/test_gpu_fullshape_$f.py -q -x -m gpu --durations=5 > $O/pytest_$f.log 2>&1; echo "$f rc=$?"
  tail -3 $O/pytest_$f.log
done
