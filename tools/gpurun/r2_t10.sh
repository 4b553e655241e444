#!/bin/bash
# round 2: full GPU suite (fused off by default), decoder stream-lookahead A/B, calibrate for the sim check
O=gpurun_out/r2_t10; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_all.log 2>&1; echo "all gpu tests rc=$?"; grep -E "passed|failed|FAILED" $O/pytest_all.log | tail -8
for d in 2 4 5 2 4 5; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 117440512 --chunk 256 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
python -c "
import json
for l in open('$O/decoder_ab.jsonl'): print(l.strip()[:160])"
for d in 4 5; do XPGB_DECODER=$d timeout 900 python tools/sweep.py budget --config mixtral --budgets 0.8 > $O/sweep_dec$d.jsonl 2> $O/sweep_dec$d.err; echo "sweep dec=$d"; cut -c1-330 $O/sweep_dec$d.jsonl; done
timeout 600 python -m paper_2604_02715_b200 calibrate --model 8,8,4096,14336 --tokens 256 --top-k 2 --out $O/calib_mixtral.json > $O/calib.log 2>&1; echo "calibrate rc=$?"; cat $O/calib_mixtral.json
