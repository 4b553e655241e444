#!/bin/bash
# round 2: FX4 fused stage-count A/B (2 decoded + 4 compressed vs 3 decoded + 2 compressed)
O=gpurun_out/r2_t34; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 600 python tools/debug_fused.py > $O/debug.jsonl 2> $O/debug.err; echo "rc=$?"; cut -c1-100 $O/debug.jsonl | head -4
XPGB_FX_STAGES=3 timeout 600 python tools/debug_fused.py > $O/debug3.jsonl 2>> $O/debug.err; cut -c1-100 $O/debug3.jsonl | head -4
for st in 2 3 2 3; do XPGB_FX_STAGES=$st timeout 900 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --device-format fx4 --modes 1 > $O/fx_st$st.jsonl 2>> $O/err.log; echo "st=$st"; cut -c1-200 $O/fx_st$st.jsonl; done
for st in 2 3; do XPGB_FX_STAGES=$st timeout 900 python tools/profile_fused.py --config qwen3 --layers 2 --tokens 256 --device-format fx4 --modes 1 > $O/fxq_st$st.jsonl 2>> $O/err.log; echo "qwen3 st=$st"; cut -c1-200 $O/fxq_st$st.jsonl; done
