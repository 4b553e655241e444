#!/bin/bash
# round 2: FX4 slot release before the decode (fence on/off), correctness + speed
O=gpurun_out/r2_t36; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for f in 1 0; do XPGB_FX_FENCE=$f timeout 600 python tools/debug_fused.py > $O/debug_f$f.jsonl 2> $O/debug.err; echo "fence=$f"; cut -c1-100 $O/debug_f$f.jsonl | head -4; done
for f in 1 0 1 0; do XPGB_FX_FENCE=$f timeout 900 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --device-format fx4 --modes 1 > $O/fx_f$f.jsonl 2>> $O/err.log; echo "fence=$f"; cut -c1-180 $O/fx_f$f.jsonl; done
timeout 900 python -m pytest tests/test_gpu_fx4.py tests/test_gpu_fused.py -q > $O/pytest.log 2>&1; echo "tests rc=$?"; tail -1 $O/pytest.log
