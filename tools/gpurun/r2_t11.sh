#!/bin/bash
# round 2: fused GEMM with the smem-fed stream window; decoder v6 (contiguous runs + smem ring)
O=gpurun_out/r2_t11; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_hazards.py -q > $O/pytest_fused.log 2>&1; echo "fused tests rc=$?"; tail -4 $O/pytest_fused.log
XPGB_DECODER=6 timeout 900 python -m pytest tests/test_gpu_codec.py -q -x > $O/pytest_codec6.log 2>&1; echo "codec tests (v6) rc=$?"; tail -3 $O/pytest_codec6.log
for d in 2 6 2 6; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 117440512 --chunk 256 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
for d in 2 6; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 14680064 --chunk 128 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
python -c "
for l in open('$O/decoder_ab.jsonl'): print(l.strip()[:200])"
timeout 900 python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 > $O/fused_mixtral.jsonl 2> $O/fused.err; echo "profile_fused rc=$?"; cut -c1-300 $O/fused_mixtral.jsonl; tail -3 $O/fused.err
XPGB_FUSED=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm_dec -s 2 -c 2 -o $O/fused python tools/profile_fused.py --config mixtral --layers 2 --tokens 256 --steps 1 --modes 1 > $O/ncu_fused.log 2>&1; echo "ncu fused rc=$?"
for d in 2 6; do XPGB_DECODER=$d timeout 900 python tools/sweep.py budget --config mixtral --budgets 0.25,0.8 > $O/sweep_dec$d.jsonl 2> $O/sweep_dec$d.err; echo "sweep dec=$d"; cut -c1-330 $O/sweep_dec$d.jsonl; done
