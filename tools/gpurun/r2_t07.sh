#!/bin/bash
# round 2: decoder v1/v2 standalone A/B + ncu of decoder v2 and the resident decode GEMMs (split activations)
O=gpurun_out/r2_t07; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for d in 1 2 1 2; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 117440512 --chunk 256 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
for d in 1 2; do XPGB_DECODER=$d timeout 300 python tools/profile_codec.py --values 14680064 --chunk 128 >> $O/decoder_ab.jsonl 2>>$O/decoder_ab.err; done
cat $O/decoder_ab.jsonl
timeout 300 python tools/profile_layer.py --config mixtral --sweep 1,16,64,256 > $O/layer_mixtral.jsonl 2>$O/layer.err; cat $O/layer_mixtral.jsonl
XPGB_DECODER=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exp_decode2 -s 3 -c 1 -o $O/dec2 python tools/profile_codec.py --values 117440512 --chunk 256 --reps 5 > $O/ncu_dec2.log 2>&1; echo "ncu dec2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm -s 2 -c 2 -o $O/gemm_T256 python tools/profile_layer.py --config mixtral --tokens 256 --reps 1 > $O/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-resident --no-cpu-baseline > $O/bench_under_ncu.log 2>&1; echo "ncu launches rc=$?"
ls -la $O
