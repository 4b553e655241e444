#!/bin/bash
O=gpurun_out/t12; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 600 python tools/profile_layer.py --config mixtral --sweep 1024,4096,16384,32768 > $O/layer_mixtral.jsonl 2> $O/layer.err
timeout 600 python tools/profile_layer.py --config qwen3 --sweep 4096,16384,32768 > $O/layer_qwen3.jsonl 2>> $O/layer.err
timeout 600 python tools/profile_layer.py --config dsv3 --sweep 4096,16384 > $O/layer_dsv3.jsonl 2>> $O/layer.err
python - <<'PY'
import json
for f in ("mixtral","qwen3","dsv3"):
    for l in open(f"gpurun_out/t12/layer_{f}.jsonl"):
        d=json.loads(l); T=d["T"]
        sh={"mixtral":(4096,14336,2),"qwen3":(2048,768,8),"dsv3":(7168,2048,8)}[f]
        H,F,k=sh
        rows=T*k if f!="dsv3" else T*8*32/256  # dsv3 profile shape is 32 experts of 256? (profile uses L=32)
        print(f, T, "gu_us", round(d["gate_up_ns"]/1e3,1), "dn_us", round(d["down_ns"]/1e3,1), "units", d["n_units_gate_up"], d["n_units_down"])
PY
timeout 900 python bench.py --prefill --tokens 32768 --steps 3 --warmup 3 --no-cpu-baseline > $O/bench_prefill32k.json 2> $O/bench_prefill32k.err; echo "prefill rc=$?"
python -c "
import json
d=json.load(open('$O/bench_prefill32k.json')); print(d['value'], d['e2e']['value'], d['resident'], d['paged_over_resident'], d['page_in']['achieved_gbps'], d['exposed_xfer_pct'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['down'])
"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_moe_gemm_pair -s 2 -c 2 -o $O/pair_T16384 python tools/profile_layer.py --config mixtral --tokens 16384 --reps 1 > $O/ncu_pair.log 2>&1
ls $O
