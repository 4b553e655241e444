#!/bin/bash
O=gpurun_out/t63; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for t in 32768 65536; do timeout 900 python bench.py --config mixtral --prefill --tokens $t --steps 3 > $O/bench_prefill$t.json 2> $O/bench_prefill$t.err; echo "prefill $t rc=$?"
python -c "
import json; d=json.load(open('$O/bench_prefill$t.json')); print(round(d['value'],1), round(d['e2e']['value'],1), d['resident'], round(d.get('paged_over_resident') or 0,3), round(d['exposed_xfer_pct'],1), round(d['page_in']['achieved_gbps'],1)); r=d['roofline']; print(r.get('kernel'), round(r.get('frac'),3), 'gemm', r.get('gemm',{}).get('bound'), round(r.get('gemm',{}).get('frac',0),3))"; done
