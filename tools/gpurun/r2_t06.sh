#!/bin/bash
# round 2 (re-entry): state check of the restored tree: GPU suite, smoke, default bench, reference arm
O=gpurun_out/r2_t06; mkdir -p $O
nproc > $O/nproc.txt; nvidia-smi > $O/smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
export XPGB_PARITY_LOG=$O/parity.jsonl
timeout 1800 python -m pytest tests -q -m gpu --durations=25 > $O/pytest.log 2>&1; echo "pytest rc=$?"
tail -40 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $O/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; tail -c 4000 $O/bench.json; tail -5 $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref rc=$?"; tail -c 2000 $O/bench_ref.json; tail -5 $O/bench_ref.err
