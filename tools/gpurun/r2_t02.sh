#!/bin/bash
# round 2: split-activation GEMMs + device EP plan: full GPU suite, full-shape parity, smoke
O=gpurun_out/r2_t02; mkdir -p $O
export XPGB_PARITY_LOG=$O/parity.jsonl
timeout 1500 python -m pytest tests -q -x -m gpu --durations=15 > $O/pytest.log 2>&1; echo "pytest rc=$?"
tail -25 $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 $O/smoke.log
