#!/bin/bash
# round 2: GPU suite after split activations + device EP plan + fault propagation
O=gpurun_out/r2_t03; mkdir -p $O
export XPGB_PARITY_LOG=$O/parity.jsonl
timeout 1800 python -m pytest tests -q -m gpu --durations=20 > $O/pytest.log 2>&1; echo "pytest rc=$?"
tail -30 $O/pytest.log
