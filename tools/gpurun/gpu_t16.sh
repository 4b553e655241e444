#!/bin/bash
O=gpurun_out/t16; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -4 $O/pytest.log
grep -E "^E |FAILED" $O/pytest.log | head -10
