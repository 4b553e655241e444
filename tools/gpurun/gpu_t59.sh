#!/bin/bash
O=gpurun_out/t59; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_ep_multiproc.py -q -x > $O/pytest_ep.log 2>&1; tail -1 $O/pytest_ep.log; grep -E "^E |Error|error|FAILED" $O/pytest_ep.log | head -20
