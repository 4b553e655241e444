#!/bin/bash
O=gpurun_out/t11; mkdir -p $O
timeout 240 python -m pytest tests/test_gpu_pair_gemm.py -q -x > $O/pytest_pair.log 2>&1; echo "pair rc=$?"; tail -15 $O/pytest_pair.log
