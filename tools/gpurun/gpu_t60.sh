#!/bin/bash
O=gpurun_out/t60; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_ep_multiproc.py -q -x -k "world1" > $O/pytest_w1.log 2>&1; tail -1 $O/pytest_w1.log; grep -E "^E " $O/pytest_w1.log | head -10
timeout 500 python -m pytest tests/test_gpu_ep_multiproc.py -q -x -k "p2p" > $O/pytest_ep.log 2>&1; tail -1 $O/pytest_ep.log; grep -E "^E |rror" $O/pytest_ep.log | head -20
