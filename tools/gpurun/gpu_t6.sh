#!/bin/bash
O=gpurun_out/t6; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 1200 python tools/sweep.py budget --config mixtral --steps 3 > $O/sweep_budget_mixtral.jsonl 2> $O/sweep.err; tail -2 $O/sweep.err
cut -c1-400 $O/sweep_budget_mixtral.jsonl
