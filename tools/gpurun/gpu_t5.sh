#!/bin/bash
O=gpurun_out/t5; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 600 python bench.py --steps 5 > $O/bench.json 2> $O/bench.err; tail -2 $O/bench.err
cut -c1-600 $O/bench.json
