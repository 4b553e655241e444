#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_codec.py -q -x 2>&1 | tail -1
for n in 117440512 29360128 3145728; do timeout 120 python tools/profile_codec.py --values $n 2>/dev/null | cut -c1-110; done
