#!/bin/bash
for ch in 1024 512 256 128; do echo "chunk=$ch"; for n in 117440512 3145728; do timeout 120 python tools/profile_codec.py --values $n --chunk $ch 2>/dev/null | cut -c1-110; done; done
