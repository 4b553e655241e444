#!/bin/bash
for d in 0 4 8 12; do echo "dbg=$d"; for n in 117440512 3145728; do XPGB_DEC_DBG=$d timeout 120 python tools/profile_codec.py --values $n 2>/dev/null | cut -c1-100; done; done
