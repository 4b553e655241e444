#!/bin/bash
for d in 0 1 2 3; do echo "dbg=$d"; XPGB_DEC_DBG=$d timeout 120 python tools/profile_codec.py --values 3145728 2>/dev/null | cut -c1-120; XPGB_DEC_DBG=$d timeout 120 python tools/profile_codec.py 2>/dev/null | cut -c1-120; done
