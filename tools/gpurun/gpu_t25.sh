#!/bin/bash
# compare decoder builds: committed v2 vs working tree v3 (same tool)
for v in cur v2; do
  if [ $v = v2 ]; then cp paper_2604_02715_b200/libxpgb.so /tmp/cur.so; cp tools/exp/libxpgb_v2.so paper_2604_02715_b200/libxpgb.so; fi
  echo "== $v"; for n in 117440512 29360128 3145728; do timeout 120 python tools/profile_codec.py --values $n 2>/dev/null | cut -c1-110; done
done
cp /tmp/cur.so paper_2604_02715_b200/libxpgb.so
