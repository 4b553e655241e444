#!/bin/bash
# Build libxpgb.so with one source file rebuilt (optionally from a replacement, with extra nvcc
# flags), for same-box A/B timing:
#   tools/micro/ab/build_variant.sh NAME path/to/moe_gemm_dec.cu [extra nvcc flags...]
#   XPGB_LIB_PATH=tools/micro/ab/NAME/libxpgb.so python tools/profile_fused.py ...
set -e
NAME=$1; SRC=$2; shift 2
BASE=$(basename $SRC .cu)
ROOT=$(cd "$(dirname "$0")/../../.." && pwd)
OUT=$ROOT/tools/micro/ab/$NAME; mkdir -p $OUT
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$ROOT/include -I$ROOT/paper_2604_02715_b200/csrc $*"
cp $SRC $OUT/$BASE.cu
nvcc $F -c $OUT/$BASE.cu -o $OUT/$BASE.o
OBJS=""
for o in $ROOT/build/obj/*.o; do
  if [ $(basename $o .o) = $BASE ]; then OBJS="$OBJS $OUT/$BASE.o"; else OBJS="$OBJS $o"; fi
done
nvcc -shared -cudart static -gencode arch=compute_100a,code=sm_100a -o $OUT/libxpgb.so $OBJS
echo $OUT/libxpgb.so
