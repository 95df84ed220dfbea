#!/bin/bash
# Same-box A/B builds of one kernel source: scripts/ab_build.sh NAME path/to/variant_of_X.cu [X.cu]
# -> build/ab/NAME/paper_2602_21144_b200 (a copy of the package whose libssmtp.so links the variant in
# place of csrc/X.o; X defaults to decode_stack.cu); run a script against it with DS_PKG_ROOT=build/ab/NAME.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; SRC=$2; BASE=${3:-decode_stack.cu}
STEM=${BASE%.cu}
OUT=$ROOT/build/ab/$NAME
rm -rf "$OUT"; mkdir -p "$OUT"
cp -r "$ROOT/paper_2602_21144_b200" "$OUT/"
rm -f "$OUT/paper_2602_21144_b200/libssmtp.so"
# the variant sits two levels below a copy of include/ (sources include "../../include/ssm_tp.h")
mkdir -p "$OUT/src/csrc"
cp -r "$ROOT/include" "$OUT/include"
cp "$SRC" "$OUT/src/csrc/$BASE"
cp "$ROOT"/paper_2602_21144_b200/csrc/*.cuh "$ROOT"/paper_2602_21144_b200/csrc/*.h "$OUT/src/csrc/"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I"$ROOT/include" --expt-relaxed-constexpr -c "$OUT/src/csrc/$BASE" -o "$OUT/$STEM.o"
OBJS=$(ls "$ROOT"/build/libssmtp/*.o | grep -v "/$STEM.o")
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC $OBJS "$OUT/$STEM.o" \
  -o "$OUT/paper_2602_21144_b200/libssmtp.so"
echo "$OUT"
