#!/bin/bash
# Same-box A/B builds of the persistent decode kernel: scripts/ab_build.sh NAME path/to/decode_stack.cu
# -> build/ab/NAME/paper_2602_21144_b200 (a copy of the package with that variant of libssmtp.so);
# run a script against it with DS_PKG_ROOT=build/ab/NAME.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; SRC=$2
OUT=$ROOT/build/ab/$NAME
rm -rf "$OUT"; mkdir -p "$OUT"
cp -r "$ROOT/paper_2602_21144_b200" "$OUT/"
rm -f "$OUT/paper_2602_21144_b200/libssmtp.so"
cp "$SRC" "$OUT/decode_stack.cu"
cp "$ROOT"/paper_2602_21144_b200/csrc/*.cuh "$ROOT"/paper_2602_21144_b200/csrc/*.h "$OUT/"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I"$ROOT/include" --expt-relaxed-constexpr -c "$OUT/decode_stack.cu" -o "$OUT/decode_stack.o"
OBJS=$(ls "$ROOT"/build/libssmtp/*.o | grep -v decode_stack.o)
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC $OBJS "$OUT/decode_stack.o" \
  -o "$OUT/paper_2602_21144_b200/libssmtp.so"
echo "$OUT"
