#!/bin/bash
# Build a variant library variants/lib<NAME>.so: rollout_tc.cu (or the files in
# $SRCS) recompiled with extra -D flags, linked with the main build's other objects.
# usage: bash profiles/build_variant.sh NAME "-DFOO=1 -DBAR=0" [rollout_tc critic_tc]
set -e
NAME=$1; FLAGS=$2; shift 2; SRCS=${@:-rollout_tc}
cd "$(dirname "$0")/.."
mkdir -p variants/build_$NAME
OBJS=""
for o in build/*.o; do
  b=$(basename $o .o)
  if [[ " $SRCS " == *" $b "* ]]; then
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Iinclude \
      --expt-relaxed-constexpr -Xptxas -warn-spills $FLAGS -c paper_2602_19699_b200/csrc/$b.cu -o variants/build_$NAME/$b.o
    OBJS="$OBJS variants/build_$NAME/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o variants/lib$NAME.so $OBJS -lcudart
echo built variants/lib$NAME.so
