#!/bin/bash
# A/B builds with compile-time knobs: tools/ab_build.sh NAME SRC "-DX=1 -DY=2"
# (SRC = sweep.cu, fused.cu, ...) -> ab/NAME/libotg.so (other objects from the
# default build); run with OTG_LIB=ab/NAME/libotg.so
set -e
cd "$(dirname "$0")/.."
NAME=$1; SRC=$2; DEFS=$3
mkdir -p ab/$NAME
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  --expt-relaxed-constexpr $DEFS -c paper_2605_30267_b200/csrc/$SRC -o ab/$NAME/$SRC.o
objs=$(ls paper_2605_30267_b200/_build/*.o | grep -v "/$SRC.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ab/$NAME/libotg.so \
  ab/$NAME/$SRC.o $objs -ldl -lpthread
echo "built ab/$NAME/libotg.so"
