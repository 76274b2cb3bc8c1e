#!/bin/bash
# Build an A/B variant of the library into ab/<name>.so: the given source compiled with extra flags, linked
# with the other objects of the current build.  usage: tools/build_variant.sh <name> <source.cu> [-Dflags...]
set -e
name=$1; src=$2; shift 2
mkdir -p abx /tmp/abobj
P=paper_2507_02809_b200
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -I include "$@" \
  -c $P/csrc/$src -o /tmp/abobj/$name.o
objs=$(ls $P/_obj/*.o | grep -v "/${src%.*}.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o abx/$name.so $objs /tmp/abobj/$name.o -lcuda
echo abx/$name.so
