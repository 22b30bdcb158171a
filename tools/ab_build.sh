#!/bin/bash
# Build an experimental libhist256 variant into tools/ablib/NAME.so from the working
# source with sed edits applied (A/B measurement only; never loaded by the package
# unless HS_LIBHIST256 points at it).
# usage: tools/ab_build.sh NAME 'sed-expr' ['sed-expr' ...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
src=/tmp/ab_$name.cu
cp paper_1011_0235_b200/csrc/hs_kernels.cu $src
for e in "$@"; do sed -i "$e" $src; done
sed -i 's|"../../include/hist256.h"|"hist256.h"|' $src
nvcc -shared -Xcompiler -fPIC -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a \
  -Xcompiler -ffp-contract=off -I include $src paper_1011_0235_b200/csrc/hs_host.cpp -o tools/ablib/$name.so
echo built tools/ablib/$name.so
