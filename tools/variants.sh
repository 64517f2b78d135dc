#!/bin/bash
# Build a variant of libtaco_b200.so with extra nvcc defines into build/variants/NAME.so
#   tools/variants.sh NAME "-DFOO=1 -DBAR=2"
set -e
NAME=$1; DEFS=$2
OUT=build/variants/$NAME; mkdir -p $OUT
cd paper_2603_24919_b200/csrc
for f in index query build exact eigen; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off --fmad=false $DEFS -c $f.cu -o ../../$OUT/$f.o &
done
g++ -O2 -fPIC -std=c++17 -ffp-contract=off -fopenmp -c jacobi.cpp -o ../../$OUT/jacobi.o
wait
cd ../../$OUT
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart=static -o ../$NAME.so index.o query.o build.o exact.o eigen.o jacobi.o -Xcompiler -fopenmp -lgomp
echo built build/variants/$NAME.so
