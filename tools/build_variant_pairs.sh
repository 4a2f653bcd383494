#!/bin/bash
# Dev A/B: libbinsketch.so with pairs.cu compiled under extra -D flags -> variants/libbinsketch_<name>.so
# usage: tools/build_variant_tc.sh <name> "<-D flags>"
set -e
cd "$(dirname "$0")/.."
mkdir -p variants/obj_$1
C=paper_1910_04658_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Iinclude -I$C -fmad=false"
nvcc -c $C/pairs.cu -o variants/obj_$1/pairs.o $F $2
nvcc -shared -o variants/libbinsketch_$1.so paper_1910_04658_b200/_build/api.o paper_1910_04658_b200/_build/build.o variants/obj_$1/pairs.o paper_1910_04658_b200/_build/join.o paper_1910_04658_b200/_build/tc.o -gencode arch=compute_100a,code=sm_100a
echo built variants/libbinsketch_$1.so
