#!/bin/bash
# Dev A/B: libbinsketch.so with build.cu compiled under extra -D flags -> variants/libbinsketch_<name>.so
# usage: tools/build_variant_build.sh <name> "<-D flags>"
set -e
cd "$(dirname "$0")/.."
mkdir -p variants/obj_$1
C=paper_1910_04658_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Iinclude -I$C"
nvcc -c $C/build.cu -o variants/obj_$1/build.o $F $2
nvcc -shared -o variants/libbinsketch_$1.so paper_1910_04658_b200/_build/api.o variants/obj_$1/build.o paper_1910_04658_b200/_build/pairs.o paper_1910_04658_b200/_build/join.o paper_1910_04658_b200/_build/tc.o -gencode arch=compute_100a,code=sm_100a
echo built variants/libbinsketch_$1.so
