#!/bin/bash
# Dev A/B: build libbinsketch.so with an alternative tc.cu -> variants/libbinsketch_<name>.so
# usage: tools/build_variant.sh <name> <tc.cu path>
set -e
cd "$(dirname "$0")/.."
mkdir -p variants/obj_$1
C=paper_1910_04658_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Iinclude -I$C"
nvcc -c $2 -o variants/obj_$1/tc.o $F -fmad=false -I$C
nvcc -shared -o variants/libbinsketch_$1.so paper_1910_04658_b200/_build/api.o paper_1910_04658_b200/_build/build.o paper_1910_04658_b200/_build/pairs.o paper_1910_04658_b200/_build/join.o variants/obj_$1/tc.o -gencode arch=compute_100a,code=sm_100a
echo built variants/libbinsketch_$1.so
