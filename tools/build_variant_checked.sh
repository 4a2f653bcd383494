#!/bin/bash
# Dev: the checked library (K1 shared-memory region checks + top-k epilogue index asserts, traps on a
# violation) -> variants/libbinsketch_checked.so; with "selftest" also the deliberately mis-bounded
# K1 checker -> variants/libbinsketch_checked_selftest.so (must trap).
set -e
cd "$(dirname "$0")/.."
C=paper_1910_04658_b200/csrc
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off -Iinclude -I$C"
mkdir -p variants/obj_checked
nvcc -c $C/build.cu -o variants/obj_checked/build.o $F -DBSK_CHECKED &
nvcc -c $C/tc.cu -o variants/obj_checked/tc.o $F -fmad=false -DBSK_CHECKED &
[ "$1" = selftest ] && nvcc -c $C/build.cu -o variants/obj_checked/build_self.o $F -DBSK_CHECKED -DBSK_CHECKED_SELFTEST &
wait
B=paper_1910_04658_b200/_build
nvcc -shared -o variants/libbinsketch_checked.so $B/api.o variants/obj_checked/build.o $B/pairs.o $B/join.o variants/obj_checked/tc.o -gencode arch=compute_100a,code=sm_100a
[ "$1" = selftest ] && nvcc -shared -o variants/libbinsketch_checked_selftest.so $B/api.o variants/obj_checked/build_self.o $B/pairs.o $B/join.o $B/tc.o -gencode arch=compute_100a,code=sm_100a
echo built checked
