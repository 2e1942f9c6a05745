#!/bin/bash
# Alternating A/B of two builds of libws.so on the GEMM sweep shapes and cuBLAS (developer script):
#   bash scripts/lib_ab.sh path/to/libA.so path/to/libB.so
A=$1; B=$2
for r in 1 2 3; do
  for L in $A $B; do
    for K in 2048 16384; do
      WS_LIB=$L ROUNDS=1 SECS=1.5 timeout 120 python scripts/gemm_ab.py $K "{}" 2>&1 | tail -1 | sed "s|^|$(basename $L) |"
    done
  done
  ROUNDS=1 SECS=1.5 timeout 120 python scripts/gemm_ab.py 16384 '{"cublas":1}' 2>&1 | tail -1 | sed "s|^|cublas |"
done
