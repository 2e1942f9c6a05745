#!/bin/bash
# Tile-policy sweep against cuBLAS (bf16 and FP8, sustained, scripts/gemm_ab.py); developer script.
for K in 256 512 1024 2048 4096; do ROUNDS=2 SECS=0.8 timeout 300 python scripts/gemm_ab.py $K "{}" "{\"cta_pair\":1,\"bn\":512}" "{\"cta_pair\":1,\"bn\":256}" "{\"cublas\":1}" 2>&1 | tail -4; done
for K in 1024 2048 4096; do FP8=1 ROUNDS=2 SECS=0.8 timeout 300 python scripts/gemm_ab.py $K "{}" "{\"cta_pair\":1,\"bn\":512}" "{\"cublas\":1}" 2>&1 | tail -3; done
