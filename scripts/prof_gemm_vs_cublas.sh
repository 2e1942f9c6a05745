#!/bin/bash
# ncu --set full of our cta-pair GEMM and cuBLAS on the same 8192 x 8192 x K bf16 problem.
mkdir -p gpurun_out
K=${K:-16384}
timeout 300 ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 -o gpurun_out/prof_cublas_k$K python -c "
import torch
a=torch.randn(8192,$K,device='cuda',dtype=torch.bfloat16)
b=torch.randn(8192,$K,device='cuda',dtype=torch.bfloat16)
for _ in range(4): a@b.T
torch.cuda.synchronize()" > gpurun_out/ncu_cublas.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ws_gemm -s 2 -c 1 -o gpurun_out/prof_ours_k$K python scripts/prof_one.py gemm --K $K --cta_pair $EXTRA > gpurun_out/ncu_ours.log 2>&1
ls -la gpurun_out/*.ncu-rep
