mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 -o gpurun_out/prof_cublas python -c "
import torch
a=torch.randn(8192,8192,device='cuda',dtype=torch.bfloat16)
b=torch.randn(8192,8192,device='cuda',dtype=torch.bfloat16)
for _ in range(4): a@b.T
torch.cuda.synchronize()" > gpurun_out/ncu_cublas.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ws_gemm -s 2 -c 1 -o gpurun_out/prof_gemm2cta_k16 python scripts/prof_one.py gemm --K 16384 --cta_pair > gpurun_out/ncu_gemm2b.log 2>&1
