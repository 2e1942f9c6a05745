mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ws_gemm -s 2 -c 1 -o gpurun_out/prof_gemm2cta python scripts/prof_one.py gemm --K 8192 --cta_pair > gpurun_out/ncu_gemm2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ws_gemm -s 2 -c 1 -o gpurun_out/prof_gemm1cta python scripts/prof_one.py gemm --K 8192 > gpurun_out/ncu_gemm1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ampere\|sm100\|gemm\|Kernel -s 2 -c 1 -o gpurun_out/prof_cublas python -c "
import torch
a=torch.randn(8192,8192,device='cuda',dtype=torch.bfloat16)
for _ in range(4): a@a.T
torch.cuda.synchronize()" > gpurun_out/ncu_cublas.log 2>&1
ls gpurun_out
