"""Bit-exactness sweep of the GEMM launch variants (developer script, run under gpurun)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
import gpu_quick_gemm as g

bf, f16, f8 = torch.bfloat16, torch.float16, torch.float8_e4m3fn
for cp, bn in [(False, 128), (False, 256), (True, 128), (True, 256), (True, 512)]:
    g.check(1024, 1024, 1024, bf, torch.float32, cta_pair=cp, bn=bn)
    g.check(1024, 1024, 512, f16, torch.float32, cta_pair=cp, bn=bn)
    g.check(2048, 1536 if bn != 512 else 2048, 1024, f8, torch.float32, cta_pair=cp, bn=bn)
    g.check(1024, 1024, 1024, bf, bf, cta_pair=cp, bn=bn)
    g.check(1024, 1024, 1024, bf, f16, cta_pair=cp, bn=bn)
    g.check(512, 1024, 256, bf, torch.float32, cta_pair=cp, bn=bn, D=2, P=1)
g.check(1024, 1024, 1024, f8, bf, cta_pair=True, bn=512, scale_a=0.5, scale_b=2.0)
