"""Tile/pipeline sweep of the bf16 GEMM at short K (developer script, run under gpurun)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws


def t_ms(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


M = N = 8192
for K in [int(x) for x in os.environ.get("KS", "256,512,1024,2048").split(",")]:
    a = torch.randn(M, K, device="cuda").bfloat16(); b = torch.randn(N, K, device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ms = t_ms(lambda: torch.matmul(a, b.T, out=c))
    print(f"K={K} cuBLAS {2*M*N*K/ms/1e9:.1f} TFLOP/s ({ms*1e3:.1f} us)", flush=True)
    res = []
    for cp in (0, 1):
        for bn in (128, 256):
            for D in (2, 3, 4, 6, 8):
                for gm in (0, 2, 4, 8):
                    try:
                        ms = t_ms(lambda: ws.gemm_tn(a, b, c, cta_pair=bool(cp), bn=bn, D=D, group_m=gm))
                    except ws.WsError:
                        continue
                    res.append((2 * M * N * K / ms / 1e9, cp, bn, D, gm, ms))
    res.sort(reverse=True)
    for r in res[:6]:
        print(f"K={K} ours {r[0]:.1f} TFLOP/s ({r[5]*1e3:.1f} us) cta_pair={r[1]} bn={r[2]} D={r[3]} group_m={r[4]}", flush=True)
    auto = t_ms(lambda: ws.gemm_tn(a, b, c))
    print(f"K={K} ours auto {2*M*N*K/auto/1e9:.1f} TFLOP/s", flush=True)
