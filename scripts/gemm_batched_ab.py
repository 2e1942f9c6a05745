"""Batched GEMM (one launch over batch x tiles) vs cuBLAS strided-batched (torch.bmm), alternating
windows on one box (developer script, GPU).  python scripts/gemm_batched_ab.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws


def window(fn, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for nb, M, N, K in [(8, 2048, 2048, 2048), (16, 1024, 1024, 4096), (4, 4096, 4096, 4096), (64, 512, 512, 1024)]:
    a = torch.randn(nb, M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(nb, N, K, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(nb, M, N, device="cuda", dtype=torch.bfloat16)
    ours = lambda: ws.gemm_tn(a, b, c)
    lib = lambda: torch.bmm(a, b.transpose(1, 2), out=c)
    ours(); lib(); torch.cuda.synchronize()
    ref = torch.bmm(a.float(), b.float().transpose(1, 2))
    err = ((c.float() - ref).abs().max() / ref.abs().max()).item() if False else None
    ours(); torch.cuda.synchronize()
    err = ((c.float() - ref).abs().max() / ref.abs().max()).item()
    fl = 2.0 * nb * M * N * K
    n = max(5, int(2e13 / fl))
    to, tl = [], []
    for w in range(6):
        time.sleep(0.2)
        for fn, acc in ((ours, to), (lib, tl)) if w % 2 == 0 else ((lib, tl), (ours, to)):
            acc.append(window(fn, n))
    mo, ml = sorted(to)[3], sorted(tl)[3]
    print(f"batch {nb} x {M}x{N}x{K}: ours {fl / mo / 1e9:.1f} TFLOP/s, cuBLAS bmm {fl / ml / 1e9:.1f} "
          f"(ratio {ml / mo:.3f}), rel err {err:.1e}", flush=True)
