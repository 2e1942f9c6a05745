"""Quick GPU validation + timing of the GEMM path (developer script, run under gpurun)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws

def vals(shape, seed, dev="cuda"):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return ((torch.randint(0, 33, shape, generator=g).float() - 16.0) / 4.0).to(dev)

def check(M, N, K, dt, out_dt, **kw):
    a = vals((M, K), 1).to(dt); b = vals((N, K), 2).to(dt)
    ref = (a.double() @ b.double().T)
    c = ws.gemm_tn(a, b, out_dtype=out_dt, **kw)
    torch.cuda.synchronize()
    if out_dt == torch.float32:
        bad = (c.double() != ref).sum().item()
        err = (c.double() - ref).abs().max().item()
        print(f"M={M} N={N} K={K} {dt} -> {out_dt} {kw}: mismatches={bad} maxabs={err}", flush=True)
    else:
        rel = ((c.double() - ref).abs().max() / ref.abs().max()).item()
        print(f"M={M} N={N} K={K} {dt} -> {out_dt} {kw}: relerr={rel:.3e}", flush=True)

def bench(M, N, K, dt, out_dt, iters=20, **kw):
    a = torch.randn(M, K, device="cuda").to(dt); b = torch.randn(N, K, device="cuda").to(dt)
    c = torch.empty(M, N, device="cuda", dtype=out_dt)
    for _ in range(3): ws.gemm_tn(a, b, c, **kw)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): ws.gemm_tn(a, b, c, **kw)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    print(f"BENCH M={M} N={N} K={K} {dt} {kw}: {ms:.3f} ms  {2*M*N*K/ms/1e9:.1f} TFLOP/s", flush=True)

if __name__ == "__main__":
    torch.cuda.init()
    check(256, 256, 64, torch.bfloat16, torch.float32, cta_pair=True)
    check(512, 512, 256, torch.bfloat16, torch.float32, cta_pair=True)
    check(1024, 1024, 1024, torch.float16, torch.float32, cta_pair=True)
    check(1024, 1024, 1024, torch.bfloat16, torch.float32, cta_pair=True, D=2, P=1)
    check(1024, 1024, 1024, torch.bfloat16, torch.float32, cta_pair=True, persistent=False)
    check(1024, 1024, 1024, torch.float8_e4m3fn, torch.float32, cta_pair=True)
    check(2048, 2048, 4096, torch.bfloat16, torch.bfloat16, cta_pair=True)
    check(4096, 4096, 4096, torch.bfloat16, torch.float32, cta_pair=True)
    check(1024, 1024, 1024, torch.bfloat16, torch.float32, cta_pair=True, bn=128)
    for K in (256, 1024, 8192, 16384):
        bench(8192, 8192, K, torch.bfloat16, torch.bfloat16)
        bench(8192, 8192, K, torch.bfloat16, torch.bfloat16, cta_pair=True)
    for gm in (4, 8, 16):
        bench(8192, 8192, 8192, torch.bfloat16, torch.bfloat16, cta_pair=True, group_m=gm)
    bench(8192, 8192, 8192, torch.float8_e4m3fn, torch.bfloat16, cta_pair=True)
    bench(8192, 8192, 16384, torch.float8_e4m3fn, torch.bfloat16, cta_pair=True)
    a = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    for _ in range(3): a @ a.T
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
    for _ in range(20): a @ a.T
    e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/20
    print(f"cuBLAS bf16 8192^3: {ms:.3f} ms {2*8192**3/ms/1e9:.1f} TFLOP/s")
