"""PCIe bounds of the e2e step (developer script, GPU): pinned H2D of every job's A and B, D2H of
every C, both at once, and gemm_tn_host over the same jobs (the bench's K sweep, bf16)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws

KS = [256, 512, 1024, 2048, 4096, 8192, 16384]
M = N = 8192
dev = torch.device("cuda")
jobs = [(torch.randn(M, K).to(torch.bfloat16).pin_memory(), torch.randn(N, K).to(torch.bfloat16).pin_memory(),
         torch.empty(M, N, dtype=torch.bfloat16).pin_memory()) for K in KS]
da = [(torch.empty(a.shape, dtype=a.dtype, device=dev), torch.empty(b.shape, dtype=b.dtype, device=dev),
       torch.empty(c.shape, dtype=c.dtype, device=dev)) for a, b, c in jobs]
h2d_bytes = sum(a.numel() * 2 + b.numel() * 2 for a, b, _ in jobs)
d2h_bytes = sum(c.numel() * 2 for _, _, c in jobs)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, n=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e3


def h2d():
    with torch.cuda.stream(s1):
        for (a, b, _), (x, y, _) in zip(jobs, da):
            x.copy_(a, non_blocking=True)
            y.copy_(b, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        for (_, _, c), (_, _, z) in zip(jobs, da):
            c.copy_(z, non_blocking=True)


t_h = timed(h2d)
t_d = timed(d2h)
t_both = timed(lambda: (h2d(), d2h()))
t_pipe = timed(lambda: ws.gemm_tn_host(jobs, device=dev))
for rc in (1, 2, 8):
    t = timed(lambda: ws.gemm_tn_host(jobs, device=dev, row_chunks=rc))
    print(f"row_chunks={rc}: {t:.2f} ms")
flops = sum(2.0 * M * N * K for K in KS)
print(f"H2D {h2d_bytes / 1e9:.2f} GB in {t_h:.2f} ms = {h2d_bytes / t_h / 1e6:.1f} GB/s")
print(f"D2H {d2h_bytes / 1e9:.2f} GB in {t_d:.2f} ms = {d2h_bytes / t_d / 1e6:.1f} GB/s")
print(f"both directions at once: {t_both:.2f} ms")
print(f"gemm_tn_host step: {t_pipe:.2f} ms = {flops / t_pipe / 1e9:.1f} TFLOP/s "
      f"(H2D-only bound {flops / t_h / 1e9:.1f})")

# job order: the sweep ascending in K front-loads 128 MB copy-outs behind tiny inputs and ends with
# 512 MB inputs behind one copy-out; interleaving large and small K keeps both directions busy
orders = {"ascending": list(range(len(KS))), "descending": list(range(len(KS)))[::-1],
          "interleaved": [6, 0, 5, 1, 4, 2, 3], "interleaved_small_first": [0, 6, 1, 5, 2, 4, 3]}
for name, order in orders.items():
    js = [jobs[i] for i in order]
    t = timed(lambda: ws.gemm_tn_host(js, device=dev))
    print(f"order {name:24s} {[KS[i] for i in order]}: {t:.2f} ms = {flops / t / 1e9:.1f} TFLOP/s")
