"""C1 (fp16 1024^3) per-call timing probe: eager ws.gemm_tn and torch.matmul, timed like bench.py
(20 back-to-back calls between CUDA events), before and after cuBLASLt FP8 calls, plus the host
time per call (developer script)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2510_14719_b200 as ws

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
a = torch.randn(1024, 1024, device=dev).half()
b = torch.randn(1024, 1024, device=dev).half()
c1 = torch.empty(1024, 1024, device=dev, dtype=torch.float32)
c16 = torch.empty(1024, 1024, device=dev, dtype=torch.float16)


def timed(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    t0 = time.perf_counter()
    for _ in range(iters):
        fn()
    t1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3, (t1 - t0) / iters * 1e6


def report(tag):
    for name, fn in (("ws fp32 out", lambda: ws.gemm_tn(a, b, c1)), ("ws fp16 out", lambda: ws.gemm_tn(a, b, c16)),
                     ("torch.matmul", lambda: torch.matmul(a, b.T, out=c16))):
        us, host = timed(fn)
        us2, host2 = timed(fn, 200)
        print(f"{tag:28s} {name:14s} 20 calls: {us:6.2f} us/call ({2 * 1024**3 / us / 1e6:6.1f} TFLOP/s), host {host:5.2f} us | "
              f"200 calls: {us2:6.2f} us/call, host {host2:5.2f} us")


report("fresh")
a8 = (torch.randn(8192, 2048, device=dev) * 0.5).to(torch.float8_e4m3fn)
b8 = (torch.randn(8192, 2048, device=dev) * 0.5).to(torch.float8_e4m3fn)
sa = torch.tensor(0.5, device=dev)
sb = torch.tensor(2.0, device=dev)
for _ in range(20):
    torch._scaled_mm(a8, b8.t(), scale_a=sa, scale_b=sb, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
report("after torch._scaled_mm")
big = torch.randn(8192, 16384, device=dev).to(torch.bfloat16)
cb = torch.empty(8192, 8192, device=dev, dtype=torch.bfloat16)
for _ in range(50):
    ws.gemm_tn(big, big[:8192], cb)
torch.cuda.synchronize()
report("right after 50 big GEMMs")
time.sleep(1.0)
report("after 1 s idle")
