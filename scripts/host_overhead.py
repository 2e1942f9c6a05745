"""Host cost per ws.gemm_tn call vs its device time on the C1 problem (developer script, GPU)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws

a = torch.randn(1024, 1024, device="cuda", dtype=torch.float16)
b = torch.randn(1024, 1024, device="cuda", dtype=torch.float16)
c = torch.empty(1024, 1024, device="cuda", dtype=torch.float32)
for _ in range(10):
    ws.gemm_tn(a, b, c)
torch.cuda.synchronize()
n = 500
t0 = time.perf_counter()
for _ in range(n):
    ws.gemm_tn(a, b, c)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host per call {1e6 * (t1 - t0) / n:.1f} us, wall per call {1e6 * (t2 - t0) / n:.1f} us")
# device time alone: a CUDA graph of the same launches replays without host work
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    ws.gemm_tn(a, b, c, stream=s)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for _ in range(50):
            ws.gemm_tn(a, b, c, stream=s)
g.replay(); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.replay()
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 500
print(f"device per launch (graph replay) {us:.1f} us = {2 * 1024**3 / us / 1e6:.1f} TFLOP/s")
