import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, ctypes
import paper_2510_14719_b200 as ws
from paper_2510_14719_b200 import _lib, ops
a = torch.randn(1024, 1024, device="cuda", dtype=torch.float16)
b = torch.randn(1024, 1024, device="cuda", dtype=torch.float16)
c = torch.empty(1024, 1024, device="cuda", dtype=torch.float32)
for _ in range(20): ws.gemm_tn(a, b, c)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n): ws.gemm_tn(a, b, c)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"full call {1e6*(t1-t0)/n:.2f} us")
# the C call alone with a prepared launch (ws_gemm_plan_launch)
key = next(iter(ops._PLAN_CACHE))
plan = ops._PLAN_CACHE[key].ptr
lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream
t0 = time.perf_counter()
for _ in range(n): lib.ws_gemm_plan_launch(plan, s)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"C-ABI plan launch alone {1e6*(t1-t0)/n:.2f} us")
# a CUDA graph of 100 calls, replayed
g = torch.cuda.CUDAGraph()
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    ws.gemm_tn(a, b, c)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        for _ in range(100): ws.gemm_tn(a, b, c)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): g.replay()
e1.record(); torch.cuda.synchronize()
print(f"graph replay {1e3 * e0.elapsed_time(e1) / 2000:.2f} us per GEMM ({2 * 1024**3 / (e0.elapsed_time(e1) / 2000 * 1e-3) / 1e12:.1f} TFLOP/s)")
t0 = time.perf_counter()
for _ in range(n): torch._C._cuda_getCurrentRawStream(0)
print(f"raw stream {1e6*(time.perf_counter()-t0)/n:.2f} us")
