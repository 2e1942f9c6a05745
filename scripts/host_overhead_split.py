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
# the C call alone with a prepared descriptor
key = next(iter(ops._DESC_CACHE))
d = ops._DESC_CACHE[key]
lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream
t0 = time.perf_counter()
for _ in range(n): lib.ws_gemm_tn(ctypes.byref(d), s)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"C-ABI call alone {1e6*(t1-t0)/n:.2f} us")
t0 = time.perf_counter()
for _ in range(n): torch._C._cuda_getCurrentRawStream(0)
print(f"raw stream {1e6*(time.perf_counter()-t0)/n:.2f} us")
