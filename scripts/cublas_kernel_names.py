"""Print the cuBLAS / cuBLASLt kernel chosen for the bench shapes (developer script, GPU)."""
import torch
from torch.profiler import profile, ProfilerActivity

for dt in (torch.bfloat16, torch.float8_e4m3fn):
    for K in (256, 512, 1024, 2048, 4096, 16384):
        a = torch.randn(8192, K, device="cuda").to(dt); b = torch.randn(8192, K, device="cuda").to(dt)
        c = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
        one = torch.ones((), device="cuda")
        fn = (lambda: torch.matmul(a, b.T, out=c)) if dt == torch.bfloat16 else \
             (lambda: torch._scaled_mm(a, b.T, one, one, out_dtype=torch.bfloat16, out=c))
        fn(); torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as p:
            fn(); torch.cuda.synchronize()
        names = [e.name for e in p.events() if e.device_type.name == "CUDA"]
        print(dt, K, names[:2], flush=True)
