import json, sys, time, torch
sys.path.insert(0, ".")
import paper_2510_14719_b200 as ws
from paper_2510_14719_b200 import trace
a = torch.randn(256, 1024, device="cuda", dtype=torch.bfloat16)
t0 = time.time()
try:
    ws.gemm_tn(a, a)
    torch.cuda.synchronize()
except Exception as e:
    print("ERR", type(e).__name__, str(e)[:300], time.time() - t0)
print(json.dumps({"watchdog": trace.watchdog()}))
