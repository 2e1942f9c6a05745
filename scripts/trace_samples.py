"""Sample device traces in the reference's trace JSON schema (developer script, GPU): the bench's
K=2048 GEMM (auto tiles) and the C4 attention at S=4K, written to gpurun_out/."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws
from paper_2510_14719_b200 import _lib, trace

os.makedirs("gpurun_out", exist_ok=True)
a = torch.randn(8192, 2048, device="cuda", dtype=torch.bfloat16)
b = torch.randn(8192, 2048, device="cuda", dtype=torch.bfloat16)
c = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ws.gemm_tn(a, b, c)
tr = torch.zeros(2 * 32 * 16, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.ws_debug_gemm_trace(ctypes.c_void_p(tr.data_ptr()))
ws.gemm_tn(a, b, c)
torch.cuda.synchronize()
lib.ws_debug_gemm_trace(None)
j = trace.gemm_trace_json(tr)
json.dump(j, open("gpurun_out/trace_gemm_k2048.json", "w"), indent=1)
print("gemm K=2048:", j["summary"])
q = torch.randn(4, 16, 4096, 128, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
t2 = torch.zeros(3 * 256 * 8, dtype=torch.int64, device="cuda")
for _ in range(2):
    ws.attn_fwd(q, k, v)
ws.attn_fwd(q, k, v, trace=t2)
torch.cuda.synchronize()
j2 = trace.attn_trace_json(t2)
json.dump(j2, open("gpurun_out/trace_attn_s4k.json", "w"))
print("attention S=4K:", j2["summary"])
