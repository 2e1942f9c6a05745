"""Small launches of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck).
  compute-sanitizer --tool racecheck python scripts/sanitize.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws

dev = torch.device("cuda")
a = torch.randn(512, 1024, device=dev).bfloat16(); b = torch.randn(1024, 1024, device=dev).bfloat16()
for kw in ({"cta_pair": False}, {"cta_pair": True, "bn": 256}, {"cta_pair": True, "bn": 512}):
    ws.gemm_tn(a, b, **kw)
# several 256 x 512 tiles per CTA pair: the half-by-half accumulator hand-over and the
# early-release epilogue across tiles; and a batched launch
a2 = torch.randn(4096, 256, device=dev).bfloat16(); b2 = torch.randn(8192, 256, device=dev).bfloat16()
ws.gemm_tn(a2, b2, cta_pair=True, bn=512)
ws.gemm_tn(a2.view(2, 2048, 256), b2.view(2, 4096, 256), cta_pair=True, bn=512)
a8, b8 = a.to(torch.float8_e4m3fn), b.to(torch.float8_e4m3fn)
ws.gemm_tn(a8, b8, cta_pair=True)
q = torch.randn(1, 2, 512, 128, device=dev).bfloat16(); k = torch.randn_like(q); v = torch.randn_like(q)
for causal in (False, True):
    ws.attn_fwd(q, k, v, causal=causal)
    if not os.environ.get("SKIP_KV64"):
        ws.attn_fwd(q, k, v, causal=causal, kv_block=64)
    ws.attn_fwd(q[..., :64].contiguous(), k[..., :64].contiguous(), v[..., :64].contiguous(), causal=causal)
    ws.attn_fwd(q.to(torch.float8_e4m3fn), k.to(torch.float8_e4m3fn), v.to(torch.float8_e4m3fn), causal=causal)
# persistent attention CTAs running more than one work item (256 items over 148 CTAs): the
# cross-item hand-overs (q_free, o_free, first QK of the next item) and, for FP8, the V converter
# warps' depth-2 ring across items
qm = torch.randn(1, 64, 1024, 128, device=dev).bfloat16(); km = torch.randn_like(qm); vm = torch.randn_like(qm)
for causal in (False, True):
    ws.attn_fwd(qm, km, vm, causal=causal)
    ws.attn_fwd(qm.to(torch.float8_e4m3fn), km.to(torch.float8_e4m3fn), vm.to(torch.float8_e4m3fn), causal=causal)
torch.cuda.synchronize()
print("sanitize workload done")
