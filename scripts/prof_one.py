"""Launch one hot-path kernel a few times (for ncu captures under gpurun)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws

ap = argparse.ArgumentParser()
ap.add_argument("what", choices=["gemm", "gemm_fp8", "attn", "attn_causal", "attn_causal64", "attn_fp8"])
ap.add_argument("--K", type=int, default=16384)
ap.add_argument("--N", type=int, default=8192)  # gemm: an N-column shard (strong scaling) when < 8192
ap.add_argument("--n", type=int, default=3)
ap.add_argument("--bn", type=int, default=0)
ap.add_argument("--D", type=int, default=0)
ap.add_argument("--P", type=int, default=0)
ap.add_argument("--cta_pair", action="store_true")
ap.add_argument("--kvb", type=int, default=0)
a = ap.parse_args()
dev = torch.device("cuda")
if a.what.startswith("gemm"):
    dt = torch.float8_e4m3fn if a.what == "gemm_fp8" else torch.bfloat16
    A = torch.randn(8192, a.K, device=dev).to(dt); B = torch.randn(a.N, a.K, device=dev).to(dt)
    C = torch.empty(8192, a.N, device=dev, dtype=torch.bfloat16)
    for _ in range(a.n):
        ws.gemm_tn(A, B, C, bn=a.bn, D=a.D, P=a.P, cta_pair=a.cta_pair)
else:
    Dh = 64 if a.what == "attn_causal64" else 128
    dt = torch.float8_e4m3fn if a.what == "attn_fp8" else torch.bfloat16
    q = torch.randn(1, 16, 16384, Dh, device=dev).to(dt); k = torch.randn(1, 16, 16384, Dh, device=dev).to(dt)
    v = torch.randn(1, 16, 16384, Dh, device=dev).to(dt)
    for _ in range(a.n):
        ws.attn_fwd(q, k, v, causal=a.what not in ("attn", "attn_fp8"), D=a.D, kv_block=a.kvb)
torch.cuda.synchronize()
print("done", a)
