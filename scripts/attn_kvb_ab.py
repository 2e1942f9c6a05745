"""hdim-64 attention: 128-key P-in-smem kernel (default) vs the 64-key S-double-buffered kernel
(kv_block=64), alternating rounds on one box (developer script, run under gpurun)."""
import os, sys, json, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws

res = {}
for Dh in (64, 128):
    for causal in (True, False):
        q = torch.randn(1, 16, 16384, Dh, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
        o = torch.empty_like(q); lse = torch.empty(1, 16, 16384, device="cuda")
        fl = 4 * 16 * 16384 * 16384 * Dh / (2 if causal else 1)
        for kvb in (0, 64):
            for _ in range(3): ws.attn_fwd(q, k, v, causal=causal, out=o, lse=lse, kv_block=kvb)
        torch.cuda.synchronize()
        acc = {0: [], 64: []}
        for r in range(6):
            for kvb in ((0, 64) if r % 2 == 0 else (64, 0)):
                e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10): ws.attn_fwd(q, k, v, causal=causal, out=o, lse=lse, kv_block=kvb)
                e1.record(); torch.cuda.synchronize()
                acc[kvb].append(fl / (e0.elapsed_time(e1) / 10 * 1e-3) / 1e12)
        res[f"d{Dh}_{'c' if causal else 'nc'}"] = {"kv128_psmem": round(statistics.median(acc[0]), 1),
                                                   "kv64": round(statistics.median(acc[64]), 1)}
print(json.dumps(res))
