"""Item-boundary timeline of the persistent P-in-smem FA kernel (CTA 0, ws_attn_fwd_traced): per
global block step, how long the step took and how long the softmax of tile 0 waited for S —
separately for the first step of an item and the rest (developer script, run under gpurun)."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws

for (B, S) in ((16, 1024), (4, 4096), (1, 16384)):
    q = torch.randn(B, 16, S, 128, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    tr = torch.zeros(3 * 256 * 8, dtype=torch.int64, device="cuda")
    for _ in range(3):
        ws.attn_fwd(q, k, v, trace=tr)
    torch.cuda.synchronize()
    t = tr.view(3, 256, 8).cpu().long()
    nb = S // 128
    steps = [g for g in range(1, 255) if t[1, g, 1] > 0 and t[1, g + 1, 1] > 0]
    first = [g for g in steps if g % nb == 0]
    rest = [g for g in steps if g % nb != 0]
    dur = lambda g: int(t[1, g + 1, 1] - t[1, g, 1])     # softmax-0 S-arrival to next S-arrival
    wait = lambda g: int(t[1, g, 1] - t[1, g, 0])        # softmax-0 waiting for S
    epi = lambda g: int(t[1, g, 0] - t[1, g - 1, 5])     # gap before the wait (the epilogue when g % nb == 0)
    last = [g - 1 for g in first]
    ep_ld = statistics.median(int(t[1, g, 6] - t[1, g, 5]) for g in last) if last else "-"
    ep_st = statistics.median(int(t[1, g, 7] - t[1, g, 6]) for g in last) if last else "-"
    print(f"  epilogue: last p_full -> O in registers {ep_ld}, -> staged + TMA issued {ep_st}")
    print(f"S={S} B={B}: steps/item {nb}; first-step of item: period {statistics.median(dur(g - 1) for g in first) if first else '-'} "
          f"wait {statistics.median(wait(g) for g in first) if first else '-'} gap {statistics.median(epi(g) for g in first) if first else '-'}; "
          f"other steps: period {statistics.median(dur(g) for g in rest)} wait {statistics.median(wait(g) for g in rest)} "
          f"gap {statistics.median(epi(g) for g in rest)}")
