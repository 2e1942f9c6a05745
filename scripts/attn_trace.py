"""Device timeline of one FA CTA (ws_attn_fwd_traced): per-step softmax stage durations and MMA waits."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws

def run(S=16384, Dh=128, causal=False, B=1, H=16):
    q = torch.randn(B, H, S, Dh, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    tr = torch.zeros(3 * 256 * 8, dtype=torch.int64, device="cuda")
    for _ in range(3):
        ws.attn_fwd(q, k, v, causal=causal, trace=tr)
    torch.cuda.synchronize()
    t = tr.view(3, 256, 8).cpu()
    n = min(S // 64, 256)
    base = int(t[0, 0, 0])
    print(f"S={S} Dh={Dh} causal={causal}: MMA-view cycles over {n} steps {int(t[0, n-1, 5]) - base}")
    per = []
    for j in range(2, min(n, 40)):
        m = t[0, j]; s0 = t[1, j]; s1 = t[2, j]
        row = dict(
            step=int(t[0, j, 0] - t[0, j - 1, 0]),
            mma_qk=int(m[1] - m[0]), mma_wait_p0=int(m[2] - m[1]), mma_pv0=int(m[3] - m[2]), mma_wait_p1=int(m[4] - m[3]),
            sm0_wait=int(s0[1] - s0[0]), sm0_ld=int(s0[2] - s0[1]), sm0_max=int(s0[3] - s0[2]), sm0_exp=int(s0[4] - s0[3]), sm0_arr=int(s0[5] - s0[4]),
            sm1_wait=int(s1[1] - s1[0]), sm1_ld=int(s1[2] - s1[1]), sm1_max=int(s1[3] - s1[2]), sm1_exp=int(s1[4] - s1[3]),
            sm0_start_vs_sm1=int(s0[1] - s1[1]))
        per.append(row)
        if j < 12: print(row)
    import statistics
    keys = per[0].keys()
    print("median:", {k: statistics.median(r[k] for r in per) for k in keys})

if __name__ == "__main__":
    run()
    run(S=4096, B=4)
    run(Dh=64, causal=True)
