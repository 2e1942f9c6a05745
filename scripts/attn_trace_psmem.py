"""Device timeline of one CTA of the P-in-shared-memory FA kernel (ws_attn_fwd_traced).

MMA events per step j: 0 start, 1 QK_0(j+1) issued, 2 QK_1(j+1) issued, 3 p_full[0] passed,
4 p_full[1] passed, 5 PV_1 issued, 6 K_{j+1} taken from the ring, 7 V_j taken from the ring. Softmax (tile t, warp 4t lane 0): 0 wait start, 1 S_t full,
2 S copied + s_free, 3 max (+ correction) done, 6 P tile free (PV_t(j-1) done), 4 exponentials done,
5 P stored + p_full."""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws


def run(S=16384, Dh=128, causal=False, B=1, H=16, D=0):
    q = torch.randn(B, H, S, Dh, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    tr = torch.zeros(3 * 256 * 8, dtype=torch.int64, device="cuda")
    for _ in range(3):
        ws.attn_fwd(q, k, v, causal=causal, trace=tr, kv_block=128, D=D)
    torch.cuda.synchronize()
    t = tr.view(3, 256, 8).cpu().long()
    n = min(S // 128, 256)
    per = []
    for j in range(2, n - 1):
        m, s0, s1 = t[0, j], t[1, j], t[2, j]
        per.append(dict(
            step=int(t[0, j + 1, 0] - m[0]), m_qk0=int(m[1] - m[0]), m_qk1=int(m[2] - m[1]), m_wp0=int(m[3] - m[2]),
            m_wp1=int(m[4] - m[3]), m_pv1=int(m[5] - m[4]), m_kwait=int(m[6] - m[0]), m_vwait=int(m[7] - m[2]),
            s0_wait=int(s0[1] - s0[0]), s0_ld=int(s0[2] - s0[1]), s0_max=int(s0[3] - s0[2]), s0_pfree=int(s0[6] - s0[3]),
            s0_exp=int(s0[4] - s0[6]),
            s0_st=int(s0[5] - s0[4]), s1_wait=int(s1[1] - s1[0]), s1_pfree=int(s1[6] - s1[3]), s1_exp=int(s1[4] - s1[6]), s1_st=int(s1[5] - s1[4]),
            s1_minus_s0=int(s1[1] - s0[1])))
    print(f"S={S} Dh={Dh} causal={causal} D={D} steps={len(per)}")
    print("  median:", {k: statistics.median(r[k] for r in per) for k in per[0]})


if __name__ == "__main__":
    run()
    run(D=2)
    run(Dh=64)
