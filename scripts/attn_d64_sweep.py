"""hdim-64 attention: K/V aref depth D x stagger, alternating rounds on one box (developer script).
  python scripts/attn_d64_sweep.py   (under gpurun)"""
import json, os, subprocess, sys

CODE = r'''
import sys, os, json, torch
sys.path.insert(0, os.getcwd())
import paper_2510_14719_b200 as ws
D = int(os.environ["SWEEP_D"])
res = {}
for causal in (True, False):
    q = torch.randn(1, 16, 16384, 64, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    o = torch.empty_like(q); lse = torch.empty(1, 16, 16384, device="cuda")
    for _ in range(3): ws.attn_fwd(q, k, v, causal=causal, out=o, lse=lse, D=D)
    torch.cuda.synchronize()
    best = 0
    for w in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): ws.attn_fwd(q, k, v, causal=causal, out=o, lse=lse, D=D)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        best = max(best, 4 * 16 * 16384 * 16384 * 64 / (2 if causal else 1) / ms / 1e9)
    res["causal" if causal else "noncausal"] = round(best, 1)
print(json.dumps(res))
'''
variants = [(d, s) for s in (1, 0) for d in (3, 4, 6, 8)]
allres = {v: [] for v in variants}
for r in range(int(os.environ.get("ROUNDS", "3"))):
    for d, s in variants:
        env = dict(os.environ, SWEEP_D=str(d), WS_ATTN_STAGGER=str(s))
        out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if line:
            allres[(d, s)].append(json.loads(line[0]))
        else:
            print(d, s, "FAILED", out.stderr[-300:])
for (d, s), rs in allres.items():
    if rs:
        print(f"D={d} stagger={s}", {k: max(x[k] for x in rs) for k in rs[0]})
