"""A/B of programmatic dependent launch for the GEMM (WS_PDL=0/1, read once per process) at short K,
next to cuBLAS, in alternating subprocess rounds on one box. Back-to-back launches of one shape
(the way a caller issues a sequence of GEMMs), 0.5 s per shape per round."""
import json, os, subprocess, sys

CODE = r'''
import sys, os, json, time, torch
sys.path.insert(0, os.getcwd())
import paper_2510_14719_b200 as ws
res = {}
for K in (256, 512, 1024, 2048):
    a = torch.randn(8192, K, device="cuda", dtype=torch.bfloat16); b = torch.randn(8192, K, device="cuda", dtype=torch.bfloat16)
    c = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
    for name, fn in (("ours", lambda: ws.gemm_tn(a, b, c)), ("cublas", lambda: torch.matmul(a, b.T, out=c))):
        if name == "cublas" and os.environ.get("WS_PDL") == "0":
            continue
        for _ in range(5): fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        n = 0; t0 = time.time(); e0.record()
        while time.time() - t0 < 0.5:
            for _ in range(20): fn()
            n += 20
            torch.cuda.synchronize()
        e1.record(); torch.cuda.synchronize()
        res[f"{name}_K{K}"] = round(2 * 8192 * 8192 * K / (e0.elapsed_time(e1) / n) / 1e9, 1)
print(json.dumps(res))
'''
variants = sys.argv[1:] or ["WS_PDL=0", "WS_PDL=1"]
rounds = int(os.environ.get("ROUNDS", "3"))
allres = {v: [] for v in variants}
for r in range(rounds):
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            k, val = kv.split("=")
            env[k] = val
        out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if not line:
            print(v, "FAILED", out.stderr[-500:]); continue
        allres[v].append(json.loads(line[0]))
for v, rs in allres.items():
    if rs:
        print(f"{v:12s}", {k: sorted(r[k] for r in rs)[len(rs) // 2] for k in rs[0]})
