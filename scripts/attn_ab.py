"""Interleaved A/B timing of attention variants selected by environment knobs (developer script).

Each variant runs in a subprocess (the knobs are read once per process); rounds alternate so
clock/power drift hits every variant alike.
  python scripts/attn_ab.py 'WS_ATTN_PTMEM=1' 'WS_ATTN_PTMEM=0' ...
AB_FP8=1 runs the hdim-128 cases with e4m3 inputs; AB_SHORT=1 the C4 cases S = 1K / 2K / 4K."""
import json, os, subprocess, sys

CODE = r'''
import sys, os, json, torch
sys.path.insert(0, os.getcwd())
import paper_2510_14719_b200 as ws
res = {}
fp8 = os.environ.get("AB_FP8") == "1"
cases = [(1, 16384, 128, False), (1, 16384, 128, True), (16, 1024, 128, False), (1, 16384, 64, True), (1, 16384, 64, False)]
if os.environ.get("AB_SHORT") == "1":  # the C4 short-sequence cases
    cases = [(16, 1024, 128, False), (8, 2048, 128, False), (4, 4096, 128, False)]
if os.environ.get("AB_D64") == "1":  # the hdim-64 cases only
    cases = [(1, 16384, 64, True), (1, 16384, 64, False)]
for (B, S, Dh, causal) in (cases[:3] if fp8 else cases):
    q = torch.randn(B, 16, S, Dh, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
    o = torch.empty_like(q); lse = torch.empty(B, 16, S, device="cuda")
    if fp8:
        q, k, v = (t.to(torch.float8_e4m3fn) for t in (q, k, v))
    for _ in range(3): ws.attn_fwd(q, k, v, causal=causal, out=o, lse=lse)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): ws.attn_fwd(q, k, v, causal=causal, out=o, lse=lse)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res[f"S{S}_d{Dh}_{'c' if causal else 'nc'}_b{B}"] = round(4 * B * 16 * S * S * Dh / (2 if causal else 1) / ms / 1e9, 1)
print(json.dumps(res))
'''

variants = sys.argv[1:] or ["WS_ATTN_PTMEM=1", "WS_ATTN_PTMEM=0"]
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
    if not rs: continue
    keys = rs[0].keys()
    stat = os.environ.get("AB_STAT", "max")  # max (default) or median over rounds
    agg = (lambda xs: sorted(xs)[len(xs) // 2]) if stat == "median" else max
    print(f"{v:40s}", {k: agg([r[k] for r in rs]) for k in keys})
