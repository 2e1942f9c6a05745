"""Interleaved, clock-aware A/B of GEMM launch configurations (developer script, run under gpurun).

Each config runs back to back for SECS seconds per round (sustained, i.e. under the power cap the
bench also sees); rounds alternate configs. Reports TFLOP/s, the mean SM clock and power sampled by
NVML during the run, and TFLOP/s per GHz (per-clock efficiency).
  python scripts/gemm_ab.py K '{"cta_pair":1}' '{"cta_pair":1,"group_m":2}' ..."""
import json, os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
import paper_2510_14719_b200 as ws

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)


def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM), pynvml.nvmlDeviceGetPowerUsage(h) / 1000))
        time.sleep(0.02)


def run(fn, flop, secs):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    stop, samples = threading.Event(), []
    th = threading.Thread(target=sample, args=(stop, samples)); th.start()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    n, t0 = 0, time.time()
    e0.record()
    while time.time() - t0 < secs:
        for _ in range(10): fn()
        n += 10
        torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    stop.set(); th.join()
    ms = e0.elapsed_time(e1) / n
    half = samples[len(samples) // 3:] or samples
    clk = sum(s[0] for s in half) / len(half); pw = sum(s[1] for s in half) / len(half)
    return flop / ms / 1e9, clk, pw


K = int(sys.argv[1])
cfgs = [json.loads(c) for c in sys.argv[2:]]
M = N = int(os.environ.get("MN", "8192"))
dt = torch.float8_e4m3fn if os.environ.get("FP8") else torch.bfloat16
a = torch.randn(M, K, device="cuda").to(dt); b = torch.randn(N, K, device="cuda").to(dt)
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
secs = float(os.environ.get("SECS", "1.0"))
res = {i: [] for i in range(len(cfgs))}
for r in range(int(os.environ.get("ROUNDS", "3"))):
    for i, cfg in enumerate(cfgs):
        if cfg.get("cublas") and dt == torch.float8_e4m3fn:
            one = torch.ones((), device="cuda")  # cuBLASLt FP8 through torch._scaled_mm (per-tensor scales)
            fn = lambda one=one: torch._scaled_mm(a, b.T, one, one, out_dtype=torch.bfloat16, out=c)
        elif cfg.get("cublas"):
            fn = lambda: torch.matmul(a, b.T, out=c)
        else:
            fn = lambda cfg=cfg: ws.gemm_tn(a, b, c, **cfg)
        res[i].append(run(fn, 2 * M * N * K, secs))
        time.sleep(0.5)
for i, cfg in enumerate(cfgs):
    tf = [x[0] for x in res[i]]; ck = [x[1] for x in res[i]]; pw = [x[2] for x in res[i]]
    best = max(range(len(tf)), key=lambda j: tf[j])
    print(f"K={K} {json.dumps(cfg):45s} TFLOP/s max {max(tf):7.1f} mean {sum(tf)/len(tf):7.1f} | "
          f"SM MHz {sum(ck)/len(ck):6.0f} | W {sum(pw)/len(pw):5.0f} | TFLOP/s per GHz {1000*sum(tf)/sum(ck):6.1f}", flush=True)
