"""Quick GPU validation + timing of the attention path (developer script, run under gpurun)."""
import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws

def vals(shape, seed):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return ((torch.randint(0, 33, shape, generator=g).float() - 16.0) / 4.0).cuda()

def ref_attn(q, k, v, causal):
    qd, kd, vd = q.double(), k.double(), v.double()
    s = qd @ kd.transpose(-1, -2) / math.sqrt(q.shape[-1])
    if causal:
        S = q.shape[-2]
        mask = torch.triu(torch.ones(S, S, dtype=torch.bool, device=q.device), 1)
        s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, -1)
    return torch.softmax(s, -1) @ vd, lse

def check(B, H, S, Dh, causal, dt=torch.bfloat16, scale_in=1.0, **kw):
    q = (vals((B, H, S, Dh), 1) * scale_in).to(dt); k = (vals((B, H, S, Dh), 2) * scale_in).to(dt); v = vals((B, H, S, Dh), 3).to(dt)
    try:
        o, lse = ws.attn_fwd(q, k, v, causal=causal, **kw)
    except ws.WsError as e:
        print(f"B={B} H={H} S={S} Dh={Dh} causal={causal} {dt} {kw}: rejected ({e})", flush=True)
        return
    torch.cuda.synchronize()
    ro, rl = ref_attn(q, k, v, causal)
    rel = ((o.double() - ro).abs().max() / ro.abs().max()).item()
    le = (lse.double() - rl).abs().max().item()
    print(f"B={B} H={H} S={S} Dh={Dh} causal={causal} {dt} {kw}: O relerr={rel:.3e} lse abserr={le:.3e} nan={torch.isnan(o).any().item()}", flush=True)

def bench(B, H, S, Dh, causal, iters=10, dt=torch.bfloat16, **kw):
    q = torch.randn(B, H, S, Dh, device="cuda", dtype=dt); k = torch.randn_like(q); v = torch.randn_like(q)
    o = torch.empty_like(q); lse = torch.empty(B, H, S, device="cuda")
    for _ in range(3): ws.attn_fwd(q, k, v, causal=causal, out=o, lse=lse, **kw)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): ws.attn_fwd(q, k, v, causal=causal, out=o, lse=lse, **kw)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    fl = 4 * B * H * S * S * Dh / (2 if causal else 1)
    print(f"BENCH attn B={B} H={H} S={S} Dh={Dh} causal={causal} {kw}: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s", flush=True)

if __name__ == "__main__":
    torch.cuda.init()
    kvb = [int(x) for x in os.environ.get("KVB", "128,64").split(",")]
    for kb in kvb:
        check(1, 1, 256, 128, False, kv_block=kb)
        check(1, 2, 512, 128, False, kv_block=kb)
        check(1, 2, 512, 64, False, kv_block=kb)
        check(1, 2, 512, 128, True, kv_block=kb)
        check(1, 2, 512, 64, True, kv_block=kb)
        check(2, 3, 1024, 128, False, dt=torch.float16, kv_block=kb)
        check(1, 2, 1024, 128, True, scale_in=0.25, kv_block=kb)
        # several work items per CTA (the persistent kernels loop over items)
        check(4, 16, 2048, 128, False, kv_block=kb)
        check(4, 16, 2048, 128, True, kv_block=kb)
        check(2, 16, 2048, 64, True, kv_block=kb)
        for D in (2, 3, 4, 5):
            check(1, 2, 1024, 128, True, D=D, kv_block=kb)
            check(1, 2, 1024, 64, False, D=D, kv_block=kb)
    for kb in kvb:
        for S in (1024, 4096, 16384):
            bench(16384 // S, 16, S, 128, False, kv_block=kb)
        bench(1, 16, 16384, 128, True, kv_block=kb)
        bench(1, 16, 16384, 64, True, kv_block=kb)
        bench(1, 16, 16384, 64, False, kv_block=kb)
    try:
        from flash_attn import flash_attn_func
        q = torch.randn(1, 16384, 16, 128, device="cuda", dtype=torch.bfloat16); k = torch.randn_like(q); v = torch.randn_like(q)
        for c in (False, True):
            for _ in range(3): flash_attn_func(q, k, v, causal=c)
            torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True); e0.record()
            for _ in range(10): flash_attn_func(q, k, v, causal=c)
            e1.record(); torch.cuda.synchronize(); ms = e0.elapsed_time(e1)/10
            print(f"flash_attn lib S=16K causal={c}: {ms:.3f} ms {4*16*16384**2*128/(2 if c else 1)/ms/1e9:.1f} TFLOP/s")
    except Exception as e:
        print("flash_attn lib unavailable:", e)


def bench_fp8(B, H, S, causal, iters=10):
    q = torch.randn(B, H, S, 128, device="cuda").to(torch.float8_e4m3fn); k = torch.randn_like(q.float()).to(torch.float8_e4m3fn)
    v = torch.randn_like(q.float()).to(torch.float8_e4m3fn)
    o = torch.empty(B, H, S, 128, device="cuda", dtype=torch.bfloat16); lse = torch.empty(B, H, S, device="cuda")
    for _ in range(3): ws.attn_fwd(q, k, v, causal=causal, out=o, lse=lse)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): ws.attn_fwd(q, k, v, causal=causal, out=o, lse=lse)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    fl = 4 * B * H * S * S * 128 / (2 if causal else 1)
    print(f"BENCH fp8 attn B={B} H=16 S={S} causal={causal}: {ms:.3f} ms {fl/ms/1e9:.1f} TFLOP/s", flush=True)
