"""Per-tile time of the GEMM at tiny K (developer script): isolates epilogue / tile-transition cost.
cycles per tile round = kernel time x SM clock / ceil(tiles / resident tile slots)."""
import math, os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, pynvml
import paper_2510_14719_b200 as ws
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
M = N = 8192
for K in (64, 128, 256, 512, 1024):
    a = torch.randn(M, K, device="cuda").bfloat16(); b = torch.randn(N, K, device="cuda").bfloat16()
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for cfg, tile, slots in (({"cta_pair": False, "bn": 256}, 128 * 256, 148), ({"cta_pair": True, "bn": 256}, 256 * 256, 74),
                             ({"cta_pair": True, "bn": 512}, 256 * 512, 74)):
        fn = lambda: ws.gemm_tn(a, b, c, **cfg)
        for _ in range(5): fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): fn()
        e1.record(); torch.cuda.synchronize()
        clk = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        ms = e0.elapsed_time(e1) / 50
        rounds = math.ceil(M * N / tile / slots)
        kb = K // 64
        ideal = kb * 4 * (tile // 256 // (2 if cfg["cta_pair"] else 1)) // 128 * 128  # MMA cycles per tile
        per = ms * 1e-3 * clk * 1e6 / rounds
        print(f"K={K:5d} {str(cfg):36s} {ms*1e3:8.1f} us  clk {clk} MHz  cycles/tile-round {per:8.0f}  mainloop ideal {kb*4*(256 if cfg['bn']==256 else 512)//2 if cfg['cta_pair'] else kb*4*128:6d}")
