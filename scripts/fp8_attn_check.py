"""FP8 attention: error vs the fp64 oracle (sampled blocks) and timing at S = 16K (context for the
P-precision choice; run under gpurun)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2510_14719_b200 as ws  # noqa: E402
from tests.gpu_helpers import as_f64, ref_tensor, rel_err  # noqa: E402

dev = torch.device("cuda", 0)
for causal in (False, True):
    for qk_div in (4.0, 1.0):
        B, H, S, Dh = 1, 16, 16384, 128
        q = ref_tensor("q", (B, H, S, Dh), torch.float32, dev, div=qk_div)
        k = ref_tensor("k", (B, H, S, Dh), torch.float32, dev, div=qk_div)
        v = ref_tensor("v", (B, H, S, Dh), torch.float32, dev)
        q8, k8, v8 = (x.to(torch.float8_e4m3fn) for x in (q, k, v))
        o, lse = ws.attn_fwd(q8, k8, v8, causal=causal)
        torch.cuda.synchronize()
        errs = []
        for bh, qb in [(0, 0), (3, 64), (15, 127)]:
            ro, rl = oracle.flash(as_f64(q[0, bh:bh + 1]), as_f64(k[0, bh:bh + 1]), as_f64(v[0, bh:bh + 1]), causal,
                                  pid_range=(qb, qb + 1))
            rows = slice(qb * 128, (qb + 1) * 128)
            errs.append(rel_err(as_f64(o[0, bh, rows]), ro[0, rows]))
        qr, kr, vr = (torch.randn(B, H, S, Dh, device=dev).to(torch.float8_e4m3fn) for _ in range(3))
        for _ in range(3):
            ws.attn_fwd(qr, kr, vr, causal=causal)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ws.attn_fwd(qr, kr, vr, causal=causal)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        fl = 4.0 * B * H * S * S * Dh / (2 if causal else 1)
        print(f"fp8 causal={causal} qk_div={qk_div}: max rel err {max(errs):.2e}, {fl / ms / 1e9:.1f} TFLOP/s")
