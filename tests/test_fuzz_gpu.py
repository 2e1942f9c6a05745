"""Randomised launch-configuration sweeps (fixed seeds) against exact / oracle references.

GEMM: integer-valued operands (exact in bf16/fp16/e4m3) make the fp32 result exact for any
summation order, so every (shape, tile, depth, raster, persistence) combination must reproduce
torch's float64 product bit for bit. Attention: random shapes and knobs against the CPU oracle at
the north star's tolerances."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from tests.gpu_helpers import as_f64, rel_err

pytestmark = pytest.mark.gpu


def _int_tensor(gen, shape, lo, hi, dtype, dev):
    return torch.randint(lo, hi + 1, shape, generator=gen).to(torch.float32).to(dev).to(dtype)


@pytest.mark.parametrize("seed", range(12))
def test_gemm_random_configs_bit_exact(ws, dev, seed):
    rng = np.random.default_rng(seed)
    gen = torch.Generator().manual_seed(seed)
    for _ in range(8):
        dt = [torch.bfloat16, torch.float16, torch.float8_e4m3fn][rng.integers(3)]
        kstep = 128 if dt == torch.float8_e4m3fn else 64
        cta_pair = bool(rng.integers(2))
        bn = int(rng.choice([128, 256, 512] if cta_pair else [128, 256]))
        M = int(rng.integers(1, 7)) * (256 if cta_pair else 128)
        N = int(rng.integers(1, 5)) * bn
        K = int(rng.integers(1, 24)) * kstep
        D = int(rng.integers(0, 5))  # 0 = auto
        P = int(rng.integers(1, D + 1)) if D > 0 and rng.integers(2) else 0
        kw = dict(cta_pair=cta_pair, bn=bn, D=D, P=P, persistent=bool(rng.integers(2)),
                  group_m=int(rng.integers(0, 5)))
        a = _int_tensor(gen, (M, K), -3, 3, dt, dev)
        b = _int_tensor(gen, (N, K), -3, 3, dt, dev)
        try:
            c = ws.gemm_tn(a, b, out_dtype=torch.float32, **kw)
        except ws.WsError as e:
            assert e.code == "smem-overflow", (e, kw)  # D beyond what fits for the tile is refused
            continue
        torch.cuda.synchronize()
        want = a.double() @ b.double().T
        assert torch.equal(c.double(), want), (M, N, K, dt, kw)


@pytest.mark.parametrize("seed", range(8))
def test_attention_random_configs(ws, dev, seed):
    rng = np.random.default_rng(100 + seed)
    for _ in range(4):
        Dh = int(rng.choice([64, 128]))
        fp8 = Dh == 128 and bool(rng.integers(3) == 0)
        kv_block = 0 if fp8 else int(rng.choice([0, 64, 128]))
        B, H = int(rng.integers(1, 3)), int(rng.integers(1, 4))
        S = int(rng.integers(1, 5)) * 256
        causal = bool(rng.integers(2))
        D = int(rng.choice([0, 2, 3]))
        shape = (B, H, S, Dh)
        gen = torch.Generator().manual_seed(int(rng.integers(1 << 30)))
        q = (torch.randint(-16, 17, shape, generator=gen).float() / 16).to(dev)
        k = (torch.randint(-16, 17, shape, generator=gen).float() / 16).to(dev)
        v = (torch.randint(-16, 17, shape, generator=gen).float() / 4).to(dev)
        dt = torch.float8_e4m3fn if fp8 else torch.bfloat16
        o, lse = ws.attn_fwd(q.to(dt), k.to(dt), v.to(dt), causal=causal, kv_block=kv_block, D=D)
        torch.cuda.synchronize()
        qq, kk, vv = (as_f64(t.to(dt)).reshape(B * H, S, Dh) for t in (q, k, v))
        ro, rl = oracle.flash(qq, kk, vv, causal)
        got_o = as_f64(o).reshape(B * H, S, Dh)
        got_l = as_f64(lse).reshape(B * H, S)
        assert np.abs(got_l - rl).max() <= 1e-3, (shape, causal, kv_block, D, fp8)
        if fp8:
            assert np.abs(got_o - ro).max() <= np.abs(vv).max() / 16, (shape, causal, D)
        else:
            assert rel_err(got_o, ro) <= 1e-2, (shape, causal, kv_block, D)
