"""Parity at the sizes the bench reports (BASELINE.json configs C3, C4 and the FP8 attention row),
against the CPU oracle on sampled rows / query blocks plus size-independent identities over the
whole output:

  C3  FP8 e4m3 GEMM M = N = 8192, K in {256, 2048, 16384}, per-tensor scales, bf16 out (the bench's
      call): sampled rows <= 5e-2 (north star FP8 bar); fp32 out: sampled rows BIT-EXACT and the
      row-sum identity sum_n c[m,n] = a[m,:] . sum_n b[n,:] exact on every row.
  C4  non-causal hdim 128, H = 16, S in {1K, 2K, 8K, 16K} with B*S = 16K: sampled query blocks of
      the first / a middle / the last (b,h) slice <= 1e-2, LSE <= 1e-3; O(V = 1) = 1 everywhere.
  FP8 attention hdim 128, S = 16K, causal and not: sampled blocks O <= 5e-2, LSE <= 1e-3.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from tests.gpu_helpers import as_f64, ref_tensor, rel_err

pytestmark = pytest.mark.gpu

BF16, E4M3, F32 = torch.bfloat16, torch.float8_e4m3fn, torch.float32


@pytest.mark.parametrize("K", [256, 2048, 16384])
def test_c3_fp8_gemm_8192_sampled(ws, dev, K):
    M = N = 8192
    a = ref_tensor("a", (M, K), E4M3, dev)
    b = ref_tensor("b", (N, K), E4M3, dev)
    sa, sb = 0.5, 2.0 ** -3
    rows = np.array([0, 255, 256, 4095, 4096, 8191] + list(np.random.default_rng(K).integers(0, M, 4)))
    ah = oracle.generate_real("a", (M, K))[rows]  # = ref_tensor's values (k/4)
    bh = oracle.generate_real("b", (N, K))
    c = ws.gemm_tn(a, b, scale_a=sa, scale_b=sb)  # the bench's call: bf16 out
    torch.cuda.synchronize()
    assert c.dtype == BF16
    want = oracle.gemm(ah, bh, scale=sa * sb)
    assert rel_err(as_f64(c[torch.from_numpy(rows).to(dev)]), want) <= 5e-2
    c32 = ws.gemm_tn(a, b, out_dtype=F32, scale_a=sa, scale_b=sb)
    torch.cuda.synchronize()
    assert np.array_equal(as_f64(c32[torch.from_numpy(rows).to(dev)]), want)  # power-of-two scales: exact
    rowsum = c32.double().sum(1)
    assert torch.equal(rowsum, (a.double() @ b.double().sum(0)) * (sa * sb))


C4 = [(16, 1024), (8, 2048), (2, 8192), (1, 16384)]


@pytest.mark.parametrize("B,S", C4)
def test_c4_noncausal_sampled_blocks(ws, dev, B, S):
    H, Dh = 16, 128
    q = ref_tensor("q", (B, H, S, Dh), BF16, dev, div=4.0)
    k = ref_tensor("k", (B, H, S, Dh), BF16, dev, div=4.0)
    v = ref_tensor("v", (B, H, S, Dh), BF16, dev)
    o, lse = ws.attn_fwd(q, k, v, causal=False)
    torch.cuda.synchronize()
    nqb = S // 128
    for b, h, qb in [(0, 0, 0), (B // 2, 7, nqb // 2), (B - 1, 15, nqb - 1)]:
        ro, rl = oracle.flash(as_f64(q[b, h:h + 1]), as_f64(k[b, h:h + 1]), as_f64(v[b, h:h + 1]), False,
                              pid_range=(qb, qb + 1))
        rows = slice(qb * 128, (qb + 1) * 128)
        assert rel_err(as_f64(o[b, h, rows]), ro[0, rows]) <= 1e-2
        assert np.abs(as_f64(lse[b, h, rows]) - rl[0, rows]).max() <= 1e-3
    # size-independent: with V = 1 every row of O is sum(p) / l = 1
    o1, _ = ws.attn_fwd(q, k, torch.ones_like(v), causal=False)
    torch.cuda.synchronize()
    assert (o1.float() - 1).abs().max().item() <= 1e-2


@pytest.mark.parametrize("causal", [False, True])
def test_fp8_attention_16k_sampled_blocks(ws, dev, causal):
    B, H, S, Dh = 1, 16, 16384, 128
    q = ref_tensor("q", (B, H, S, Dh), F32, dev, div=4.0)
    k = ref_tensor("k", (B, H, S, Dh), F32, dev, div=4.0)
    v = ref_tensor("v", (B, H, S, Dh), F32, dev)
    sq, sk, sv = 0.5, 0.25, 2.0
    q8, k8, v8 = (q / sq).to(E4M3), (k / sk).to(E4M3), (v / sv).to(E4M3)
    o, lse = ws.attn_fwd(q8, k8, v8, causal=causal, scale_q=sq, scale_k=sk, scale_v=sv)
    torch.cuda.synchronize()
    nqb = S // 128
    qh, kh, vh = (as_f64(t[0]) for t in (q, k, v))
    for bh, qb in [(0, 0), (0, nqb - 1), (7, nqb // 2 + 1), (15, nqb - 1)]:
        ro, rl = oracle.flash(qh[bh:bh + 1], kh[bh:bh + 1], vh[bh:bh + 1], causal, pid_range=(qb, qb + 1))
        rows = slice(qb * 128, (qb + 1) * 128)
        assert rel_err(as_f64(o[0, bh, rows]), ro[0, rows]) <= 5e-2
        assert np.abs(as_f64(lse[0, bh, rows]) - rl[0, rows]).max() <= 1e-3
