"""The `.k` front end (ws_run_kernel / paper_2510_14719_b200.run_kernel): kernels written in the
reference grammar run on the B200 path and must reproduce the reference interpreter.

CPU tests cover the front end's rejections (they happen before any CUDA call). GPU tests run the
gemm.k-family goldens produced by the reference's own interpret_sequential (tests/golden/, see
make_golden.py) and compare EXACTLY: integer payloads and k/4 reals are exact in bf16 and every
partial sum is exact in fp32, so the tensor-core result equals the reference's int64 / double one.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from oracle import kernels as K

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _status(ws, text, buffers=(), lo=0, hi=1):
    lib = ws._lib.load()
    arr = (ws._lib.KBuffer * max(1, len(buffers)))(*buffers)
    st = lib.ws_run_kernel(text.encode(), arr, len(buffers), lo, hi, ws._lib.WS_BF16, None)
    return ws._lib.STATUS_NAMES[st], lib.ws_last_error().decode()


@pytest.mark.parametrize("text,code", [
    ("kernel x(a: buf<2x2 int>) {\n  %z = bogus 3\n}\n", "parse"),
    ("kernel x(a: buf<2x2 int>) {\n  %z = const zeros : 2x2 int\n", "parse"),           # not closed
    ("kernel x(a: buf<2x2 int>) {\n  yield %a\n}\n", "parse"),                          # yield outside loop
    ("kernel x(a: buf<2xq int>) {\n}\n", "parse"),
    ("kernel x(a: buf<2x2 float>) {\n}\n", "parse"),                                    # element kind
])
def test_grammar_errors(ws, text, code):
    assert _status(ws, text)[0] == code


def test_attention_toy_is_not_flash(ws):
    """The shipped integer attention.k computes a max-shift, not softmax attention: the
    front end refuses it instead of running something else."""
    toy = ("kernel attention(q: buf<32x8 int>, kt: buf<8x64 int>, v: buf<64x8 int>, o: buf<32x8 int>) {\n"
           "  %p = pid\n  %r = mul %p, 8\n  %zs = const zeros : 8x8 int\n  %zacc = const zeros : 8x8 int\n"
           "  %k0 = const 0\n  loop %k in 0..8 iter (%acc = %zacc, %ok = %k0) {\n"
           "    %tq = tma_load q[%r, 0] : 8x8 int\n    %tk = tma_load kt[0, %ok] : 8x8 int\n"
           "    %tv = tma_load v[%ok, 0] : 8x8 int\n    %s = dot %tq, %tk.T, acc=%zs\n"
           "    %m = reduce max %s axis=1\n    %sub = ew sub %s, %m\n    %acc1 = dot %sub, %tv, acc=%acc\n"
           "    %ok1 = add %ok, 8\n    yield %acc1, %ok1\n  }\n  store o[%r, 0] = %acc\n}\n")
    assert _status(ws, toy)[0] == "unsupported-kernel"


def test_small_flash_is_refused_not_faked(ws):
    code, msg = _status(ws, K.flash_src(3, 64, 16, 16, causal=False))
    assert code == "unsupported-kernel" and "S % 128" in msg


def test_buffer_shape_mismatch(ws):
    a = np.zeros((4, 4))
    b = ws._lib.KBuffer(name=b"a", rows=4, cols=4, is_real=1, data=a.ctypes.data)
    assert _status(ws, K.gemm_src(8, 8, 8, 8, 8, 8), [b])[0] == "eval"


# ---------------------------------------------------------------------------------------------
gpu = pytest.mark.gpu


@gpu
@pytest.mark.parametrize("name", ["gemm_real_64x48x96", "gemm_real_128x128x256", "gemm_real_scaled_64x64x128",
                                  "gemm_int_32x32x32", "gemm_int_seed7_16x16x24", "gemm_batched_int_4x16x16",
                                  "gemm_act_int_32x32x32", "gemm_large_int_32x32x32", "gemm_act_real_64x64x64"])
def test_golden_gemm_family_exact(ws, dev, name):
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    text = str(g["kernel"])
    bufs = {"a": g["in_a"].copy(), "b": g["in_b"].copy(), "c": np.zeros_like(g["out_c"])}
    ws.run_kernel(text, bufs, pid_range=(0, int(g["pids"])))
    assert np.array_equal(bufs["c"], g["out_c"]), name


@gpu
def test_pid_range_stores_only_its_tiles(ws, dev):
    """A pid range (a multi-GPU shard) writes exactly its tiles; other buffer contents stay."""
    M = N = 512
    Kd = 256
    src = K.gemm_src(M, N, Kd, 128, 256, 64)
    a = oracle.generate_real("a", (M, Kd))
    b = oracle.generate_real("b", (N, Kd))
    c = np.full((M, N), -7.0)
    ws.run_kernel(src, {"a": a, "b": b, "c": c}, pid_range=(4, 8))  # pn = 1: columns 256..511
    want = oracle.gemm(a, b)
    assert np.array_equal(c[:, 256:], want[:, 256:])
    assert (c[:, :256] == -7.0).all()


@gpu
def test_large_gemm_k_matches_oracle(ws, dev):
    M, N, Kd = 1024, 768, 2048
    src = K.gemm_src(M, N, Kd, 128, 256, 64)
    a = oracle.generate_real("a", (M, Kd))
    b = oracle.generate_real("b", (N, Kd))
    out = ws.run_kernel(src, {"a": a, "b": b}, pid_range=(0, K.gemm_tiles(M, N, 128, 256)))
    assert np.array_equal(out["c"], oracle.gemm(a, b))


@gpu
@pytest.mark.parametrize("causal", [False, True])
def test_flash_k_on_gpu(ws, dev, causal):
    """The flash .k of SURVEY Appendix A through the front end: o/lsum and mx + log(lsum) match the
    oracle within the attention tolerances."""
    BH, S, D, BR = 2, 512, 128, 64
    src = K.flash_src(BH, S, D, BR, causal)
    q = oracle.generate_real("q", (BH * S, D)) / 4
    k = oracle.generate_real("k", (BH * S, D)) / 4
    v = oracle.generate_real("v", (BH * S, D))
    bufs = {"q": q, "k": k, "v": v, "mb": K.flash_mask_bank(BR)}
    out = ws.run_kernel(src, bufs, pid_range=(0, BH * S // BR))
    ro, rl = oracle.flash(q.reshape(BH, S, D), k.reshape(BH, S, D), v.reshape(BH, S, D), causal)
    o = (out["o"] / out["lsum"]).reshape(BH, S, D)
    lse = (out["mx"] + np.log(out["lsum"])).reshape(BH, S)
    assert np.abs(o - ro).max() / np.abs(ro).max() <= 1e-2
    assert np.abs(lse - rl).max() <= 1e-3
