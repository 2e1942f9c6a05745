"""The `.k` front end (ws_run_kernel / paper_2510_14719_b200.run_kernel): kernels written in the
reference grammar run on the B200 path and must reproduce the reference interpreter.

CPU tests cover the front end's rejections (they happen before any CUDA call). GPU tests run the
gemm.k-family goldens produced by the reference's own interpret_sequential (tests/golden/, see
make_golden.py) and compare EXACTLY: integer payloads and k/4 reals are exact in bf16 and every
partial sum is exact in fp32, so the tensor-core result equals the reference's int64 / double one.
"""
from __future__ import annotations

import ctypes
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


def _spec_status(ws, text, d=0, p=0, mode="auto", coop=0, persistent=1):
    lib = ws._lib.load()
    rs = ws._lib.RunSpec(d=d, p=p, mode=ws._lib.MODES[mode], coop_wgs=coop, persistent=persistent)
    arr = (ws._lib.KBuffer * 1)()
    st = lib.ws_run_kernel_spec(text.encode(), arr, 0, 0, 0, ws._lib.WS_BF16, ctypes.byref(rs), None)
    return ws._lib.STATUS_NAMES[st], lib.ws_last_error().decode()


GEMM_K = K.gemm_src(64, 64, 64, 32, 32, 16)
ACT_K = K.gemm_act_src(64, 64, 64, 32, 32, 16, elem="real")
FLASH_K = K.flash_src(2, 256, 64, 64, causal=True)
ATTN_K = K.maxshift_src(32, 8, 64, 8)


@pytest.mark.parametrize("text,kw,code", [
    # compile_kernel's rejections, in its order (ref proj/include/warpspec/driver.hpp:116-189)
    (GEMM_K, dict(d=-1), "pipeline-infeasible"),                  # driver.hpp:117
    (GEMM_K, dict(p=-1), "pipeline-infeasible"),                  # driver.hpp:118
    (GEMM_K, dict(d=2, p=3), "pipeline-infeasible"),              # auto -> fine, P > D (pipeline.hpp:84-92)
    (GEMM_K, dict(d=2, p=3, mode="fine"), "pipeline-infeasible"),
    (GEMM_K, dict(d=2, mode="coarse"), "pipeline-infeasible"),    # no transform stage (pipeline.hpp:264-267)
    (ACT_K, dict(d=2, mode="fine"), "pipeline-infeasible"),       # not a pure dot chain (pipeline.hpp:57-75)
    (FLASH_K, dict(d=2, mode="fine"), "pipeline-infeasible"),
    (FLASH_K, dict(d=1, mode="coarse"), "pipeline-infeasible"),   # coarse needs D >= 2 (pipeline.hpp:309-315)
    (ATTN_K, dict(d=1, mode="coarse"), "pipeline-infeasible"),
    (GEMM_K, dict(coop=-1), "indivisible-tile"),                  # grid.hpp:26-27
    (K.gemm_src(48, 64, 64, 16, 32, 16), dict(coop=3), "indivisible-tile"),  # 16 rows / 3 WGs (grid.hpp:43-46)
    (GEMM_K, dict(mode="bogus"), None),
])
def test_runspec_rejections(ws, text, kw, code):
    """RunSpec through the .k path is rejected exactly as the reference's compile_kernel rejects it,
    before any device work (these run on a CPU host)."""
    if kw.get("mode") == "bogus":
        lib = ws._lib.load()
        rs = ws._lib.RunSpec(d=0, p=0, mode=9, coop_wgs=0, persistent=1)
        arr = (ws._lib.KBuffer * 1)()
        assert ws._lib.STATUS_NAMES[lib.ws_run_kernel_spec(GEMM_K.encode(), arr, 0, 0, 1, ws._lib.WS_BF16,
                                                          ctypes.byref(rs), None)] == "parse"
        return
    assert _spec_status(ws, text, **kw)[0] == code


def test_runspec_feasible_specs_pass_validation(ws):
    """The specs the reference accepts pass the front end's checks (0 pids: no device work): auto with
    D = 1 on the flash kernel degrades to plain warp specialization (driver.hpp:137-150), none works
    on any kernel, coop 2 divides 32-row tiles."""
    for text, kw in [(FLASH_K, dict(d=1)), (FLASH_K, dict(mode="none")), (GEMM_K, dict(d=2, p=2, mode="fine")),
                     (GEMM_K, dict(d=3, p=1)), (ACT_K, dict(d=2, mode="coarse")), (GEMM_K, dict(coop=2)),
                     (ATTN_K, dict(d=2))]:
        assert _spec_status(ws, text, **kw)[0] == "ok", (kw, _spec_status(ws, text, **kw))


def test_maxshift_inexact_payloads_are_refused(ws):
    """Int payloads whose shifted scores could leave fp16's exact integer range (|s - m| > 2048) are
    refused before any device work instead of being rounded."""
    src = K.maxshift_src(64, 16, 128, 16)
    q = oracle.generate_int("q", (64, 16))
    bufs = [ws._lib.KBuffer(name=b"q", rows=64, cols=16, is_real=0, data=q.ctypes.data)]
    kt = oracle.generate_int("kt", (16, 128))
    bufs.append(ws._lib.KBuffer(name=b"kt", rows=16, cols=128, is_real=0, data=kt.ctypes.data))
    code, msg = _status(ws, src, bufs, 0, 4)
    assert code == "unsupported-kernel" and "exact" in msg


def test_oracle_maxshift_matches_reference_golden():
    """The numpy restatement of the shipped attention.k equals the reference interpreter's output."""
    g = np.load(os.path.join(GOLDEN, "attention_shipped.npz"))
    assert np.array_equal(oracle.maxshift(g["in_q"], g["in_kt"], g["in_v"], 8), g["out_o"])


@pytest.mark.parametrize("name,causal", [("flash_bh2_s256_d64", False), ("flash_causal_bh2_s256_d64", True)])
def test_oracle_flash_stats_match_reference_golden(name, causal):
    """The oracle's (o, lse) plus its row max reproduce the flash .k's three stored buffers
    (acc, l, m) as the reference interpreter computes them."""
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    q, k, v = (g["in_" + x].reshape(2, 256, 64) for x in "qkv")
    o, lse = oracle.flash(q, k, v, causal, block=64)
    m = oracle.flash_stats(q, k, causal)
    l = np.exp(lse - m)
    assert np.array_equal(m.ravel(), g["out_mx"].ravel())
    assert np.allclose(l.ravel(), g["out_lsum"].ravel(), rtol=1e-12)
    assert np.allclose((o * l[..., None]).ravel(), g["out_o"].ravel(), rtol=1e-12, atol=1e-12 * np.abs(g["out_o"]).max())


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
    q3, k3, v3 = (x.reshape(BH, S, D) for x in (q, k, v))
    ro, rl = oracle.flash(q3, k3, v3, causal)
    rm = oracle.flash_stats(q3, k3, causal)
    _check_flash_buffers(out, ro, rl, rm, BH, S, D)


def _check_flash_buffers(out, ro, rl, rm, BH, S, D):
    """All three .k buffers against the oracle: m (the running max) to fp32 rounding, l (row sums)
    to 1e-3, acc (un-normalised) to 1e-2 of its largest entry; and the derived o = acc/l,
    lse = m + log l at the north-star bars."""
    rlsum = np.exp(rl - rm)
    racc = ro * rlsum[..., None]
    m = out["mx"].reshape(BH, S)
    l = out["lsum"].reshape(BH, S)
    acc = out["o"].reshape(BH, S, D)
    assert np.abs(m - rm).max() <= 1e-5 * max(1.0, np.abs(rm).max())
    assert np.abs(l - rlsum).max() / np.abs(rlsum).max() <= 1e-3
    assert (np.abs(l - rlsum) / rlsum).max() <= 1e-3
    assert np.abs(acc - racc).max() / np.abs(racc).max() <= 1e-2
    assert np.abs(acc / l[..., None] - ro).max() / np.abs(ro).max() <= 1e-2
    assert np.abs(m + np.log(l) - rl).max() <= 1e-3


@gpu
@pytest.mark.parametrize("name,causal", [("flash_bh2_s256_d64", False), ("flash_causal_bh2_s256_d64", True)])
def test_golden_flash_k_all_buffers(ws, dev, name, causal):
    """The reference interpreter's own flash outputs (acc, l, m) reproduced by the GPU front end."""
    g = np.load(os.path.join(GOLDEN, name + ".npz"))
    bufs = {x: g["in_" + x].copy() for x in ("q", "k", "v", "mb")}
    out = ws.run_kernel(str(g["kernel"]), bufs, pid_range=(0, int(g["pids"])))
    gm, gl, go = g["out_mx"].reshape(2, 256), g["out_lsum"].reshape(2, 256), g["out_o"].reshape(2, 256, 64)
    _check_flash_buffers(out, go / gl[..., None], gm + np.log(gl), gm, 2, 256, 64)


@gpu
def test_golden_attention_k_exact(ws, dev):
    """The shipped integer attention.k (ref proj/kernels/attention.k) on the tensor cores, exactly."""
    g = np.load(os.path.join(GOLDEN, "attention_shipped.npz"))
    bufs = {x: g["in_" + x].copy() for x in ("q", "kt", "v")}
    out = ws.run_kernel(str(g["kernel"]), bufs, pid_range=(0, int(g["pids"])))
    assert np.array_equal(out["o"], g["out_o"])


@gpu
@pytest.mark.parametrize("R,D,S,BR,lo,hi", [(1024, 8, 1024, 8, 0, 128), (256, 8, 512, 16, 3, 7)])
def test_maxshift_k_larger_exact(ws, dev, R, D, S, BR, lo, hi):
    """Max-shift attention at larger sizes and a pid sub-range: exact vs the int64 restatement
    (head width 8 as shipped: the shift bound 2*9*9*8 = 1296 keeps s - m exact in fp16)."""
    src = K.maxshift_src(R, D, S, BR)
    q = oracle.generate_int("q", (R, D))
    kt = oracle.generate_int("kt", (D, S))
    v = oracle.generate_int("v", (S, D))
    o = np.full((R, D), 12345, dtype=np.int64)
    ws.run_kernel(src, {"q": q, "kt": kt, "v": v, "o": o}, pid_range=(lo, hi))
    want = oracle.maxshift(q, kt, v, D)
    assert np.array_equal(o[lo * BR:hi * BR], want[lo * BR:hi * BR])
    assert (o[:lo * BR] == 12345).all() and (o[hi * BR:] == 12345).all()


@gpu
@pytest.mark.parametrize("spec", [dict(d=2, p=1), dict(d=4, p=2, mode="fine"), dict(mode="none"),
                                  dict(d=3, coop=1, persistent=0), dict(d=2, coop=2, persistent=1)])
def test_runspec_gemm_k_exact(ws, dev, spec):
    """Every feasible RunSpec runs the gemm.k on the GPU with the reference's bit-exact result."""
    M, N, Kd = 512, 512, 1024
    src = K.gemm_src(M, N, Kd, 128, 128, 64)
    a = oracle.generate_real("a", (M, Kd))
    b = oracle.generate_real("b", (N, Kd))
    out = ws.run_kernel(src, {"a": a, "b": b}, pid_range=(0, K.gemm_tiles(M, N, 128, 128)), spec=spec)
    assert np.array_equal(out["c"], oracle.gemm(a, b))


@gpu
@pytest.mark.parametrize("spec", [dict(d=1), dict(mode="none"), dict(d=3, mode="coarse", persistent=0)])
def test_runspec_flash_k(ws, dev, spec):
    BH, S, D, BR = 2, 256, 64, 64
    src = K.flash_src(BH, S, D, BR, True)
    q = oracle.generate_real("q", (BH * S, D)) / 4
    k = oracle.generate_real("k", (BH * S, D)) / 4
    v = oracle.generate_real("v", (BH * S, D))
    out = ws.run_kernel(src, {"q": q, "k": k, "v": v, "mb": K.flash_mask_bank(BR)}, pid_range=(0, BH * S // BR),
                        spec=spec)
    q3, k3, v3 = (x.reshape(BH, S, D) for x in (q, k, v))
    ro, rl = oracle.flash(q3, k3, v3, True)
    _check_flash_buffers(out, ro, rl, oracle.flash_stats(q3, k3, True), BH, S, D)
