"""Pin the CPU oracle (oracle/ws_oracle.c) to the reference.

1. Golden vectors produced by the reference's own interpreter (tests/golden/*.npz, made by
   tests/golden/make_golden.py from oracle/_ref/libwsref.so).
2. The reference's known-answer tests for this path, restated:
     1x1 product 2*3 = 6                          ref proj/tests/test_ir.cpp:120-141
     brute-force triple loop, 2x2 tiles, trip 2   ref proj/tests/test_ir.cpp:143-156
     all shapes <= 4x4, trip <= 4 vs element loop ref proj/tests/test_ir.cpp:183-202
3. Live comparison against oracle/_ref where it has been built (skipped otherwise).
"""
from __future__ import annotations

import glob
import os

import numpy as np
import pytest

import oracle
from oracle import kernels as K

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def test_golden_files_present():
    assert len(glob.glob(os.path.join(GOLDEN, "*.npz"))) >= 9


@pytest.mark.parametrize("name", ["gemm_real_64x48x96", "gemm_real_128x128x256", "gemm_real_scaled_64x64x128"])
def test_gemm_real_matches_reference_golden(name):
    g = _golden(name)
    seed = int(g["seed"])
    a, b = g["in_a"], g["in_b"]
    # the restated generator reproduces the reference's generate_inputs bit for bit
    assert np.array_equal(oracle.generate_real("a", a.shape, seed), a)
    assert np.array_equal(oracle.generate_real("b", b.shape, seed), b)
    scale = 0.25 if "scaled" in name else 1.0
    c = oracle.gemm(a, b, scale=scale, threads=2)
    assert np.array_equal(c, g["out_c"])  # bit-exact, same summation order


@pytest.mark.parametrize("name", ["gemm_int_32x32x32", "gemm_int_seed7_16x16x24"])
def test_gemm_int_matches_reference_golden(name):
    g = _golden(name)
    seed = int(g["seed"])
    a, b = g["in_a"], g["in_b"]
    assert np.array_equal(oracle.generate_int("a", a.shape, seed), a)
    assert np.array_equal(oracle.gemm_int(a, b), g["out_c"])


@pytest.mark.parametrize("name", ["flash_bh3_s64_d16", "flash_causal_bh3_s64_d16", "flash_bh2_s128_d32",
                                  "flash_causal_bh2_s128_d32"])
def test_flash_matches_reference_golden(name):
    g = _golden(name)
    causal = "causal" in name
    src = str(g["kernel"])
    BH = int(name.split("_bh")[1].split("_")[0])
    S = int(name.split("_s")[1].split("_")[0])
    D = int(name.split("_d")[1])
    BR = int(g["in_mb"].shape[0])
    q, k, v = (g[f"in_{n}"].reshape(BH, S, D) for n in "qkv")
    assert np.array_equal(oracle.generate_real("q", (BH * S, D)).reshape(BH, S, D), q)
    o, lse = oracle.flash(q, k, v, causal, block=BR, threads=2)
    want_o = (g["out_o"] / g["out_lsum"]).reshape(BH, S, D)  # harness step o = acc / l
    want_lse = (g["out_mx"] + np.log(g["out_lsum"])).reshape(BH, S)
    assert np.array_equal(o, want_o)
    assert np.array_equal(lse, want_lse)
    assert "flash" in src


def test_flash_against_dense_softmax():
    """Independent of the reference: the .k equals dense softmax attention."""
    rng = np.random.default_rng(0)
    BH, S, D = 2, 256, 32
    q, k, v = (rng.integers(-16, 17, (BH, S, D)) / 4.0 for _ in range(3))
    for causal in (False, True):
        o, lse = oracle.flash(q, k, v, causal, block=64, threads=2)
        s = np.einsum("bqd,bkd->bqk", q, k) / np.sqrt(D)
        if causal:
            s = np.where(np.triu(np.ones((S, S), bool), 1), -np.inf, s)
        m = s.max(-1, keepdims=True)
        p = np.exp(s - m)
        ref = p @ v / p.sum(-1, keepdims=True)
        assert np.abs(o - ref).max() / np.abs(ref).max() < 1e-12
        assert np.abs(lse - (m[..., 0] + np.log(p.sum(-1)))).max() < 1e-12


def test_flash_pid_range_is_a_shard():
    rng = np.random.default_rng(1)
    BH, S, D = 3, 128, 16
    q, k, v = (rng.integers(-16, 17, (BH, S, D)) / 4.0 for _ in range(3))
    full, _ = oracle.flash(q, k, v, True, block=32, threads=1)
    part, _ = oracle.flash(q, k, v, True, block=32, pid_range=(4, 8), threads=1)  # bh = 1
    assert np.array_equal(part[1], full[1])
    assert np.isnan(part[0]).all() and np.isnan(part[2]).all()


# ---- the reference's known-answer tests (integer payloads) ---------------------------------------
def test_known_answer_1x1():
    assert oracle.gemm_int(np.array([[2]]), np.array([[3]]))[0, 0] == 6


def test_known_answer_brute_force_2x2():
    a = oracle.generate_int("a", (2, 4), 7)
    b = oracle.generate_int("b", (2, 4), 7)
    c = oracle.gemm_int(a, b)
    for r in range(2):
        for n in range(2):
            assert c[r, n] == sum(int(a[r, i]) * int(b[n, i]) for i in range(4))


@pytest.mark.parametrize("m", [1, 2, 3, 4])
@pytest.mark.parametrize("kk", [1, 2, 4])
@pytest.mark.parametrize("trip", [1, 2, 4])
def test_known_answer_shapes(m, kk, trip):
    seed = 100 * m + 10 * kk + trip
    a = oracle.generate_int("a", (m, kk * trip), seed)
    b = oracle.generate_int("b", (m, kk * trip), seed)
    c = oracle.gemm_int(a, b)
    assert np.array_equal(c, a @ b.T)


def test_real_payloads_are_exact_in_device_types():
    """All 33 reference real values round-trip exactly through fp16, bf16 and e4m3."""
    torch = pytest.importorskip("torch")
    vals = torch.arange(-16, 17, dtype=torch.float64) / 4
    for dt in (torch.float16, torch.bfloat16, torch.float8_e4m3fn):
        assert torch.equal(vals.to(dt).to(torch.float64), vals)


def test_x4_generator_matches_real():
    r = oracle.generate_real("a", (64, 64))
    x4 = oracle.generate_real_x4("a", (64, 64))
    assert np.array_equal(x4.astype(np.float64) / 4, r)


# ---- live reference (where built) ------------------------------------------------------------------
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


@needs_ref
def test_live_reference_gemm_tiled():
    src = K.gemm_src(96, 64, 64, 32, 32, 16)
    rk = oracle.RefKernel(src)
    ins = rk.generate()
    out = rk.run(ins, 0, K.gemm_tiles(96, 64, 32, 32))
    assert np.array_equal(out["c"], oracle.gemm(ins["a"], ins["b"], threads=1))


@needs_ref
@pytest.mark.parametrize("causal", [False, True])
def test_live_reference_flash(causal):
    BH, S, D, BR = 2, 96, 8, 16
    rk = oracle.RefKernel(K.flash_src(BH, S, D, BR, causal))
    ins = rk.generate(99)
    ins["mb"] = K.flash_mask_bank(BR)
    out = rk.run(ins, 0, BH * S // BR)
    q, k, v = (ins[n].reshape(BH, S, D) for n in "qkv")
    o, lse = oracle.flash(q, k, v, causal, block=BR, threads=1)
    assert np.array_equal(o, (out["o"] / out["lsum"]).reshape(BH, S, D))
