"""The reference-side C++ binding (include/ws.hpp) in the reference's own flow: integration/dropin.cpp,
compiled against the unmodified reference headers (build container) into oracle/_ref/ws_dropin,
parses each `.k` with warpspec::parse_kernel, generates inputs with warpspec::generate_inputs, runs
every pid through warpspec::interpret_sequential AND through ws::run on the GPU, and compares the
Buffers maps (exact for the gemm.k family)."""
from __future__ import annotations

import os
import subprocess

import pytest

from oracle import kernels as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ws_dropin")


def test_dropin_binary_builds_here():
    """Build check (CPU): where the reference headers exist, the C++ binding compiles against them."""
    if not os.path.isdir("/root/reference/proj/include"):
        pytest.skip("reference headers are only present in the build container")
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "integration")])
    assert os.access(BIN, os.X_OK)


def _run(tmp_path, texts, *args):
    paths = []
    for i, t in enumerate(texts):
        p = tmp_path / f"k{i}.k"
        p.write_text(t)
        paths.append(str(p))
    out = subprocess.run([BIN, *paths, *args], capture_output=True, text=True, timeout=600)
    return out.returncode, out.stdout + out.stderr


@pytest.mark.gpu
def test_gemm_family_through_the_reference_flow(ws, dev, tmp_path):
    if not os.access(BIN, os.X_OK):
        pytest.skip("oracle/_ref/ws_dropin not built (needs the reference headers at build time)")
    texts = [K.gemm_src(256, 256, 512, 128, 128, 64),               # real gemm.k, 4 pids
             K.gemm_src(256, 256, 256, 128, 128, 64, elem="int"),    # the shipped integer form
             K.gemm_src(256, 512, 256, 128, 256, 64, scale=0.25)]    # scaled epilogue (FP8 form)
    rc, log = _run(tmp_path, texts, "--pids", "4")
    assert rc == 0, log
    assert log.count("PASS") == 3, log


@pytest.mark.gpu
@pytest.mark.parametrize("causal", [False, True])
def test_flash_through_the_reference_flow(ws, dev, tmp_path, causal):
    if not os.access(BIN, os.X_OK):
        pytest.skip("oracle/_ref/ws_dropin not built (needs the reference headers at build time)")
    # B*H = 2 slices of S = 256, hdim 64, 128-row blocks: 4 pids = everything
    rc, log = _run(tmp_path, [K.flash_src(2, 256, 64, 128, causal)], "--pids", "4", "--flash")
    assert rc == 0, log
    assert "PASS" in log, log
    # S = 384: three 128-row query blocks per slice (an odd count), 6 pids
    rc, log = _run(tmp_path, [K.flash_src(2, 384, 64, 128, causal)], "--pids", "6", "--flash")
    assert rc == 0, log
    assert "PASS" in log, log


def test_runspec_rejection_through_the_reference_flow(tmp_path):
    """The reference's own RunSpec with P > D, set on ws::Launch from a warpspec::RunSpec, is rejected
    by the GPU path with the reference's PipelineInfeasible before any device work (so this runs
    on a CPU host too), exactly as compile_kernel rejects it (ref pipeline.hpp:84-92)."""
    if not os.access(BIN, os.X_OK):
        pytest.skip("oracle/_ref/ws_dropin not built (needs the reference headers at build time)")
    rc, log = _run(tmp_path, [K.gemm_src(256, 256, 512, 128, 128, 64)], "--pids", "4", "--spec", "2,3,fine,1,0")
    assert rc == 1 and "REJECTED" in log and "pipeline-infeasible" in log, log
    rc, log = _run(tmp_path, [K.flash_src(2, 256, 64, 128, True)], "--pids", "4", "--flash", "--spec",
                   "1,1,coarse,1,0")
    assert rc == 1 and "pipeline-infeasible" in log, log


@pytest.mark.gpu
def test_attention_k_through_the_reference_flow(ws, dev, tmp_path):
    """The shipped integer attention.k (text from the reference-made golden): generate_inputs,
    interpret_tiles and ws::run agree exactly, also under the reference's default RunSpec."""
    if not os.access(BIN, os.X_OK):
        pytest.skip("oracle/_ref/ws_dropin not built (needs the reference headers at build time)")
    import numpy as np

    text = str(np.load(os.path.join(ROOT, "tests", "golden", "attention_shipped.npz"))["kernel"])
    rc, log = _run(tmp_path, [text], "--pids", "4")
    assert rc == 0 and "PASS" in log, log
    rc, log = _run(tmp_path, [text], "--pids", "4", "--spec", "2,1,auto,1,0")
    assert rc == 0 and "PASS" in log, log


@pytest.mark.gpu
def test_runspec_through_the_reference_flow(ws, dev, tmp_path):
    """Feasible reference RunSpecs (fine D=4 P=2 persistent, none, coarse flash D=3) give the same
    buffers as the reference interpreter."""
    if not os.access(BIN, os.X_OK):
        pytest.skip("oracle/_ref/ws_dropin not built (needs the reference headers at build time)")
    rc, log = _run(tmp_path, [K.gemm_src(256, 256, 512, 128, 128, 64)], "--pids", "4", "--spec", "4,2,fine,2,1")
    assert rc == 0 and "PASS" in log, log
    rc, log = _run(tmp_path, [K.gemm_src(256, 256, 512, 128, 128, 64)], "--pids", "4", "--spec", "1,1,none,1,0")
    assert rc == 0 and "PASS" in log, log
    rc, log = _run(tmp_path, [K.flash_src(2, 256, 64, 128, True)], "--pids", "4", "--flash", "--spec",
                   "3,1,coarse,1,0")
    assert rc == 0 and "PASS" in log, log


# The reference's own test-fixture kernels (ref proj/tests/support/fixtures.hpp:14-143), restated
# as text generators: the shapes its compiler/interpreter tests run, here through ws::run on the GPU
# against interpret_sequential in the reference's own flow (exact, integer payloads).
def _fx_gemm(m, n, kk, trip):  # fixtures.hpp:14-29
    return (f"kernel gemm(a: buf<{m}x{kk * trip} int>, b: buf<{n}x{kk * trip} int>, c: buf<{m}x{n} int>) {{\n"
            f"  %z = const zeros : {m}x{n} int\n  %k0 = const 0\n"
            f"  loop %k in 0..{trip} iter (%acc = %z, %ok = %k0) {{\n"
            f"    %ta = tma_load a[0, %ok] : {m}x{kk} int\n    %tb = tma_load b[0, %ok] : {n}x{kk} int\n"
            f"    %acc1 = dot %ta, %tb.T, acc=%acc\n    %ok1 = add %ok, {kk}\n    yield %acc1, %ok1\n  }}\n"
            f"  store c[0, 0] = %acc\n}}\n")


def _fx_attention(r, trip):  # fixtures.hpp:38-56 (r = 4, trip = 2) and :77-100
    return (f"kernel attn{trip}(q: buf<{r}x{r} int>, kt: buf<{r}x{r * trip} int>, v: buf<{r * trip}x{r} int>, "
            f"o: buf<{r}x{r} int>) {{\n"
            f"  %zs = const zeros : {r}x{r} int\n  %zacc = const zeros : {r}x{r} int\n  %k0 = const 0\n"
            f"  loop %k in 0..{trip} iter (%acc = %zacc, %ok = %k0) {{\n"
            f"    %tq = tma_load q[0, 0] : {r}x{r} int\n    %tk = tma_load kt[0, %ok] : {r}x{r} int\n"
            f"    %tv = tma_load v[%ok, 0] : {r}x{r} int\n    %s = dot %tq, %tk.T, acc=%zs\n"
            f"    %m = reduce max %s axis=1\n    %sub = ew sub %s, %m\n    %acc1 = dot %sub, %tv, acc=%acc\n"
            f"    %ok1 = add %ok, {r}\n    yield %acc1, %ok1\n  }}\n  store o[0, 0] = %acc\n}}\n")


def _fx_gemm_act(m, kk, trip):  # fixtures.hpp:59-75 (m = 4, kk = 4, trip = 2) and :103-121
    return (f"kernel gemm_act{trip}(a: buf<{m}x{kk * trip} int>, b: buf<{m}x{kk * trip} int>, c: buf<{m}x{m} int>) {{\n"
            f"  %z = const zeros : {m}x{m} int\n  %k0 = const 0\n"
            f"  loop %k in 0..{trip} iter (%acc = %z, %last = %z, %ok = %k0) {{\n"
            f"    %ta = tma_load a[0, %ok] : {m}x{kk} int\n    %tb = tma_load b[0, %ok] : {m}x{kk} int\n"
            f"    %acc1 = dot %ta, %tb.T, acc=%acc\n    %rl = ew relu %acc1\n    %ok1 = add %ok, {kk}\n"
            f"    yield %acc1, %rl, %ok1\n  }}\n  store c[0, 0] = %last\n}}\n")


def _fx_gemm_tiled(tm, tn, tr, tc, kk, trip):  # fixtures.hpp:123-143
    ra, rb, depth = tm * tr, tn * tc, kk * trip
    return (f"kernel gemm_tiled(a: buf<{ra}x{depth} int>, b: buf<{rb}x{depth} int>, c: buf<{ra}x{rb} int>) {{\n"
            f"  %p = pid\n  %pm = mod %p, {tm}\n  %pn = div %p, {tm}\n  %r = mul %pm, {tr}\n  %cn = mul %pn, {tc}\n"
            f"  %z = const zeros : {tr}x{tc} int\n  %k0 = const 0\n"
            f"  loop %k in 0..{trip} iter (%acc = %z, %ok = %k0) {{\n"
            f"    %ta = tma_load a[%r, %ok] : {tr}x{kk} int\n    %tb = tma_load b[%cn, %ok] : {tc}x{kk} int\n"
            f"    %acc1 = dot %ta, %tb.T, acc=%acc\n    %ok1 = add %ok, {kk}\n    yield %acc1, %ok1\n  }}\n"
            f"  store c[%r, %cn] = %acc\n}}\n")


def _fx_twochain(m, kk, trip):  # kernel_gen.hpp:55-78: two independent Gram chains a.a^T, b.b^T
    return (f"kernel twochain(a: buf<{m}x{kk * trip} int>, b: buf<{m}x{kk * trip} int>, c: buf<{m}x{m} int>, "
            f"d: buf<{m}x{m} int>) {{\n"
            f"  %z1 = const zeros : {m}x{m} int\n  %z2 = const zeros : {m}x{m} int\n  %k0 = const 0\n"
            f"  loop %k in 0..{trip} iter (%u = %z1, %v = %z2, %ok = %k0) {{\n"
            f"    %ta = tma_load a[0, %ok] : {m}x{kk} int\n    %tb = tma_load b[0, %ok] : {m}x{kk} int\n"
            f"    %u1 = dot %ta, %ta.T, acc=%u\n    %v1 = dot %tb, %tb.T, acc=%v\n    %ok1 = add %ok, {kk}\n"
            f"    yield %u1, %v1, %ok1\n  }}\n  store c[0, 0] = %u\n  store d[0, 0] = %v\n}}\n")


MINI = ("kernel mini(kb: buf<4x8 int>, vb: buf<8x4 int>, q: buf<4x4 int>, o: buf<4x4 int>) {\n"  # test_partition.cpp:50-66
        "  %zs = const zeros : 4x4 int\n  %zacc = const zeros : 4x4 int\n  %k0 = const 0\n"
        "  loop %k in 0..2 iter (%acc = %zacc, %ok = %k0) {\n"
        "    %tk = tma_load kb[0, %ok] : 4x4 int\n    %tv = tma_load vb[%ok, 0] : 4x4 int\n"
        "    %tq = tma_load q[0, 0] : 4x4 int\n    %s = dot %tq, %tk.T, acc=%zs\n"
        "    %m = reduce max %s axis=1\n    %p = ew sub %s, %m\n    %acc1 = dot %p, %tv, acc=%acc\n"
        "    %ok1 = add %ok, 4\n    yield %acc1, %ok1\n  }\n  store o[0, 0] = %acc\n}\n")


@pytest.mark.gpu
@pytest.mark.parametrize("name,text,pids", [
    ("gemm_2x2", _fx_gemm(2, 2, 2, 2), 1),
    ("mini_attention", MINI, 1),
    ("twochain_4x2x3", _fx_twochain(4, 2, 3), 1),
    ("gemm_8x4x3", _fx_gemm(8, 8, 4, 3), 1),
    ("attention_small", _fx_attention(4, 2), 1),
    ("attention_n3", _fx_attention(4, 3), 1),
    ("attention_n8_r8", _fx_attention(8, 8), 1),
    ("gemm_act", _fx_gemm_act(4, 4, 2), 1),
    ("gemm_act_n3", _fx_gemm_act(4, 4, 3), 1),
    ("gemm_tiled_2x3", _fx_gemm_tiled(2, 3, 4, 4, 4, 2), 6),
    ("gemm_tiled_4x4_k8", _fx_gemm_tiled(4, 4, 8, 8, 8, 4), 16),
])
def test_reference_fixture_kernels_through_the_reference_flow(ws, dev, tmp_path, name, text, pids):
    if not os.access(BIN, os.X_OK):
        pytest.skip("oracle/_ref/ws_dropin not built (needs the reference headers at build time)")
    rc, log = _run(tmp_path, [text], "--pids", str(pids))
    assert rc == 0 and "PASS" in log, f"{name}: {log}"
