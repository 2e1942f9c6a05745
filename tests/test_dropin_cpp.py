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
