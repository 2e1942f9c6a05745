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
