"""The C-ABI library (no GPU needed): it loads, exports every symbol include/ws.h declares, and
rejects bad launches with the reference's error codes before touching the device."""
from __future__ import annotations

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    text = open(os.path.join(ROOT, "include", "ws.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(ws_[a-z_0-9]+)\s*\(", text, re.M)))


def test_header_declares_the_path():
    assert _declared_functions() == ["ws_attn_fwd", "ws_attn_fwd_traced", "ws_debug_gemm_clock", "ws_debug_gemm_trace", "ws_gemm_plan_create",
                                    "ws_gemm_plan_destroy", "ws_gemm_plan_launch", "ws_gemm_tn", "ws_last_error",
                                    "ws_launch_count", "ws_run_kernel", "ws_run_kernel_spec", "ws_version",
                                    "ws_watchdog"]


def test_library_exports_every_declared_symbol(ws):
    lib = ws._lib.load()
    for name in _declared_functions():
        assert hasattr(lib, name), name
    assert set(ws._lib.EXPORTS) == set(_declared_functions())
    assert lib.ws_version().decode().startswith("ws-b200")
    assert lib.ws_launch_count() >= 0


def test_desc_layout_matches_header(tmp_path):
    """The ctypes mirrors have the C structs' size and every field's offset (checked against the
    header compiled by the host C compiler, when one is present)."""
    import shutil
    import subprocess

    from paper_2510_14719_b200 import _lib

    # in_dtype,out_dtype (8) + M,N,K (24) + A,lda,B,ldb,C,ldc (48) + scales (8) + 7 ints (28) -> 116, padded 120
    assert ctypes.sizeof(_lib.GemmDesc) == 120
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no host C compiler")
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{os.path.join(ROOT, "include", "ws.h")}"',
             "int main(void) {"]
    structs = (("ws_gemm_desc", _lib.GemmDesc), ("ws_attn_desc", _lib.AttnDesc), ("ws_runspec", _lib.RunSpec),
               ("ws_kbuffer", _lib.KBuffer))
    for cname, py in structs:
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call([cc, "-o", str(exe), str(src)])
    got = dict((" ".join(l.split()[:2]), int(l.split()[2])) for l in subprocess.check_output([str(exe)], text=True).splitlines())
    for cname, py in structs:
        assert got[f"{cname} size"] == ctypes.sizeof(py)
        for f, _ in py._fields_:
            assert got[f"{cname} {f}"] == getattr(py, f).offset, (cname, f)


def _gemm_desc(ws, **kw):
    d = ws._lib.GemmDesc()
    d.in_dtype, d.out_dtype = ws._lib.WS_BF16, ws._lib.WS_F32
    d.M, d.N, d.K = 256, 256, 256
    d.A = d.B = d.C = 0x100000  # never dereferenced: validation fails first
    d.lda = d.ldb = d.ldc = 256
    d.scale_a = d.scale_b = 1.0
    d.persistent = 1
    for k, v in kw.items():
        setattr(d, k, v)
    return d


@pytest.mark.parametrize("kw,code", [
    (dict(D=2, P=3), "pipeline-infeasible"),        # ref pipeline.hpp:84-92
    (dict(D=-1), "pipeline-infeasible"),            # ref driver.hpp:117-118
    (dict(M=200), "indivisible-tile"),              # ref grid.hpp:43-46
    (dict(N=320), "indivisible-tile"),
    (dict(K=100), "indivisible-tile"),
    (dict(D=7), "smem-overflow"),                   # 7 x 48 KB stages > 227 KB
    (dict(in_dtype=0), "type"),                     # fp32 inputs are not a tensor-core kind here
    (dict(bn=96), "type"),
    (dict(lda=128), "type"),
    (dict(act=2), "type"),
    (dict(M=0), "type"),                            # empty products are refused, not launched
    (dict(N=0), "type"),
    (dict(K=0), "type"),
    (dict(M=-256), "type"),
])
def test_gemm_validation_codes(ws, kw, code):
    lib = ws._lib.load()
    st = lib.ws_gemm_tn(ctypes.byref(_gemm_desc(ws, **kw)), None)
    assert ws._lib.STATUS_NAMES[st] == code, lib.ws_last_error()
    assert lib.ws_last_error()


@pytest.mark.parametrize("kw,code", [(dict(D=2, P=3), "pipeline-infeasible"), (dict(M=200), "indivisible-tile"),
                                     (dict(D=7), "smem-overflow"), (dict(in_dtype=0), "type")])
def test_gemm_plan_validation_codes(ws, kw, code):
    """A prepared launch validates exactly like ws_gemm_tn and hands out no plan on failure."""
    lib = ws._lib.load()
    plan = ctypes.c_void_p(0x1234)
    st = lib.ws_gemm_plan_create(ctypes.byref(_gemm_desc(ws, **kw)), ctypes.byref(plan))
    assert ws._lib.STATUS_NAMES[st] == code, lib.ws_last_error()
    assert not plan.value
    assert ws._lib.STATUS_NAMES[lib.ws_gemm_plan_launch(None, None)] == "type"
    lib.ws_gemm_plan_destroy(None)


def _attn_desc(ws, **kw):
    d = ws._lib.AttnDesc()
    d.dtype = ws._lib.WS_BF16
    d.B, d.H, d.S, d.Dh = 1, 2, 512, 128
    d.Q = d.K = d.V = d.O = 0x100000
    for k, v in kw.items():
        setattr(d, k, v)
    return d


@pytest.mark.parametrize("kw,code", [
    (dict(S=320), "indivisible-tile"),
    (dict(S=384, kv_block=64), "indivisible-tile"),  # the 64-key kernel pairs query tiles
    (dict(Dh=96), "unsupported-kernel"),
    (dict(D=1), "pipeline-infeasible"),             # coarse schedule needs D >= 2 (ref pipeline.hpp:309-315)
    (dict(D=9), "smem-overflow"),
    (dict(D=4), "smem-overflow"),                   # hdim 128, P in shared memory: room for 3 K/V slots
    (dict(D=9, kv_block=64), "smem-overflow"),
    (dict(kv_block=96), "type"),
    (dict(dtype=0), "type"),                        # fp32 attention is not a tensor-core kind here
    (dict(dtype=3, Dh=64), "unsupported-kernel"),   # FP8 attention: hdim 128 only
    (dict(dtype=3, kv_block=64), "unsupported-kernel"),
    (dict(dtype=3, D=5), "smem-overflow"),          # FP8: f16 P and V buffers leave room for 4 K slots
    (dict(bh_begin=1, bh_end=1), "type"),
    (dict(S=0), "type"),                            # empty inputs are refused, not launched
    (dict(B=0), "type"),
    (dict(H=0), "type"),
])
def test_attn_validation_codes(ws, kw, code):
    lib = ws._lib.load()
    st = lib.ws_attn_fwd(ctypes.byref(_attn_desc(ws, **kw)), None)
    assert ws._lib.STATUS_NAMES[st] == code, lib.ws_last_error()


def test_python_api_raises_wserror_without_cuda_tensors(ws):
    torch = pytest.importorskip("torch")
    a = torch.zeros(128, 64, dtype=torch.bfloat16)
    with pytest.raises(ws.WsError) as e:
        ws.gemm_tn(a, a)
    assert e.value.code == "type"


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2510_14719_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "liboracle" not in src and "libwsref" not in src, f


def test_trace_json_schema_from_a_synthetic_gemm_trace():
    """trace.gemm_trace_json turns stamps into the reference's trace JSON (intervals / blocks /
    summary with utilization = busy / cycles, ref trace.hpp:15-22,59-83) — host logic, no GPU."""
    import numpy as np
    from paper_2510_14719_b200 import trace
    t = np.zeros((2, 32, 16), dtype=np.int64)
    for ti in range(3):
        b = 1000 + ti * 10000
        t[0, ti, 12], t[0, ti, 13] = b, b + 8000              # producer
        t[0, ti, 0], t[0, ti, 1], t[0, ti, 5], t[0, ti, 4] = b + 50, b + 100, b + 300, b + 9000  # MMA
        t[0, ti, 6], t[0, ti, 7], t[0, ti, 8] = b + 9500, b + 9900, b + 11000  # epilogue half 0
        t[0, ti, 9], t[0, ti, 10], t[0, ti, 11] = b + 9700, b + 10000, b + 11500
    j = trace.gemm_trace_json(t)
    assert set(j) == {"intervals", "blocks", "summary"}
    s = j["summary"]
    assert s["verdict"] == "completed" and s["cycles"] == max(iv["end"] for iv in j["intervals"] + j["blocks"])
    assert set(s["utilization"]) == {"tma0", "tensor_core", "cuda_wg2"}
    assert all(0.0 < u <= 1.0 for k, u in s["utilization"].items() if k != "cuda_wg2")
    assert all(iv["start"] >= 0 and iv["end"] >= iv["start"] for iv in j["intervals"])
    assert {b["reason"] for b in j["blocks"]} == {"wait tmem_empty (accumulator)", "wait full (first K block)"}
    tc = [iv for iv in j["intervals"] if iv["unit"] == "tensor_core"]
    assert len(tc) == 3 and tc[0]["end"] - tc[0]["start"] == 8700


def test_watchdog_reports_nothing_without_a_timeout(ws):
    """ws_watchdog is callable without a GPU and reports no Deadlock when no wait has timed out."""
    from paper_2510_14719_b200 import trace
    assert trace.watchdog() is None


def test_host_pipeline_row_chunk_policy():
    """gemm_tn_host's row chunking (host logic): ~32 MB of C per chunk, whole 256-row pair blocks,
    an explicit count reduced until it divides M into such blocks."""
    from paper_2510_14719_b200.hostpipe import _row_chunks
    assert _row_chunks(8192, 8192 * 8192 * 2, None) == 4        # 128 MB of bf16 C -> 4 chunks
    assert _row_chunks(8192, 8192 * 8192 * 2, 8) == 8
    assert _row_chunks(256, 256 * 512 * 4, None) == 1
    assert _row_chunks(768, 768 * 768 * 4, 4) == 3             # 4 does not divide 768 into 256-row blocks
    assert _row_chunks(1024, 1024 * 512 * 4, 2) == 2
    assert _row_chunks(640, 640 * 768 * 4, 4) == 1             # 640 rows: no whole 256-row split


def test_trace_json_schema_from_a_synthetic_attention_trace():
    """trace.attn_trace_json (host logic): MMA issue spans, softmax spans per warpgroup, epilogue
    intervals and the waits on S / P become the reference's intervals / blocks / summary."""
    import numpy as np
    from paper_2510_14719_b200 import trace
    t = np.zeros((3, 256, 8), dtype=np.int64)
    for j in range(4):
        b = 10_000 + 3000 * j
        t[0, j, :6] = [b, b + 100, b + 200, b + 900, b + 1500, b + 1700]      # MMA issuer
        for tt in (0, 1):
            o = 300 * tt
            t[1 + tt, j, :6] = [b + o, b + o + 150, b + o + 400, b + o + 600, b + o + 1300, b + o + 1450]
    t[1, 3, 6], t[1, 3, 7] = 22_000, 23_000                                  # tile 0 epilogue
    j = trace.attn_trace_json(t)
    s = j["summary"]
    assert s["verdict"] == "completed" and set(s["utilization"]) == {"tensor_core", "cuda_wg1", "cuda_wg2"}
    assert len([iv for iv in j["intervals"] if iv["unit"] == "tensor_core"]) == 4
    assert any(iv["label"] == "epilogue3" for iv in j["intervals"])
    assert {b["reason"] for b in j["blocks"]} >= {"wait p_full[0]", "wait p_full[1]", "wait s_full[0]", "wait s_full[1]"}
    assert all(0 <= iv["start"] <= iv["end"] <= s["cycles"] for iv in j["intervals"])
