"""Device traces in the reference's trace JSON schema and the watchdog's Deadlock verdict, on the
B200 (ref proj/include/warpspec/trace.hpp:59-83, sim.hpp:49-54,112-115)."""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _check_schema(j, units):
    assert set(j) == {"intervals", "blocks", "summary"}
    s = j["summary"]
    assert s["verdict"] == "completed" and s["cycles"] > 0
    assert units <= set(s["utilization"])
    for iv in j["intervals"]:
        assert set(iv) == {"unit", "wg", "start", "end", "label"}
        assert 0 <= iv["start"] <= iv["end"] <= s["cycles"]
    for b in j["blocks"]:
        assert set(b) == {"wg", "start", "end", "reason"} and b["end"] >= b["start"]
    json.dumps(j)  # serialisable as is


def test_gemm_trace_json(ws, dev):
    from paper_2510_14719_b200 import _lib, trace
    a = torch.randn(2048, 2048, device=dev, dtype=torch.bfloat16)
    b = torch.randn(4096, 2048, device=dev, dtype=torch.bfloat16)
    tr = torch.zeros(2 * 32 * 16, dtype=torch.int64, device=dev)
    lib = _lib.load()
    lib.ws_debug_gemm_trace(ctypes.c_void_p(tr.data_ptr()))
    try:
        ws.gemm_tn(a, b)
        torch.cuda.synchronize()
    finally:
        lib.ws_debug_gemm_trace(None)
    j = trace.gemm_trace_json(tr)
    _check_schema(j, {"tma0", "tensor_core", "cuda_wg2"})
    # the MMA issuer is busy for most of the run on a 32-K-block mainloop
    assert j["summary"]["utilization"]["tensor_core"] > 0.5


def test_attention_trace_json(ws, dev):
    from paper_2510_14719_b200 import trace
    q = torch.randn(1, 2, 4096, 128, device=dev, dtype=torch.bfloat16)
    k, v = torch.randn_like(q), torch.randn_like(q)
    tr = torch.zeros(3 * 256 * 8, dtype=torch.int64, device=dev)
    ws.attn_fwd(q, k, v, trace=tr)
    torch.cuda.synchronize()
    j = trace.attn_trace_json(tr)
    _check_schema(j, {"tensor_core", "cuda_wg1", "cuda_wg2"})


DEADLOCK = r'''
import json, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2510_14719_b200 as ws
from paper_2510_14719_b200 import trace
a = torch.randn(256, 1024, device="cuda", dtype=torch.bfloat16)
err = None
try:
    ws.gemm_tn(a, a)
    torch.cuda.synchronize()
except Exception as e:  # the trap surfaces as a CUDA error
    err = type(e).__name__
print(json.dumps({"error": err, "watchdog": trace.watchdog()}))
'''


def test_watchdog_reports_a_deadlock():
    """WS_DEBUG_DEADLOCK=1: CTA 0's producer never stages its first K block, the MMA warp waits on
    the aref's full barrier, the watchdog traps after 4 s and leaves the Deadlock record in pinned
    host memory (run in a subprocess: the trap ends that process's CUDA context)."""
    env = dict(os.environ, WS_DEBUG_DEADLOCK="1")
    out = subprocess.run([sys.executable, "-c", DEADLOCK, ROOT], env=env, capture_output=True, text=True,
                         timeout=120)
    line = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert line, out.stdout + out.stderr
    r = json.loads(line[-1])
    assert r["error"] is not None
    w = r["watchdog"]
    assert w["summary"]["verdict"] == "deadlock"
    assert w["block"] == [0, 0] or w["block"][0] in (0, 1)  # the pair stalled on CTA 0's first stage
    assert w["tag"] in (1, 2, 3, 5)  # a waiter on the aref or the accumulator hand-over
    assert w["deadlock"][0]["waiting_on"]
