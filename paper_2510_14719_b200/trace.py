"""Device traces and the watchdog in the reference's trace JSON schema.

The reference's simulator reports a run as `trace_json(SimTrace, RunSummary)`
(ref proj/include/warpspec/trace.hpp:59-83): `intervals` ({unit, wg, start, end, label} — busy time
of a unit, e.g. "tma0", "tensor_core", "cuda_wg1", ref sim.hpp:16-22,188-191), `blocks` ({wg, start,
end, reason} — an agent waiting on a barrier, ref sim.hpp:24-29,266-281) and `summary` ({cycles,
verdict, utilization, launch_cycles}, utilization = busy / cycles per unit, ref trace.hpp:15-22).
On the B200 the same picture comes from %clock64 stamps the kernels write for CTA 0
(`ws_attn_fwd_traced`, `ws_debug_gemm_trace`), and the Deadlock verdict with its waiting agent
(`DeadlockEntry`, ref sim.hpp:49-54) from the device watchdog (`ws_watchdog`).
"""
from __future__ import annotations

import ctypes
from typing import Dict, List, Optional

from . import _lib

# wait sites the kernels pass to the watchdog (csrc/*.cuh mbar_wait tags)
TAGS: Dict[int, str] = {
    1: "aref empty (producer put)", 2: "aref full (MMA get)", 3: "tmem_empty (accumulator hand-over)",
    4: "aref empty (literal P window)", 5: "tmem_full (epilogue)", 9: "q_free", 11: "q_full",
    15: "p_full[0]", 16: "p_full[1]", 17: "s_free[0]", 18: "s_free[1]", 19: "o_free",
    20: "s_full[0]", 21: "s_full[1]", 24: "pv_done[0] (correction)", 25: "pv_done[1] (correction)",
    26: "pv_done[0] (epilogue)", 27: "pv_done[1] (epilogue)",
}


def _summary(intervals: List[dict], cycles: int, verdict: str = "completed") -> dict:
    busy: Dict[str, int] = {}
    for iv in intervals:
        busy[iv["unit"]] = busy.get(iv["unit"], 0) + iv["end"] - iv["start"]
    util = {u: (b / cycles if cycles > 0 else 0.0) for u, b in sorted(busy.items())}
    return {"cycles": cycles, "verdict": verdict, "utilization": util, "launch_cycles": 0}


def _finish(intervals: List[dict], blocks: List[dict]) -> dict:
    stamps = [x for iv in intervals + blocks for x in (iv["start"], iv["end"])]
    t0 = min(stamps) if stamps else 0
    for e in intervals + blocks:
        e["start"] -= t0
        e["end"] -= t0
    cycles = max((e["end"] for e in intervals + blocks), default=0)
    return {"intervals": intervals, "blocks": blocks, "summary": _summary(intervals, cycles)}


def gemm_trace_json(trace, cta: int = 0) -> dict:
    """`trace`: the 2*32*16 int64 buffer given to ws_debug_gemm_trace (tensor or array). Units: the
    producer ("tma0", wg 0), the MMA issuer ("tensor_core", wg 1, from its first staged K block to
    its last issue) and the epilogue ("cuda_wg2", one interval per N half drained and stored)."""
    import numpy as np
    t = np.asarray(trace.cpu() if hasattr(trace, "cpu") else trace, dtype=np.int64).reshape(2, 32, 16)[cta]
    iv: List[dict] = []
    bl: List[dict] = []
    for ti in range(32):
        r = [int(x) for x in t[ti]]
        if r[12] == 0:
            break
        iv.append({"unit": "tma0", "wg": 0, "start": r[12], "end": r[13], "label": f"tile{ti} a,b"})
        if r[5] and r[4]:
            iv.append({"unit": "tensor_core", "wg": 1, "start": r[5], "end": r[4], "label": f"tile{ti}"})
        if r[0] and r[1] and r[1] > r[0]:
            bl.append({"wg": 1, "start": r[0], "end": r[1], "reason": "wait tmem_empty (accumulator)"})
        if r[1] and r[5] and r[5] > r[1]:
            bl.append({"wg": 1, "start": r[1], "end": r[5], "reason": "wait full (first K block)"})
        for h, (f, rel, done) in enumerate(((6, 7, 8), (9, 10, 11))):
            if r[f] and r[done]:
                iv.append({"unit": "cuda_wg2", "wg": 2, "start": r[f], "end": r[done], "label": f"tile{ti} epilogue{h}"})
    return _finish(iv, bl)


def attn_trace_json(trace, steps: Optional[int] = None) -> dict:
    """`trace`: the 3*256*8 int64 buffer of ws_attn_fwd_traced (P-in-shared-memory kernel).
    Units: "tensor_core" (wg 0, the MMA issuer's span per step), "cuda_wg1" / "cuda_wg2" (the two
    softmax warpgroups: S loaded to P stored, and their epilogues). Blocks: softmax waiting for
    S_t, MMA waiting for P_t."""
    import numpy as np
    t = np.asarray(trace.cpu() if hasattr(trace, "cpu") else trace, dtype=np.int64).reshape(3, 256, 8)
    n = steps if steps is not None else int((t[0, :, 0] != 0).sum())
    iv: List[dict] = []
    bl: List[dict] = []
    for j in range(min(n, 256)):
        m = [int(x) for x in t[0, j]]
        if m[0] and m[5] and m[5] >= m[0]:
            iv.append({"unit": "tensor_core", "wg": 0, "start": m[0], "end": m[5], "label": f"step{j}"})
        if m[2] and m[3] and m[3] > m[2]:
            bl.append({"wg": 0, "start": m[2], "end": m[3], "reason": "wait p_full[0]"})
        if m[3] and m[4] and m[4] > m[3]:
            bl.append({"wg": 0, "start": m[3], "end": m[4], "reason": "wait p_full[1]"})
        for tt in (0, 1):
            s = [int(x) for x in t[1 + tt, j]]
            if s[1] and s[5] and s[5] >= s[1]:
                iv.append({"unit": f"cuda_wg{1 + tt}", "wg": 1 + tt, "start": s[1], "end": s[5], "label": f"C{j}"})
            if s[0] and s[1] and s[1] > s[0]:
                bl.append({"wg": 1 + tt, "start": s[0], "end": s[1], "reason": f"wait s_full[{tt}]"})
            if s[6] and s[7] and s[7] >= s[6]:
                iv.append({"unit": f"cuda_wg{1 + tt}", "wg": 1 + tt, "start": s[6], "end": s[7], "label": f"epilogue{j}"})
    return _finish(iv, bl)


def watchdog() -> Optional[dict]:
    """The device watchdog's record if one fired in this process (the kernel trapped), in the
    reference's Deadlock form: summary.verdict = "deadlock" and `deadlock` = [DeadlockEntry]
    ({wg, waiting_on, want_parity, completed}, ref sim.hpp:49-54; `completed` is not observable
    on hardware and reads -1). None if no wait has timed out."""
    lib = _lib.load()
    info = _lib.WatchdogInfo()
    if lib.ws_watchdog(ctypes.byref(info)) != 1:
        return None
    where = TAGS.get(info.tag, f"tag {info.tag}")
    return {"summary": {"verdict": "deadlock", "cycles": -1, "utilization": {}, "launch_cycles": 0,
                        "detail": f"block ({info.block_x},{info.block_y}) thread {info.thread} waited > 4 s on "
                                  f"{where} (smem barrier 0x{info.barrier:x}, parity {info.parity})"},
            "deadlock": [{"wg": info.thread // 32, "waiting_on": where, "want_parity": info.parity, "completed": -1}],
            "block": [info.block_x, info.block_y], "thread": info.thread, "tag": info.tag}
