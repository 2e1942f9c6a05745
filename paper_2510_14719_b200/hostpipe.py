"""Host-buffer GEMM pipeline: c_i = a_i . b_i^T for host tensors, through ws_gemm_tn.

The reference runs every pid on host buffers (interpret_sequential / simulate take and return
`Buffers` by value, ref proj/include/warpspec/interp.hpp:157-185, sim.hpp:686). A GPU caller with
host data pays PCIe both ways; this stages a sequence of jobs over three CUDA streams so that the
host->device copy of job i+1, the GEMM of job i and the device->host copy of job i-1 overlap
(PCIe is full duplex: both copy engines run at once). Device staging is double-buffered per job
slot (i % 2); events order every reuse:
  H2D(i)   waits GEMM(i-2)   (its A/B slot has been read)
  GEMM(i)  waits H2D(i), D2H(i-2)   (inputs landed; its C slot has been copied out)
  D2H(i)   waits GEMM(i)
Slot events persist across calls, so consecutive calls keep the pipeline full.

Large jobs are also split into row chunks (A rows, C rows; B is copied once per job): the GEMM of
chunk j starts when its A rows have landed and its C rows leave as soon as it is done, so the
pipeline's tail — the last job's GEMM plus its whole C copy-out, during which the host->device
direction idles — shrinks to one chunk (scripts/e2e_probe.py).
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import torch

from . import _lib
from .ops import gemm_tn


class _Pipe:
    def __init__(self, dev: torch.device):
        self.dev = dev
        self.s_h2d = torch.cuda.Stream(dev)
        self.s_comp = torch.cuda.Stream(dev)
        self.s_d2h = torch.cuda.Stream(dev)
        self.bufs: Dict[Tuple, torch.Tensor] = {}
        self.gemm_done: List[Optional[torch.cuda.Event]] = [None, None]
        self.d2h_done: List[Optional[torch.cuda.Event]] = [None, None]

    def buf(self, key, shape, dtype) -> torch.Tensor:
        t = self.bufs.get(key)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype:
            with torch.cuda.stream(self.s_comp):
                t = torch.empty(shape, dtype=dtype, device=self.dev)
            # the copy streams use the buffer too: when a shape change drops it, the caching
            # allocator must not hand the block out again before their queued copies are done
            t.record_stream(self.s_h2d)
            t.record_stream(self.s_d2h)
            # ... and the new block may have been freed on s_comp by work still queued there, so
            # the copy streams writing it start after that work
            ev = torch.cuda.Event()
            ev.record(self.s_comp)
            self.s_h2d.wait_event(ev)
            self.s_d2h.wait_event(ev)
            self.bufs[key] = t
        return t


_pipes: Dict[int, _Pipe] = {}


def _row_chunks(M: int, c_bytes: int, row_chunks: Optional[int]) -> int:
    if row_chunks is not None:
        n = max(1, int(row_chunks))
    else:
        n = max(1, round(c_bytes / (32 << 20)))  # ~32 MB of C per chunk
    # every chunk a whole number of 256-row CTA-pair blocks
    while n > 1 and (M % n or (M // n) % 256):
        n -= 1
    return n


def gemm_tn_host(jobs: Sequence[Tuple[torch.Tensor, torch.Tensor, torch.Tensor]], *,
                 device: Optional[torch.device] = None, row_chunks: Optional[int] = None,
                 **gemm_kw) -> torch.cuda.Event:
    """Run c = a . b^T for every (a, b, c) in `jobs`: a [M,K], b [N,K], c [M,N] host tensors
    (pinned for asynchronous copies). Returns a CUDA event that completes when every c is in host
    memory; the caller's current stream is made to wait on it. row_chunks: pieces each job's rows
    are split into (None = auto, ~32 MB of C each). gemm_kw: ws.gemm_tn knobs."""
    dev = device or torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        raise _lib.WsError(2, "gemm_tn_host needs a CUDA device (no CPU path)")
    p = _pipes.get(dev.index)
    if p is None:
        p = _pipes[dev.index] = _Pipe(dev)
    cur = torch.cuda.current_stream(dev)
    # work enqueued by the caller before this call (e.g. a timing event) precedes the pipeline
    start = torch.cuda.Event()
    start.record(cur)
    for s in (p.s_h2d, p.s_comp, p.s_d2h):
        s.wait_event(start)
    last = None
    for i, (a, b, c) in enumerate(jobs):
        if a.device.type != "cpu" or b.device.type != "cpu" or c.device.type != "cpu":
            raise _lib.WsError(2, "gemm_tn_host takes host tensors (use gemm_tn for device tensors)")
        slot = i % 2
        da = p.buf(("a", slot), a.shape, a.dtype)
        db = p.buf(("b", slot), b.shape, b.dtype)
        dc = p.buf(("c", slot), c.shape, c.dtype)
        M = a.shape[0]
        n = _row_chunks(M, c.numel() * c.element_size(), row_chunks)
        if row_chunks is None and i == len(jobs) - 1:
            # the last job's final chunk (its GEMM and copy-out) is the pipeline's exposed tail
            n = _row_chunks(M, c.numel() * c.element_size(), 2 * n)  # 2x: 22.8 vs 23.2 ms (4x, 8x slower)
        rows = M // n
        # H2D(i) after every GEMM of job i-2 has read the slot
        if p.gemm_done[slot] is not None:
            p.s_h2d.wait_event(p.gemm_done[slot])
        # GEMMs of job i after D2H(i-2) has copied the C slot out
        if p.d2h_done[slot] is not None:
            p.s_comp.wait_event(p.d2h_done[slot])
        with torch.cuda.stream(p.s_h2d):
            db.copy_(b, non_blocking=True)
        g = d = None
        for j in range(n):
            r = slice(j * rows, (j + 1) * rows)
            with torch.cuda.stream(p.s_h2d):
                da[r].copy_(a[r], non_blocking=True)
                h2d = torch.cuda.Event()
                h2d.record(p.s_h2d)
            p.s_comp.wait_event(h2d)
            gemm_tn(da[r], db, dc[r], stream=p.s_comp, **gemm_kw)
            g = torch.cuda.Event()
            g.record(p.s_comp)
            p.s_d2h.wait_event(g)
            with torch.cuda.stream(p.s_d2h):
                c[r].copy_(dc[r], non_blocking=True)
                d = torch.cuda.Event()
                d.record(p.s_d2h)
        p.gemm_done[slot] = g
        p.d2h_done[slot] = d
        last = d
    done = torch.cuda.Event()
    if last is not None:
        cur.wait_event(last)
    done.record(cur)
    return done
