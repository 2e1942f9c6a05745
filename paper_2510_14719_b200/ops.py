"""Host-side mirror of the reference operator interface for the hot path.

The reference runs a `.k` kernel per pid with `interpret_sequential(g, buffers, ExecContext{pid})`
(ref proj/include/warpspec/interp.hpp:157-185) or through `simulate` / `run_grid`
(ref proj/include/warpspec/sim.hpp:686, grid.hpp:140). On B200 the two kernel shapes of the path
run as one launch each over all pids:

  gemm_tn(a, b)        <- gemm.k family: c = a . b^T  (ref proj/kernels/gemm.k:2-17)
  attn_fwd(q, k, v)    <- the flash .k of SURVEY.md Appendix A (o = acc / l, lse = m + log l)

Both call the C-ABI (include/ws.h) through ctypes on torch's current CUDA stream. Torch is only
used for device memory and streams. Knob names follow RunSpec (ref driver.hpp:42-57).
"""
from __future__ import annotations

import ctypes
import math
from typing import Optional

import torch

from . import _lib

_DT = {torch.float32: _lib.WS_F32, torch.float16: _lib.WS_F16, torch.bfloat16: _lib.WS_BF16,
       torch.float8_e4m3fn: _lib.WS_E4M3}


def _stream_ptr(stream: Optional[torch.cuda.Stream], device: Optional[torch.device] = None) -> int:
    if stream is not None:
        return stream.cuda_stream
    idx = device.index if device is not None and device.index is not None else torch.cuda.current_device()
    return torch._C._cuda_getCurrentRawStream(idx)  # the current stream's handle, without a Stream object


_SMS: dict = {}
_PLAN_CACHE: dict = {}
_FAST_PLANS: dict = {}  # repeat-call key (see gemm_tn) -> the same plan handles as _PLAN_CACHE


class _OnDevice:
    """Make `device` current for the C-ABI call (the library launches on the current device, whose
    stream the descriptor names); a no-op, without torch's context-manager cost, when it already is."""
    __slots__ = ("idx", "prev")

    def __init__(self, device: torch.device):
        self.idx = device.index if device.index is not None else torch.cuda.current_device()

    def __enter__(self):
        self.prev = torch.cuda.current_device()
        if self.prev != self.idx:
            torch.cuda.set_device(self.idx)

    def __exit__(self, *exc):
        if self.prev != self.idx:
            torch.cuda.set_device(self.prev)


def _sm_count(device: torch.device) -> int:
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx not in _SMS:
        _SMS[idx] = torch.cuda.get_device_properties(idx).multi_processor_count
    return _SMS[idx]


def gemm_tn(a: torch.Tensor, b: torch.Tensor, out: Optional[torch.Tensor] = None, *,
            out_dtype: Optional[torch.dtype] = None, scale_a: float = 1.0, scale_b: float = 1.0,
            D: int = 0, P: int = 0, persistent: bool = True, cta_pair: Optional[bool] = None, bn: int = 0,
            group_m: int = 0, stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """c[M,N] = scale_a*scale_b * a[M,K] . b[N,K]^T with fp32 accumulation on the tensor cores
    (or, for 3-D a [batch,M,K] and b [batch,N,K], every product of the batch in one launch).

    a, b: row-major (last dim contiguous) CUDA tensors of dtype f16/bf16/float8_e4m3fn.
    out: optional [M,N] tensor (may be a column slice of a wider matrix; its row stride is ldc).
    cta_pair: None = auto (cta_group::2 CTA pairs when M % 256 == 0, K >= 256 and the pair tiles
    fill the GPU; single-CTA tiles otherwise).
    bn: 0 = auto (the library picks 256 x 512 pair tiles from 4 K blocks when they fill the GPU,
    else 256-wide tiles, or 128-wide single-CTA tiles for small problems).
    """
    if out is not None:
        # repeat call on buffers already validated and planned (same addresses, shapes, strides,
        # dtypes and knobs): straight to the prepared launch. Device pointers are unique across
        # devices (UVA), so the key also pins the device.
        fkey = (a.data_ptr(), b.data_ptr(), out.data_ptr(), a.shape, b.shape, out.shape, a.stride(),
                b.stride(), out.stride(), a.dtype, b.dtype, out.dtype, scale_a, scale_b, D, P, persistent,
                cta_pair, bn, group_m)
        plan = _FAST_PLANS.get(fkey)
        if plan is not None:
            plan.launch(stream)
            return out
    else:
        fkey = None
    if a.device.type != "cuda" or b.device.type != "cuda":
        raise _lib.WsError(2, "operands must be CUDA tensors (no CPU path)")
    if a.dtype != b.dtype or a.dtype not in (torch.float16, torch.bfloat16, torch.float8_e4m3fn):
        raise _lib.WsError(2, f"unsupported operand dtypes {a.dtype}, {b.dtype}")
    # [batch, M, K] x [batch, N, K] -> [batch, M, N]: one launch over every product (the .k's
    # gemm_batched, ref proj/kernels/gemm_batched.k:1-22); each operand's batches must be stacked
    # rows (stride(0) = rows * stride(1)), which the 2-D tensor maps then walk as one matrix
    batched = a.dim() == 3
    if batched != (b.dim() == 3) or a.dim() not in (2, 3):
        raise _lib.WsError(2, "a and b must both be 2-D, or both 3-D [batch, rows, K]")
    nbat = a.shape[0] if batched else 1
    if batched and b.shape[0] != nbat:
        raise _lib.WsError(2, f"batch sizes disagree: {nbat} vs {b.shape[0]}")
    M, K = a.shape[-2:]
    N, K2 = b.shape[-2:]
    if K != K2:
        raise _lib.WsError(2, f"inner dimensions disagree: {K} vs {K2}")
    if a.stride(-1) != 1 or b.stride(-1) != 1:
        raise _lib.WsError(2, "operands must be K-contiguous (row-major)")
    if batched and (a.stride(0) != M * a.stride(1) or b.stride(0) != N * b.stride(1)):
        raise _lib.WsError(2, "batched operands must stack their batches along rows")
    if cta_pair is None:
        # pairs only when the 256 x 256 pair tiles still give every SM pair a tile
        cta_pair = (M % 256 == 0 and K >= 256 and N % 128 == 0 and
                    nbat * (M // 256) * (N // 128) >= _sm_count(a.device))
    shape = (nbat, M, N) if batched else (M, N)
    if out is None:
        od = out_dtype or (torch.bfloat16 if a.dtype == torch.float8_e4m3fn else a.dtype)
        out = torch.empty(shape, dtype=od, device=a.device)
    if out.stride(-1) != 1 or tuple(out.shape) != shape or (batched and out.stride(0) != M * out.stride(1)):
        raise _lib.WsError(2, f"out must be {list(shape)} with contiguous rows" +
                           (" and batches stacked along rows" if batched else ""))
    lda, ldb, ldc = a.stride(-2), b.stride(-2), out.stride(-2)
    # prepared launches (ws_gemm_plan_*) are reused for repeated calls on the same buffers and
    # knobs: a repeat is one kernel launch (host cost per call matters for small GEMMs)
    key = (a.data_ptr(), b.data_ptr(), out.data_ptr(), M, N, K, lda, ldb, ldc, nbat,
           a.dtype, out.dtype, scale_a, scale_b, D, P, persistent, cta_pair, bn, group_m, a.device.index)
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        if b.device != a.device or out.device != a.device:
            raise _lib.WsError(2, "a, b and out must be on the same CUDA device")
        d = _lib.GemmDesc()
        d.in_dtype = _DT[a.dtype]
        d.out_dtype = _DT[out.dtype]
        d.M, d.N, d.K = M, N, K
        d.A, d.lda = a.data_ptr(), lda
        d.B, d.ldb = b.data_ptr(), ldb
        d.C, d.ldc = out.data_ptr(), ldc
        d.batch = nbat
        d.scale_a, d.scale_b = scale_a, scale_b
        d.D, d.P = D, P
        d.persistent, d.cta_pair, d.bn, d.group_m = int(persistent), int(cta_pair), bn, group_m
        plan = _GemmPlanHandle(d, a.device)
        if len(_PLAN_CACHE) >= 64:
            _PLAN_CACHE.clear()  # handles free their plans when dropped
            _FAST_PLANS.clear()
        _PLAN_CACHE[key] = plan
    if fkey is not None:
        _FAST_PLANS[fkey] = plan
    plan.launch(stream)
    return out


class _GemmPlanHandle:
    """Owns one ws_gemm_plan (include/ws.h): created on `device`, freed with the handle."""
    __slots__ = ("ptr", "device", "idx", "_lib", "_launch")

    def __init__(self, desc, device: torch.device):
        self._lib = _lib.load()
        self.device = device
        self.idx = device.index if device.index is not None else torch.cuda.current_device()
        self._launch = self._lib.ws_gemm_plan_launch
        self.ptr = ctypes.c_void_p()
        with _OnDevice(device):
            _lib.check(self._lib.ws_gemm_plan_create(ctypes.byref(desc), ctypes.byref(self.ptr)))

    def launch(self, stream: Optional[torch.cuda.Stream] = None):
        cur = torch._C._cuda_getDevice()
        if cur == self.idx:  # the common case: one cheap device query, no context switch
            s = stream.cuda_stream if stream is not None else torch._C._cuda_getCurrentRawStream(cur)
            rc = self._launch(self.ptr, s)
            if rc:
                _lib.check(rc)
            return
        with _OnDevice(self.device):
            _lib.check(self._launch(self.ptr, _stream_ptr(stream, self.device)))

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value:
            self._lib.ws_gemm_plan_destroy(self.ptr)
            self.ptr = ctypes.c_void_p()


def attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, causal: bool = False,
             softmax_scale: Optional[float] = None, out: Optional[torch.Tensor] = None,
             lse: Optional[torch.Tensor] = None, D: int = 0, bh_range: Optional[tuple] = None,
             stream: Optional[torch.cuda.Stream] = None, trace: Optional[torch.Tensor] = None,
             kv_block: int = 0, scale_q: float = 1.0, scale_k: float = 1.0, scale_v: float = 1.0,
             mx: Optional[torch.Tensor] = None, persistent: Optional[bool] = None):
    """FlashAttention forward over [B, H, S, Dh] tensors. Returns (o, lse) with lse fp32 [B, H, S]
    in natural-log units (lse = m + log l of the .k's running max m and row sum l).

    trace: optional int64 CUDA tensor of 3*256*8 entries receiving %clock64 stamps of CTA (0,0)
    (see ws_attn_fwd_traced in include/ws.h). kv_block: keys per K/V block (0 = auto = 128, or 64).
    float8_e4m3fn q/k/v (hdim 128): scale_q/k/v are the per-tensor descales; o is bf16.
    mx: optional fp32 [B, H, S] tensor receiving the exact row max m of the scaled scores (the
    .k's %m): the .k's row sum is then l = exp(lse - mx) and its accumulator acc = o * l.
    persistent: True = persistent grid, False = one CTA per work item (RunSpec persistent, ref
    driver.hpp:42-57), None = the measured default (persistent)."""
    if q.device.type != "cuda":
        raise _lib.WsError(2, "operands must be CUDA tensors (no CPU path)")
    if not (q.dtype == k.dtype == v.dtype) or q.dtype not in (torch.float16, torch.bfloat16, torch.float8_e4m3fn):
        raise _lib.WsError(2, f"unsupported dtype {q.dtype}")
    if q.dim() != 4:
        raise _lib.WsError(2, "q, k, v must be [B, H, S, Dh]")
    B, H, S, Dh = q.shape
    for t in (q, k, v):
        if tuple(t.shape) != (B, H, S, Dh) or not t.is_contiguous() or t.device != q.device:
            raise _lib.WsError(2, "q, k, v must be contiguous [B, H, S, Dh] on one device")
    # the kernel writes O through a tensor map built from B*H*S*Dh and q's dtype (bf16 for FP8
    # inputs) and B*H*S fp32 LSE values: caller buffers must be exactly that
    odt = torch.bfloat16 if q.dtype == torch.float8_e4m3fn else q.dtype
    if out is None:
        out = torch.empty_like(q, dtype=odt)
    elif tuple(out.shape) != (B, H, S, Dh) or out.dtype != odt or not out.is_contiguous() or out.device != q.device:
        raise _lib.WsError(2, f"out must be a contiguous {odt} [B, H, S, Dh] tensor on {q.device}")
    if lse is None:
        lse = torch.empty((B, H, S), dtype=torch.float32, device=q.device)
    elif (tuple(lse.shape) != (B, H, S) or lse.dtype != torch.float32 or not lse.is_contiguous()
          or lse.device != q.device):
        raise _lib.WsError(2, f"lse must be a contiguous float32 [B, H, S] tensor on {q.device}")
    if mx is not None and (tuple(mx.shape) != (B, H, S) or mx.dtype != torch.float32 or not mx.is_contiguous()
                           or mx.device != q.device):
        raise _lib.WsError(2, f"mx must be a contiguous float32 [B, H, S] tensor on {q.device}")
    if trace is not None and (trace.dtype != torch.int64 or trace.numel() < 3 * 256 * 8 or
                              not trace.is_contiguous() or trace.device != q.device):
        raise _lib.WsError(2, "trace must be a contiguous int64 tensor of >= 3*256*8 entries on q's device")
    d = _lib.AttnDesc()
    d.dtype = _DT[q.dtype]
    d.B, d.H, d.S, d.Dh = B, H, S, Dh
    d.causal = int(causal)
    d.softmax_scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(Dh)
    d.Q, d.K, d.V, d.O = q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr()
    d.LSE = lse.data_ptr()
    d.MX = mx.data_ptr() if mx is not None else None
    d.grid_per_item = 0 if persistent is None else (2 if persistent else 1)
    d.D = D
    lo, hi = bh_range if bh_range is not None else (0, B * H)
    d.bh_begin, d.bh_end = lo, hi
    d.kv_block = kv_block
    d.scale_q, d.scale_k, d.scale_v = scale_q, scale_k, scale_v
    lib = _lib.load()
    with _OnDevice(q.device):
        if trace is not None:
            _lib.check(lib.ws_attn_fwd_traced(ctypes.byref(d), ctypes.c_void_p(_stream_ptr(stream, q.device)),
                                              ctypes.c_void_p(trace.data_ptr())))
        else:
            _lib.check(lib.ws_attn_fwd(ctypes.byref(d), ctypes.c_void_p(_stream_ptr(stream, q.device))))
    return out, lse


def run_kernel(text: str, buffers: dict, pid_range=(0, 1), dtype: torch.dtype = torch.bfloat16,
               stream: Optional[torch.cuda.Stream] = None, spec: Optional[dict] = None) -> dict:
    """Run pids [lo, hi) of a `.k` kernel (reference grammar) on the GPU — the drop-in for the
    reference's tile-by-tile oracle run `interpret_tiles` (ref proj/tests/support/fixtures.hpp:148-157).

    buffers: {param name: numpy array} (float64 for `real`, int64 for `int` params); arrays are
    updated in place with the kernel's stores and also returned. Parameters without a buffer start
    zeroed (and are returned). See ws_run_kernel in include/ws.h for the supported kernel shapes.

    spec: the reference's RunSpec (ref driver.hpp:42-57) as a dict of d, p, mode ("auto" | "fine" |
    "coarse" | "none"), coop_wgs (or coop), persistent; rejected exactly as compile_kernel rejects
    it (ws_run_kernel_spec). None = the library's measured defaults."""
    import re

    import numpy as np

    # parameters the caller did not pass start zeroed (ref interp.hpp:140-154) and are returned
    header = text[text.index("(") + 1:text.index(")")]
    for name, r, c, elem in re.findall(r"(\w+)\s*:\s*buf<(\d+)x(\d+)\s+(int|real)>", header):
        if name not in buffers:
            buffers[name] = np.zeros((int(r), int(c)), dtype=np.float64 if elem == "real" else np.int64)
    keep = []
    arr = []
    for name, a in buffers.items():
        a = np.asarray(a)
        if a.dtype not in (np.float64, np.int64) or not a.flags.c_contiguous:
            raise _lib.WsError(2, f"buffer {name!r} must be a C-contiguous float64 or int64 array")
        b = _lib.KBuffer()
        nm = name.encode()
        keep.append(nm)
        b.name = nm
        b.rows, b.cols = (a.shape[0], a.shape[1]) if a.ndim == 2 else (a.shape[0], 1)
        b.is_real = int(a.dtype == np.float64)
        b.data = a.ctypes.data
        arr.append(b)
        buffers[name] = a
    bufs = (_lib.KBuffer * max(1, len(arr)))(*arr)
    lo, hi = pid_range
    lib = _lib.load()
    sp = None
    if spec is not None:
        unknown = set(spec) - {"d", "p", "mode", "coop_wgs", "coop", "persistent"}
        if unknown:
            raise _lib.WsError(2, f"unknown RunSpec fields {sorted(unknown)}")
        mode = spec.get("mode", "auto")
        if mode not in _lib.MODES:
            raise _lib.WsError(1, f"unknown pipeline mode '{mode}'")  # ref driver.hpp:34-40
        sp = _lib.RunSpec(d=int(spec.get("d", 0)), p=int(spec.get("p", 0)), mode=_lib.MODES[mode],
                          coop_wgs=int(spec.get("coop_wgs", spec.get("coop", 0))),
                          persistent=int(spec.get("persistent", 1)))
    _lib.check(lib.ws_run_kernel_spec(text.encode(), bufs, len(arr), lo, hi, _DT[dtype],
                                      ctypes.byref(sp) if sp is not None else None,
                                      ctypes.c_void_p(_stream_ptr(stream) if torch.cuda.is_available() else 0)))
    return buffers


def launch_count() -> int:
    return int(_lib.load().ws_launch_count())
