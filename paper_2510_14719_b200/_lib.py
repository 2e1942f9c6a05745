"""ctypes binding of the C-ABI in include/ws.h (libws.so, built in-tree by __graft_entry__.build()).

This is the reference-side binding a maintainer would add: plain pointers, sizes and status
codes. There is no CPU fallback — if libws.so is missing, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# WS_LIB overrides the library path (developer A/B of two builds, scripts/attn_ab.py)
LIB_PATH = os.environ.get("WS_LIB") or os.path.join(_HERE, "libws.so")

# ws_status values; 1..12 follow warpspec::ErrorCode (ref proj/include/warpspec/errors.hpp:10-23)
STATUS_NAMES = {
    0: "ok", 1: "parse", 2: "type", 3: "unsupported-kernel", 4: "pipeline-infeasible",
    5: "stage-plan-ambiguous", 6: "unlowered-aref", 7: "smem-overflow", 8: "indivisible-tile",
    9: "register-budget", 10: "protocol-violation", 11: "io", 12: "eval", 100: "cuda-error",
}

WS_F32, WS_F16, WS_BF16, WS_E4M3 = 0, 1, 2, 3


class GemmDesc(ctypes.Structure):
    _fields_ = [
        ("in_dtype", ctypes.c_int32), ("out_dtype", ctypes.c_int32),
        ("M", ctypes.c_int64), ("N", ctypes.c_int64), ("K", ctypes.c_int64),
        ("A", ctypes.c_void_p), ("lda", ctypes.c_int64),
        ("B", ctypes.c_void_p), ("ldb", ctypes.c_int64),
        ("C", ctypes.c_void_p), ("ldc", ctypes.c_int64),
        ("scale_a", ctypes.c_float), ("scale_b", ctypes.c_float),
        ("D", ctypes.c_int32), ("P", ctypes.c_int32),
        ("persistent", ctypes.c_int32), ("cta_pair", ctypes.c_int32),
        ("bn", ctypes.c_int32), ("group_m", ctypes.c_int32),
        ("act", ctypes.c_int32), ("batch", ctypes.c_int32),
    ]


class AttnDesc(ctypes.Structure):
    _fields_ = [
        ("dtype", ctypes.c_int32),
        ("B", ctypes.c_int32), ("H", ctypes.c_int32), ("S", ctypes.c_int32), ("Dh", ctypes.c_int32),
        ("causal", ctypes.c_int32),
        ("softmax_scale", ctypes.c_float),
        ("Q", ctypes.c_void_p), ("K", ctypes.c_void_p), ("V", ctypes.c_void_p),
        ("O", ctypes.c_void_p),
        ("LSE", ctypes.c_void_p),
        ("D", ctypes.c_int32),
        ("bh_begin", ctypes.c_int32), ("bh_end", ctypes.c_int32),
        ("kv_block", ctypes.c_int32),
        ("scale_q", ctypes.c_float), ("scale_k", ctypes.c_float), ("scale_v", ctypes.c_float),
        ("MX", ctypes.c_void_p),
        ("grid_per_item", ctypes.c_int32),
    ]


class KBuffer(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char_p),
        ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
        ("is_real", ctypes.c_int32),
        ("data", ctypes.c_void_p),
    ]


class RunSpec(ctypes.Structure):
    """Mirror of ws_runspec (include/ws.h): the reference's RunSpec (ref driver.hpp:42-57)."""
    _fields_ = [("d", ctypes.c_int32), ("p", ctypes.c_int32), ("mode", ctypes.c_int32),
                ("coop_wgs", ctypes.c_int32), ("persistent", ctypes.c_int32)]


MODES = {"auto": 0, "fine": 1, "coarse": 2, "none": 3}  # ref driver.hpp:34-40 parse_pipeline_mode


# every symbol include/ws.h declares, with its ctypes signature
class WatchdogInfo(ctypes.Structure):
    """Mirror of ws_watchdog_info (include/ws.h)."""
    _fields_ = [("fired", ctypes.c_int32), ("block_x", ctypes.c_uint32), ("block_y", ctypes.c_uint32),
                ("thread", ctypes.c_uint32), ("barrier", ctypes.c_uint32), ("parity", ctypes.c_uint32),
                ("tag", ctypes.c_uint32)]


EXPORTS = {
    "ws_gemm_tn": (ctypes.c_int, [ctypes.POINTER(GemmDesc), ctypes.c_void_p]),
    "ws_gemm_plan_create": (ctypes.c_int, [ctypes.POINTER(GemmDesc), ctypes.POINTER(ctypes.c_void_p)]),
    "ws_gemm_plan_launch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "ws_gemm_plan_destroy": (None, [ctypes.c_void_p]),
    "ws_attn_fwd": (ctypes.c_int, [ctypes.POINTER(AttnDesc), ctypes.c_void_p]),
    "ws_attn_fwd_traced": (ctypes.c_int, [ctypes.POINTER(AttnDesc), ctypes.c_void_p, ctypes.c_void_p]),
    "ws_debug_gemm_trace": (None, [ctypes.c_void_p]),
    "ws_debug_gemm_clock": (None, [ctypes.c_void_p]),
    "ws_watchdog": (ctypes.c_int32, [ctypes.c_void_p]),
    "ws_run_kernel": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(KBuffer), ctypes.c_int32, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p]),
    "ws_run_kernel_spec": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(KBuffer), ctypes.c_int32, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(RunSpec), ctypes.c_void_p]),
    "ws_last_error": (ctypes.c_char_p, []),
    "ws_launch_count": (ctypes.c_int64, []),
    "ws_version": (ctypes.c_char_p, []),
}


OPTIONAL = {"ws_debug_gemm_trace", "ws_debug_gemm_clock", "ws_watchdog"}


class WsError(RuntimeError):
    """Mirror of warpspec::CompileError: carries the ErrorCode name (ref errors.hpp:43-55)."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.code = STATUS_NAMES.get(status, f"status-{status}")
        super().__init__(f"{self.code}: {message}")


_lib = None


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(
                f"{path} not found: build the CUDA extension first (python -c 'import __graft_entry__ as g; g.build()'). "
                "There is no CPU fallback on this path.")
        lib = ctypes.CDLL(path)
        for name, (res, args) in EXPORTS.items():
            if name in OPTIONAL and not hasattr(lib, name):
                continue  # diagnostics absent from an older build selected with WS_LIB
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = load().ws_last_error().decode(errors="replace")
        raise WsError(status, msg)
