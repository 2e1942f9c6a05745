"""paper_2510_14719_b200 — B200 (sm_100a) warp-specialized GEMM + FlashAttention forward.

The hot path of arxiv 2510.14719 (Tawa) behind the reference's operator interface; see
DESIGN.md. Public API: gemm_tn, attn_fwd (ops.py), gemm_tn_host (hostpipe.py: host buffers, copies
overlapped with compute), the C-ABI in include/ws.h (libws.so).
"""
from .ops import attn_fwd, gemm_tn, launch_count, run_kernel  # noqa: F401
from .hostpipe import gemm_tn_host  # noqa: F401
from ._lib import WsError  # noqa: F401

__all__ = ["gemm_tn", "gemm_tn_host", "attn_fwd", "run_kernel", "launch_count", "WsError"]
