"""Multi-GPU execution of the hot path: one process per GPU, shards from shard.py, no reduction.

GEMM: rank g computes the output columns [n_lo, n_hi) of c = a . b^T from all of a and rows
[n_lo, n_hi) of b. Attention: rank g computes (b,h) slices [bh_lo, bh_hi). The outputs are
gathered only to verify them (all_gather over the default process group: NCCL over NVLink on a
GPU box, gloo in the CPU tests); nothing on the compute path communicates.

The compute function is injectable so the same host logic runs against a CPU stand-in in the gloo
tests; the default is the CUDA path (ops.gemm_tn / ops.attn_fwd), which has no CPU fallback.
"""
from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist

from . import shard


def gemm_forward_shard(a: torch.Tensor, b: torch.Tensor, rank: int, world: int, bn: int = 256,
                       gemm: Optional[Callable] = None, **kw) -> torch.Tensor:
    """This rank's [M, n_hi - n_lo] block of a . b^T."""
    if gemm is None:
        from .ops import gemm_tn as gemm
    lo, hi = shard.gemm_shard(b.shape[0], world, rank, bn)
    return gemm(a, b[lo:hi], **kw)


def gather_gemm_columns(local: torch.Tensor, N: int, world: int, bn: int = 256, group=None) -> torch.Tensor:
    """All-gather column blocks (possibly of unequal width) into the full [M, N] matrix."""
    widths = [hi - lo for lo, hi in (shard.gemm_shard(N, world, r, bn) for r in range(world))]
    wmax = max(widths)
    M = local.shape[0]
    padded = torch.zeros((M, wmax), dtype=local.dtype, device=local.device)
    padded[:, :local.shape[1]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded.contiguous(), group=group)
    return torch.cat([p[:, :w] for p, w in zip(parts, widths)], dim=1)


def attn_forward_shard(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, rank: int, world: int,
                       causal: bool = False, attn: Optional[Callable] = None, **kw):
    """This rank's (b,h) slices: returns (o_local, lse_local) of shape [n_bh, S, Dh] / [n_bh, S]."""
    B, H, S, Dh = q.shape
    lo, hi = shard.attn_shard(B * H, world, rank)
    if attn is None:
        from .ops import attn_fwd

        o, lse = attn_fwd(q, k, v, causal=causal, bh_range=(lo, hi), **kw)
        return o.view(B * H, S, Dh)[lo:hi], lse.view(B * H, S)[lo:hi]
    flat = lambda t: t.reshape(B * H, S, Dh)[lo:hi]
    return attn(flat(q), flat(k), flat(v), causal)


def gather_attn_slices(o_local: torch.Tensor, lse_local: torch.Tensor, BH: int, world: int, group=None):
    """All-gather (b,h) slice blocks into full [BH, S, Dh] / [BH, S] tensors."""
    counts = [hi - lo for lo, hi in (shard.attn_shard(BH, world, r) for r in range(world))]
    cmax = max(counts)
    S, Dh = o_local.shape[1], o_local.shape[2]
    po = torch.zeros((cmax, S, Dh), dtype=o_local.dtype, device=o_local.device)
    pl = torch.zeros((cmax, S), dtype=lse_local.dtype, device=lse_local.device)
    po[:o_local.shape[0]] = o_local
    pl[:lse_local.shape[0]] = lse_local
    os_ = [torch.empty_like(po) for _ in range(world)]
    ls_ = [torch.empty_like(pl) for _ in range(world)]
    dist.all_gather(os_, po, group=group)
    dist.all_gather(ls_, pl, group=group)
    return (torch.cat([o[:c] for o, c in zip(os_, counts)]), torch.cat([l[:c] for l, c in zip(ls_, counts)]))
