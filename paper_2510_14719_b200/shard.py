"""Multi-GPU partitioning of the hot path: one process per GPU, no reduction.

GEMM: N-column blocks. With the .k pid map pid = pm + pn*TM (ref proj/kernels/gemm.k:4-7) a block
of output columns is a contiguous pid range; rank g owns columns [n_lo, n_hi) and needs all of A
plus rows [n_lo, n_hi) of B (contiguous in the N x K row-major b).

Attention: (b,h) slices. pid = bh * (S/BR) + query block, so rank g owns the
contiguous slice range [bh_lo, bh_hi).

The only collective is an all-gather of the output shards for verification, outside any timed
region (NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Tuple


def split_even(units: int, world: int, rank: int, align: int = 1) -> Tuple[int, int]:
    """Contiguous [lo, hi) share of `units` for `rank`, in multiples of `align` (units % align == 0).
    Earlier ranks take the remainder blocks, so shares differ by at most one block."""
    if units % align:
        raise ValueError(f"{units} units are not a multiple of the block {align}")
    blocks = units // align
    base, rem = divmod(blocks, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo * align, hi * align


def gemm_shard(N: int, world: int, rank: int, bn: int = 256) -> Tuple[int, int]:
    """Output-column range [n_lo, n_hi) of `rank` for a GEMM with N columns and N-tile bn."""
    return split_even(N, world, rank, bn)


def gemm_pid_range(M: int, N: int, BM: int, BN: int, world: int, rank: int) -> Tuple[int, int]:
    """The same shard expressed as a .k pid range: columns [n_lo, n_hi) <-> pids
    [n_lo/BN * TM, n_hi/BN * TM) with TM = M/BM (pid column-major over tiles)."""
    lo, hi = gemm_shard(N, world, rank, BN)
    tm = M // BM
    return lo // BN * tm, hi // BN * tm


def attn_shard(BH: int, world: int, rank: int) -> Tuple[int, int]:
    """(b,h) slice range [bh_lo, bh_hi) of `rank`."""
    return split_even(BH, world, rank, 1)


def attn_pid_range(BH: int, S: int, BR: int, world: int, rank: int) -> Tuple[int, int]:
    lo, hi = attn_shard(BH, world, rank)
    nqb = S // BR
    return lo * nqb, hi * nqb

