"""Multi-process host logic of the sharded path on CPU (gloo, world_size 2 and 3).

The data-path kernels are replaced by a CPU stand-in (the tests' fake backend: double matmul /
the C oracle), so what is tested is the shard planning and the verification all-gather that the
GPU run uses with NCCL."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_14719_b200 import multi, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_gemm(a, b, **kw):
    return (a.double() @ b.double().T)


def _cpu_attn(q, k, v, causal):
    import oracle

    o, lse = oracle.flash(q.double().numpy(), k.double().numpy(), v.double().numpy(), causal, block=32, threads=1)
    return torch.from_numpy(o), torch.from_numpy(lse)


def _worker(rank, world, port, kind, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        if kind == "gemm":
            M, N, K = 64, 768, 96
            a = torch.randint(-16, 17, (M, K), generator=g).double() / 4
            b = torch.randint(-16, 17, (N, K), generator=g).double() / 4
            local = multi.gemm_forward_shard(a, b, rank, world, bn=128, gemm=_cpu_gemm)
            full = multi.gather_gemm_columns(local, N, world, bn=128)
            ok = torch.equal(full, a @ b.T)
        else:
            B, H, S, Dh = 1, 5, 64, 16
            q, k, v = (torch.randint(-16, 17, (B, H, S, Dh), generator=g).double() / 4 for _ in range(3))
            o_l, l_l = multi.attn_forward_shard(q, k, v, rank, world, causal=True, attn=_cpu_attn)
            o, lse = multi.gather_attn_slices(o_l, l_l, B * H, world)
            ro, rl = _cpu_attn(q.view(B * H, S, Dh), k.view(B * H, S, Dh), v.view(B * H, S, Dh), True)
            ok = torch.equal(o, ro) and torch.equal(lse, rl)
        with open(os.path.join(result_dir, f"r{rank}"), "w") as f:
            f.write("ok" if ok else "mismatch")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["gemm", "attn"])
def test_sharded_forward_and_gather(tmp_path, world, kind):
    mp.spawn(_worker, args=(world, _free_port(), kind, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert (tmp_path / f"r{r}").read_text() == "ok"


def test_shards_partition_columns_and_pids():
    for world in (1, 2, 4, 8):
        cols = [shard.gemm_shard(8192 * world, world, r) for r in range(world)]
        assert cols[0][0] == 0 and cols[-1][1] == 8192 * world
        assert all(cols[i][1] == cols[i + 1][0] for i in range(world - 1))
        assert all(hi - lo == 8192 for lo, hi in cols)  # equal blocks
        pids = [shard.gemm_pid_range(8192, 8192 * world, 128, 256, world, r) for r in range(world)]
        assert pids[0][0] == 0 and pids[-1][1] == 64 * 32 * world
        assert all(pids[i][1] == pids[i + 1][0] for i in range(world - 1))


def test_attn_shards_partition_slices():
    for BH, world in [(16, 8), (16, 3), (5, 2)]:
        rs = [shard.attn_shard(BH, world, r) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == BH
        assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1
        ps = [shard.attn_pid_range(BH, 1024, 128, world, r) for r in range(world)]
        assert ps[-1][1] == BH * 8


def test_uneven_split_rejects_unaligned():
    with pytest.raises(ValueError):
        shard.gemm_shard(1000, 2, 0, 256)


def _bench(*args, env=None):
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args], capture_output=True, text=True,
                          timeout=600, env=e)


@pytest.mark.parametrize("n", [2, 3])
def test_bench_self_launches_n_ranks(n):
    """`bench.py --gpus N` without a torchrun environment re-launches itself as N ranks (gloo here,
    --selftest: the launcher, strong-scaling shard plan, max-over-ranks timing and verification
    all-gather with a CPU stand-in for the kernels); rank 0 prints one line with n_gpus = N."""
    import json

    out = _bench("--gpus", str(n), "--selftest")
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    j = json.loads(lines[0])
    assert j["n_gpus"] == n and j["scaling"] == "strong" and j["verify"] == "bit-exact"
    assert len(j["per_rank_ms"]) == n and j["max_ms"] == max(j["per_rank_ms"])
    cols = j["shards"]
    assert cols[0][0] == 0 and cols[-1][1] == 8192 and all(cols[i][1] == cols[i + 1][0] for i in range(n - 1))


def test_bench_rejects_world_size_mismatch():
    out = _bench("--gpus", "4", "--selftest", env={"WORLD_SIZE": "2", "RANK": "0"})
    assert out.returncode == 2 and "WORLD_SIZE" in out.stdout
