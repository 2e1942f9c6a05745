"""Multi-GPU verification run (outside any timed region): every rank computes its shard of the hot
path on its GPU, the shards are all-gathered over NCCL, and rank 0 checks them against the CPU
oracle.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 scripts/multi_gpu_verify.py
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker only)
import paper_2510_14719_b200 as ws  # noqa: E402
from paper_2510_14719_b200 import multi  # noqa: E402
from tests.gpu_helpers import ref_tensor  # noqa: E402


def main():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)

    # GEMM: global N = 2048 * world (weak), fp32 out -> bit-exact
    M, K, N = 2048, 1024, 2048 * world
    a = ref_tensor("a", (M, K), torch.bfloat16, dev)
    b = ref_tensor("b", (N, K), torch.bfloat16, dev)
    local_c = multi.gemm_forward_shard(a, b, rank, world, out_dtype=torch.float32)
    full = multi.gather_gemm_columns(local_c, N, world)
    ok_gemm = True
    if rank == 0:
        rows = np.array([0, 1, 255, 1024, 2047])
        want = oracle.gemm(oracle.generate_real("a", (M, K))[rows], oracle.generate_real("b", (N, K)))
        ok_gemm = np.array_equal(full[torch.from_numpy(rows).to(dev)].double().cpu().numpy(), want)

    # attention: (b,h) shards of B=1, H=16, S=2048, causal
    B, H, S, Dh = 1, 16, 2048, 128
    q = ref_tensor("q", (B, H, S, Dh), torch.bfloat16, dev, div=16.0)
    k = ref_tensor("k", (B, H, S, Dh), torch.bfloat16, dev, div=16.0)
    v = ref_tensor("v", (B, H, S, Dh), torch.bfloat16, dev)
    o_l, l_l = multi.attn_forward_shard(q, k, v, rank, world, causal=True)
    o, lse = multi.gather_attn_slices(o_l.contiguous(), l_l.contiguous(), B * H, world)
    ok_attn = True
    if rank == 0:
        qh, kh, vh = (t[0].double().cpu().numpy() for t in (q, k, v))
        for bh in (0, H // 2, H - 1):
            ro, rl = oracle.flash(qh[bh:bh + 1], kh[bh:bh + 1], vh[bh:bh + 1], True)
            got = o[bh].double().cpu().numpy()
            ok_attn &= np.abs(got - ro[0]).max() / np.abs(ro[0]).max() <= 1e-2
            ok_attn &= np.abs(lse[bh].double().cpu().numpy() - rl[0]).max() <= 1e-3
        print(f"multi_gpu_verify world={world}: gemm {'ok' if ok_gemm else 'MISMATCH'}, "
              f"attention {'ok' if ok_attn else 'MISMATCH'}", flush=True)
    dist.destroy_process_group()
    return 0 if (ok_gemm and ok_attn) else 1


if __name__ == "__main__":
    sys.exit(main())
