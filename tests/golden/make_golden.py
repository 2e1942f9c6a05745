"""Generate the golden vectors in this directory from the REFERENCE ITSELF.

Runs the reference's own parse_kernel / generate_inputs / interpret_sequential (compiled from
/root/reference by oracle/Makefile into oracle/_ref/libwsref.so) on small `.k` instances of the hot
path and stores inputs and outputs as .npz. Only runnable where /root/reference exists; the
fixtures are committed so the CPU tests can pin the oracle restatement anywhere.

  python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from oracle import kernels as K  # noqa: E402

CASES = {
    # name: (kernel text, seed, pid count, extra fixed inputs)
    "gemm_real_64x48x96": (K.gemm_src(64, 48, 96, 32, 16, 32), 2026, K.gemm_tiles(64, 48, 32, 16), {}),
    "gemm_real_128x128x256": (K.gemm_src(128, 128, 256, 64, 64, 64), 2026, K.gemm_tiles(128, 128, 64, 64), {}),
    "gemm_real_scaled_64x64x128": (K.gemm_src(64, 64, 128, 32, 32, 32, scale=0.25), 2026,
                                   K.gemm_tiles(64, 64, 32, 32), {}),
    "gemm_int_32x32x32": (K.gemm_src(32, 32, 32, 8, 8, 8, elem="int"), 2026, 16, {}),
    "gemm_int_seed7_16x16x24": (K.gemm_src(16, 16, 24, 8, 8, 8, elem="int"), 7, 4, {}),
    # the other gemm.k-family forms (shapes of ref proj/kernels/gemm_batched.k, gemm_act.k,
    # gemm_large.k), integer payloads like the shipped files
    "gemm_batched_int_4x16x16": (K.gemm_batched_src(4, 16, 8, 16, 8), 2026, 16, {}),
    "gemm_act_int_32x32x32": (K.gemm_act_src(32, 32, 32, 8, 8, 8), 2026, 16, {}),
    "gemm_large_int_32x32x32": (K.gemm_src(32, 32, 32, 16, 16, 16, elem="int"), 2026, 4, {}),
    "gemm_act_real_64x64x64": (K.gemm_act_src(64, 64, 64, 32, 32, 16, elem="real"), 2026, 4, {}),
    "flash_bh3_s64_d16": (K.flash_src(3, 64, 16, 16, causal=False), 2026, 3 * 4, {"mb": K.flash_mask_bank(16)}),
    "flash_causal_bh3_s64_d16": (K.flash_src(3, 64, 16, 16, causal=True), 2026, 3 * 4,
                                 {"mb": K.flash_mask_bank(16)}),
    "flash_bh2_s128_d32": (K.flash_src(2, 128, 32, 32, causal=False), 2026, 2 * 4, {"mb": K.flash_mask_bank(32)}),
    "flash_causal_bh2_s128_d32": (K.flash_src(2, 128, 32, 32, causal=True), 2026, 2 * 4,
                                  {"mb": K.flash_mask_bank(32)}),
    # device-sized flash instances (head dim 64, S % 128 == 0) for the GPU front end: all three
    # outputs (acc, l, m) of the .k compared buffer by buffer
    "flash_bh2_s256_d64": (K.flash_src(2, 256, 64, 64, causal=False), 2026, 2 * 4, {"mb": K.flash_mask_bank(64)}),
    "flash_causal_bh2_s256_d64": (K.flash_src(2, 256, 64, 64, causal=True), 2026, 2 * 4,
                                  {"mb": K.flash_mask_bank(64)}),
    # the shipped integer max-shift attention kernel, verbatim (ref proj/kernels/attention.k)
    "attention_shipped": (K.shipped("attention.k"), 2026, 4, {}),
}


def main() -> None:
    only = set(sys.argv[1:])
    for name, (src, seed, pids, extra) in CASES.items():
        if only and name not in only:
            continue
        rk = oracle.RefKernel(src)
        ins = rk.generate(seed)
        ins.update(extra)
        out = rk.run(ins, 0, pids)
        payload = {f"in_{k}": v for k, v in ins.items()}
        payload.update({f"out_{k}": v for k, v in out.items()})
        payload["kernel"] = np.array(src)
        payload["seed"] = np.array(seed)
        payload["pids"] = np.array(pids)
        path = os.path.join(HERE, name + ".npz")
        np.savez_compressed(path, **payload)
        print(f"wrote {path}")


if __name__ == "__main__":
    main()
