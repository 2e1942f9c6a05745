"""Time the .k front end end to end (gemm.k M=N=8192 K=2048, double host buffers in and out), as
bench.py's e2e.through_k_front_end does (developer script, GPU)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2510_14719_b200 as ws
from bench import gemm_k_text

M = N = 8192
K = 2048
text = gemm_k_text(M, N, K, 128, 256, 64)
rng = np.random.default_rng(2026)
bufs = {"a": rng.integers(-16, 17, (M, K)) / 4.0, "b": rng.integers(-16, 17, (N, K)) / 4.0, "c": np.zeros((M, N))}
ws.run_kernel(text, bufs, pid_range=(0, (M // 128) * (N // 256)))
want = bufs["a"][:64] @ bufs["b"].T
assert np.array_equal(bufs["c"][:64], want), "rows 0..63 differ from numpy"
reps = []
for _ in range(5):
    t0 = time.perf_counter()
    ws.run_kernel(text, bufs, pid_range=(0, (M // 128) * (N // 256)))
    reps.append(time.perf_counter() - t0)
sec = sorted(reps)[2]
print(f"gemm.k 8192x8192x2048 through ws.run_kernel: {sec * 1e3:.1f} ms = {2 * M * N * K / sec / 1e12:.2f} TFLOP/s "
      f"(reps {[round(r * 1e3, 1) for r in reps]})")
