"""Shared helpers for the GPU parity tests: reference inputs on the device and comparisons."""
from __future__ import annotations

import numpy as np
import torch

import oracle


def ref_tensor(name: str, shape, dtype, dev, seed: int = oracle.SEED, div: float = 4.0) -> torch.Tensor:
    """The reference generator's real payloads ((rng%33-16)/4, ref driver.hpp:79-89) as a device
    tensor of `dtype` (exact in f16/bf16/e4m3). Built from the int8 x4 stream for speed."""
    x4 = oracle.generate_real_x4(name, shape, seed)
    t = torch.from_numpy(x4).to(dev).to(torch.float32) / div
    return t.to(dtype)


def as_f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to(torch.float64).cpu().numpy()


def rel_err(got: np.ndarray, want: np.ndarray) -> float:
    """max |got - want| / max |want| (norm-wise)."""
    return float(np.abs(got - want).max() / max(np.abs(want).max(), 1e-300))
