"""The CPU oracle for the hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference` legs may
import this package, and only as the checker or the timed CPU baseline; the product package
(paper_2510_14719_b200) never imports it.

Two implementations:
  * liboracle.so  — ws_oracle.c, a C restatement of the reference arithmetic (file:line cited
                    there); runs anywhere (rebuilt with gcc on demand).
  * _ref/libwsref.so — the reference's own interpret_sequential / generate_inputs compiled from
                    /root/reference by oracle/Makefile (only buildable where the reference exists;
                    the built .so travels to the GPU box).
The restatement is pinned against the reference by tests/test_oracle.py and the golden vectors in
tests/golden/ (produced from libwsref.so by tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libwsref.so")

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
_i8p = ctypes.POINTER(ctypes.c_int8)

_olib = None
_rlib = None


def build_oracle() -> None:
    src = os.path.join(HERE, "ws_oracle.c")
    if not os.path.exists(ORACLE_SO) or os.path.getmtime(ORACLE_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o", ORACLE_SO, src,
                               "-lpthread", "-lm"])


def olib() -> ctypes.CDLL:
    global _olib
    if _olib is None:
        build_oracle()
        L = ctypes.CDLL(ORACLE_SO)
        L.ws_oracle_fnv1a64.restype = ctypes.c_uint64
        L.ws_oracle_fnv1a64.argtypes = [ctypes.c_char_p]
        L.ws_oracle_generate_real.argtypes = [ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int64, _dp]
        L.ws_oracle_generate_real_x4.argtypes = [ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int64, _i8p]
        L.ws_oracle_generate_int.argtypes = [ctypes.c_uint64, ctypes.c_char_p, ctypes.c_int64, _i64p]
        L.ws_oracle_gemm_real.argtypes = [_dp, _dp, _dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_double, ctypes.c_int]
        L.ws_oracle_gemm_int.argtypes = [_i64p, _i64p, _i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        L.ws_oracle_flash.argtypes = [_dp, _dp, _dp, _dp, _dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
        _olib = L
    return _olib


def _p(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


# ----------------------------------------------------------------------------------------------
# generate_inputs (ref proj/include/warpspec/driver.hpp:79-89)
# ----------------------------------------------------------------------------------------------
SEED = 2026


def generate_real(name: str, shape, seed: int = SEED) -> np.ndarray:
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.float64)
    olib().ws_oracle_generate_real(seed, name.encode(), n, _p(out))
    return out.reshape(shape)


def generate_real_x4(name: str, shape, seed: int = SEED) -> np.ndarray:
    """4x the real payloads as int8 (exact, cheap to ship to the GPU at 8192^2 scale)."""
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.int8)
    olib().ws_oracle_generate_real_x4(seed, name.encode(), n, _p(out, _i8p))
    return out.reshape(shape)


def generate_int(name: str, shape, seed: int = SEED) -> np.ndarray:
    n = int(np.prod(shape))
    out = np.empty(n, dtype=np.int64)
    olib().ws_oracle_generate_int(seed, name.encode(), n, _p(out, _i64p))
    return out.reshape(shape)


# ----------------------------------------------------------------------------------------------
# arithmetic
# ----------------------------------------------------------------------------------------------
def gemm(a: np.ndarray, b: np.ndarray, scale: float = 1.0, threads: int | None = None) -> np.ndarray:
    """c = scale * a . b^T with the reference's sequential double accumulation."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    M, K = a.shape
    N = b.shape[0]
    c = np.empty((M, N), dtype=np.float64)
    olib().ws_oracle_gemm_real(_p(a), _p(b), _p(c), M, N, K, N, scale, threads or default_threads())
    return c


def gemm_int(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.int64)
    b = np.ascontiguousarray(b, dtype=np.int64)
    M, K = a.shape
    N = b.shape[0]
    c = np.empty((M, N), dtype=np.int64)
    olib().ws_oracle_gemm_int(_p(a, _i64p), _p(b, _i64p), _p(c, _i64p), M, N, K)
    return c


def flash(q: np.ndarray, k: np.ndarray, v: np.ndarray, causal: bool, softmax_scale: float | None = None,
          block: int = 128, pid_range=None, threads: int | None = None):
    """Flash .k over [BH, S, Dh] (or [B, H, S, Dh]) float64 arrays -> (o, lse).

    pid_range restricts the computation to query blocks [lo, hi) of the batched pid order
    (pid = bh * (S/block) + qb); rows outside stay NaN."""
    shape = q.shape
    S, Dh = shape[-2], shape[-1]
    BH = int(np.prod(shape[:-2]))
    q = np.ascontiguousarray(q, dtype=np.float64).reshape(BH, S, Dh)
    k = np.ascontiguousarray(k, dtype=np.float64).reshape(BH, S, Dh)
    v = np.ascontiguousarray(v, dtype=np.float64).reshape(BH, S, Dh)
    o = np.full((BH, S, Dh), np.nan)
    lse = np.full((BH, S), np.nan)
    sc = softmax_scale if softmax_scale is not None else 1.0 / np.sqrt(Dh)
    lo, hi = pid_range if pid_range is not None else (0, BH * (S // block))
    olib().ws_oracle_flash(_p(q), _p(k), _p(v), _p(o), _p(lse), BH, S, Dh, block, block, int(causal), sc, lo, hi,
                           threads or default_threads())
    return o.reshape(shape), lse.reshape(shape[:-1])


def flash_stats(q: np.ndarray, k: np.ndarray, causal: bool, softmax_scale: float | None = None) -> np.ndarray:
    """The flash .k's stored running max m (ref: the `%mn` chain of SURVEY App. A): the row max of
    the scaled scores, causal positions above the diagonal excluded. [BH, S, Dh] -> [BH, S]."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    S, Dh = q.shape[-2], q.shape[-1]
    sc = softmax_scale if softmax_scale is not None else 1.0 / np.sqrt(Dh)
    s = np.einsum("bqd,bkd->bqk", q.reshape(-1, S, Dh), k.reshape(-1, S, Dh)) * sc
    if causal:
        s = np.where(np.tril(np.ones((S, S), dtype=bool)), s, -np.inf)
    return s.max(axis=-1)


def maxshift(q: np.ndarray, kt: np.ndarray, v: np.ndarray, D: int) -> np.ndarray:
    """The shipped max-shift attention.k (ref proj/kernels/attention.k:1-21) over all its pids, in
    exact int64: per key block j (kt[0:D, jD:(j+1)D], v[jD:(j+1)D]) s = q . tk^T,
    acc += (s - rowmax s) . tv (ref tile.hpp eval_dot / eval_reduce / eval_ew_binary)."""
    q = np.asarray(q, dtype=np.int64)
    kt = np.asarray(kt, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    o = np.zeros((q.shape[0], v.shape[1]), dtype=np.int64)
    for j in range(kt.shape[1] // D):
        s = q[:, :D] @ kt[:D, j * D:(j + 1) * D].T
        o += (s - s.max(axis=1, keepdims=True)) @ v[j * D:(j + 1) * D]
    return o


# ----------------------------------------------------------------------------------------------
# the reference itself (oracle/_ref/libwsref.so)
# ----------------------------------------------------------------------------------------------
def ref_available() -> bool:
    return os.path.exists(REF_SO)


def rlib() -> ctypes.CDLL:
    global _rlib
    if _rlib is None:
        if not ref_available():
            raise FileNotFoundError(f"{REF_SO} not built (make -C oracle ref, needs /root/reference)")
        L = ctypes.CDLL(REF_SO)
        L.wsref_num_params.argtypes = [ctypes.c_char_p]
        L.wsref_param.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, _i64p, _i64p,
                                  ctypes.POINTER(ctypes.c_int)]
        L.wsref_generate.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.c_char_p, ctypes.c_void_p]
        L.wsref_run.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_char_p, ctypes.c_int]
        L.wsref_last_error.restype = ctypes.c_char_p
        _rlib = L
    return _rlib


class RefKernel:
    """A `.k` kernel run by the reference's own interpreter."""

    def __init__(self, text: str):
        self.text = text.encode()
        L = rlib()
        n = L.wsref_num_params(self.text)
        if n < 0:
            raise ValueError(L.wsref_last_error().decode())
        self.params = []
        for i in range(n):
            name = ctypes.create_string_buffer(128)
            r, c, real = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
            L.wsref_param(self.text, i, name, 128, ctypes.byref(r), ctypes.byref(c), ctypes.byref(real))
            self.params.append((name.value.decode(), (r.value, c.value), bool(real.value)))

    def generate(self, seed: int = SEED) -> dict:
        out = {}
        for name, shape, real in self.params:
            arr = np.empty(shape, dtype=np.float64 if real else np.int64)
            rc = rlib().wsref_generate(self.text, seed, name.encode(), arr.ctypes.data_as(ctypes.c_void_p))
            if rc != 0:
                raise RuntimeError(rlib().wsref_last_error().decode())
            out[name] = arr
        return out

    def run(self, buffers: dict, pid_lo: int = 0, pid_hi: int = 1) -> dict:
        """interpret_sequential for pids [pid_lo, pid_hi); missing buffers start zeroed."""
        arrs = []
        for name, shape, real in self.params:
            dt = np.float64 if real else np.int64
            a = buffers.get(name)
            a = np.zeros(shape, dtype=dt) if a is None else np.array(a, dtype=dt, copy=True, order="C")
            assert a.shape == tuple(shape), (name, a.shape, shape)
            arrs.append(a)
        ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data_as(ctypes.c_void_p) for a in arrs])
        err = ctypes.create_string_buffer(512)
        rc = rlib().wsref_run(self.text, ptrs, pid_lo, pid_hi, err, 512)
        if rc != 0:
            raise RuntimeError(f"reference interpreter failed ({rc}): {err.value.decode()}")
        return {name: a for (name, _, _), a in zip(self.params, arrs)}
