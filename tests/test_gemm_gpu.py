"""GEMM parity on the B200 through the C-ABI vs the CPU oracle (gemm.k, ref proj/kernels/gemm.k:2-17).

Bar (BASELINE.json north_star / SURVEY.md §8c):
  * fp32 output: BIT-EXACT. Reference inputs are k/4 with |k| <= 16, so every partial sum is a
    multiple of 1/16 below 2^20 and any fp32 summation order equals the double oracle.
  * bf16/fp16 output: max|d|/max|ref| <= 1e-2.      * FP8 e4m3 (scaled): <= 5e-2.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2510_14719_b200 import shard
from tests.gpu_helpers import as_f64, ref_tensor, rel_err

pytestmark = pytest.mark.gpu

F16, BF16, E4M3, F32 = torch.float16, torch.bfloat16, torch.float8_e4m3fn, torch.float32


def _run(ws, dev, M, N, K, dt, out_dt, seed=oracle.SEED, **kw):
    a = ref_tensor("a", (M, K), dt, dev, seed)
    b = ref_tensor("b", (N, K), dt, dev, seed)
    c = ws.gemm_tn(a, b, out_dtype=out_dt, **kw)
    torch.cuda.synchronize()
    return a, b, c


def _want(M, N, K, seed=oracle.SEED, scale=1.0, rows=None):
    a = oracle.generate_real("a", (M, K), seed)
    b = oracle.generate_real("b", (N, K), seed)
    if rows is not None:
        a = a[rows]
    return oracle.gemm(a, b, scale=scale)


def test_c1_fp16_1024_cubed_bit_exact(ws, dev):
    """C1: fp16 GEMM M=N=K=1024, fp32 accumulate — the config the CPU oracle runs in full."""
    _, _, c = _run(ws, dev, 1024, 1024, 1024, F16, F32)
    assert np.array_equal(as_f64(c), _want(1024, 1024, 1024))


@pytest.mark.parametrize("dt", [F16, BF16, E4M3])
@pytest.mark.parametrize("shape", [(128, 256, 128), (256, 512, 1024), (384, 768, 2048)])
def test_fp32_out_bit_exact(ws, dev, dt, shape):
    M, N, K = shape
    _, _, c = _run(ws, dev, M, N, K, dt, F32)
    assert np.array_equal(as_f64(c), _want(M, N, K))


@pytest.mark.parametrize("dt,out_dt", [(BF16, BF16), (F16, F16), (BF16, F16), (E4M3, BF16)])
def test_low_precision_out_within_tolerance(ws, dev, dt, out_dt):
    M, N, K = 512, 512, 1024
    _, _, c = _run(ws, dev, M, N, K, dt, out_dt)
    assert rel_err(as_f64(c), _want(M, N, K)) <= 1e-2


def test_fp8_per_tensor_scales(ws, dev):
    """C3 semantics: c = (sa*sb) * a.b^T (the .k's %o = ew mul %acc, %s), tol 5e-2."""
    M, N, K = 512, 768, 2048
    _, _, c = _run(ws, dev, M, N, K, E4M3, BF16, scale_a=0.5, scale_b=2.0 ** -3)
    assert rel_err(as_f64(c), _want(M, N, K, scale=0.5 * 2.0 ** -3)) <= 5e-2
    _, _, c32 = _run(ws, dev, M, N, K, E4M3, F32, scale_a=0.5, scale_b=2.0)
    assert np.array_equal(as_f64(c32), _want(M, N, K, scale=1.0))  # power-of-two scales stay exact


@pytest.mark.parametrize("D", [1, 2, 3, 4])
def test_aref_depth_and_mma_depth_sweep(ws, dev, D):
    """Every (D, P <= D) pipeline computes the same bits (ref pipeline.hpp:44-142)."""
    M, N, K = 256, 512, 1024
    want = _want(M, N, K)
    for P in range(1, D + 1):
        _, _, c = _run(ws, dev, M, N, K, BF16, F32, D=D, P=P)
        assert np.array_equal(as_f64(c), want), (D, P)


def test_p_greater_than_d_is_rejected(ws, dev):
    a = torch.zeros(128, 64, dtype=BF16, device=dev)
    with pytest.raises(ws.WsError) as e:
        ws.gemm_tn(a, a, D=2, P=3)
    assert e.value.code == "pipeline-infeasible"


@pytest.mark.parametrize("kw", [dict(bn=128), dict(persistent=False), dict(group_m=1), dict(group_m=3),
                                dict(bn=128, persistent=False, D=6)])
def test_schedule_variants(ws, dev, kw):
    M, N, K = 640, 768, 512
    _, _, c = _run(ws, dev, M, N, K, BF16, F32, **kw)
    assert np.array_equal(as_f64(c), _want(M, N, K))


def test_single_tile_single_kblock(ws, dev):
    _, _, c = _run(ws, dev, 128, 256, 64, BF16, F32)
    assert np.array_equal(as_f64(c), _want(128, 256, 64))


def test_long_k(ws, dev):
    _, _, c = _run(ws, dev, 256, 256, 16384, BF16, F32)
    assert np.array_equal(as_f64(c), _want(256, 256, 16384))


@pytest.mark.parametrize("world", [2, 4, 8])
def test_n_column_shards_cover_the_output(ws, dev, world):
    """rank g computes columns [n_lo, n_hi) from B rows [n_lo, n_hi) into a column
    slice of C (ldc = N); the union of the shards equals the unsharded product."""
    M, N, K = 256, 2048, 512
    a = ref_tensor("a", (M, K), BF16, dev)
    b = ref_tensor("b", (N, K), BF16, dev)
    c = torch.full((M, N), float("nan"), dtype=F32, device=dev)
    for r in range(world):
        lo, hi = shard.gemm_shard(N, world, r)
        ws.gemm_tn(a, b[lo:hi], out=c[:, lo:hi])
    torch.cuda.synchronize()
    assert np.array_equal(as_f64(c), _want(M, N, K))


@pytest.mark.parametrize("K,kw", [(256, {}), (8192, {}), (64, dict(cta_pair=True, bn=512)),
                                  (192, dict(cta_pair=True, bn=512)), (1024, dict(cta_pair=True, bn=512))])
def test_full_size_8192_sampled_rows_exact(ws, dev, K, kw):
    """C2 at full size: every row checked for the size-independent row-sum identity
    sum_n c[m,n] = a[m,:] . (sum_n b[n,:]), and 24 sampled rows (first/last of tiles and groups)
    bit-exact against the oracle. The 256x512 cases run ~7 tiles per CTA pair with 1, 3 and 16 K
    blocks: the half-by-half accumulator hand-over with head deferral (fewer K blocks than stages),
    tail deferral and both."""
    M = N = 8192
    a = ref_tensor("a", (M, K), BF16, dev)
    b = ref_tensor("b", (N, K), BF16, dev)
    c = ws.gemm_tn(a, b, out_dtype=F32, **kw)
    torch.cuda.synchronize()
    rowsum = c.double().sum(1)
    want_rowsum = a.double() @ b.double().sum(0)
    assert torch.equal(rowsum, want_rowsum)  # exact: all terms are multiples of 1/16 well below 2^53
    rows = np.array([0, 1, 127, 128, 255, 2047, 2048, 4095, 4096, 6143, 8063, 8064, 8191]
                    + list(np.random.default_rng(K).integers(0, M, 11)))
    want = _want(M, N, K, rows=rows)
    got = as_f64(c[torch.from_numpy(rows).to(dev)])
    assert np.array_equal(got, want)


def test_full_size_bf16_out_bench_config(ws, dev):
    """The bench configuration (bf16 in/out, 8192^3) on sampled rows, tol 1e-2."""
    M = N = K = 8192
    a = ref_tensor("a", (M, K), BF16, dev)
    b = ref_tensor("b", (N, K), BF16, dev)
    c = ws.gemm_tn(a, b)
    torch.cuda.synchronize()
    rows = np.array([0, 4097, 8191])
    assert rel_err(as_f64(c[torch.from_numpy(rows).to(dev)]), _want(M, N, K, rows=rows)) <= 1e-2


def test_launches_are_counted(ws, dev):
    n0 = ws.launch_count()
    _run(ws, dev, 128, 256, 64, BF16, F32)
    assert ws.launch_count() == n0 + 1


@pytest.mark.parametrize("row_chunks", [None, 2, 4])
def test_host_pipeline_matches_device_path_bit_exact(ws, dev, row_chunks):
    """gemm_tn_host (host buffers, H2D / GEMM / D2H overlapped on three streams, slots reused every
    other job, jobs split into 256-row chunks where row_chunks asks and M allows) gives the oracle's
    exact fp32 results for every job, across two calls."""
    shapes = [(256, 512, 128), (512, 256, 1024), (256, 256, 64), (1024, 512, 256), (768, 768, 512)]
    jobs, want = [], []
    for i, (M, N, K) in enumerate(shapes):
        a = oracle.generate_real(f"a{i}", (M, K))
        b = oracle.generate_real(f"b{i}", (N, K))
        jobs.append((torch.from_numpy(a).to(torch.bfloat16).pin_memory(),
                     torch.from_numpy(b).to(torch.bfloat16).pin_memory(),
                     torch.full((M, N), float("nan"), dtype=torch.float32).pin_memory()))
        want.append(oracle.gemm(a, b))
    for _ in range(2):
        for _, _, c in jobs:
            c.fill_(float("nan"))
        ev = ws.gemm_tn_host(jobs, device=dev, row_chunks=row_chunks)
        ev.synchronize()
        for (_, _, c), w in zip(jobs, want):
            assert np.array_equal(c.numpy().astype(np.float64), w)


@pytest.mark.parametrize("D,P", [(2, 2), (3, 3), (4, 4), (3, 1), (4, 2)])
def test_pair_512_tiles_pipeline_depths(ws, dev, D, P):
    """256 x 512 pair tiles over several tiles per pair: the half-by-half accumulator hand-over
    (P = D) and the plain path the literal P window takes (P < D) give the same exact bits."""
    M, N, K = 2048, 8192, 320  # 128 tiles (~2 per CTA pair), 5 K blocks
    _, _, c = _run(ws, dev, M, N, K, BF16, F32, cta_pair=True, bn=512, D=D, P=P, persistent=True)
    assert np.array_equal(as_f64(c), _want(M, N, K))


@pytest.mark.parametrize("out_dt", [BF16, F16])
@pytest.mark.parametrize("K,kw", [(128, dict(D=4)), (1024, {}), (2048, dict(D=3)), (4096, dict(scale_a=0.5))])
def test_pair_512_16bit_out_equals_rounded_oracle(ws, dev, out_dt, K, kw):
    """256 x 512 pair tiles with 16-bit output (the early-release epilogue: all eight epilogue
    warps drain one N half into registers, release it, then store). The fp32 accumulation is exact
    for the reference payloads, so the output must equal the oracle rounded once to out_dt."""
    M, N = 1024, 4096  # 32 pair tiles (fewer than the 74 pairs), then 64 at 2048 rows
    for m in (M, 2048):
        a = ref_tensor("a", (m, K), BF16, dev)
        b = ref_tensor("b", (N, K), BF16, dev)
        c = ws.gemm_tn(a, b, out_dtype=out_dt, cta_pair=True, bn=512, **kw)
        torch.cuda.synchronize()
        scale = kw.get("scale_a", 1.0)
        want = torch.from_numpy(_want(m, N, K, scale=scale)).to(dev).to(out_dt)
        assert torch.equal(c, want), (m, K, kw)


def test_pair_512_many_tiles_per_pair_16bit(ws, dev):
    """~14 tiles per CTA pair (8192 x 8192 with 256 x 512 tiles): every hand-over of both N halves
    between the MMA warp and the early-release epilogue, sampled rows exact after rounding."""
    M = N = 8192
    K = 512
    a = ref_tensor("a", (M, K), BF16, dev)
    b = ref_tensor("b", (N, K), BF16, dev)
    c = ws.gemm_tn(a, b, out_dtype=BF16, cta_pair=True, bn=512)
    torch.cuda.synchronize()
    rows = np.array([0, 255, 256, 4095, 4096, 8191] + list(np.random.default_rng(7).integers(0, M, 10)))
    want = torch.from_numpy(_want(M, N, K, rows=rows)).to(dev).to(BF16)
    assert torch.equal(c[torch.from_numpy(rows).to(dev)], want)


@pytest.mark.parametrize("kw", [dict(cta_pair=False, bn=256), dict(cta_pair=False, bn=128), dict(cta_pair=True, bn=256),
                                dict(cta_pair=True, bn=512), {}])
def test_batched_one_launch_bit_exact(ws, dev, kw):
    """gemm_batched.k semantics (ref proj/kernels/gemm_batched.k:1-22): products stacked along rows,
    one launch over batch x tiles; every product equals the oracle exactly (fp32 out)."""
    nb, M, N, K = 3, 512, 1024, 320
    a = torch.stack([ref_tensor(f"a{i}", (M, K), BF16, dev) for i in range(nb)])
    b = torch.stack([ref_tensor(f"b{i}", (N, K), BF16, dev) for i in range(nb)])
    n0 = ws.launch_count()
    c = ws.gemm_tn(a, b, out_dtype=F32, **kw)
    torch.cuda.synchronize()
    assert ws.launch_count() == n0 + 1 and tuple(c.shape) == (nb, M, N)
    for i in range(nb):
        want = oracle.gemm(oracle.generate_real(f"a{i}", (M, K)), oracle.generate_real(f"b{i}", (N, K)))
        assert np.array_equal(as_f64(c[i]), want), (i, kw)


def test_batched_rejects_unstacked_operands(ws, dev):
    a = torch.zeros(2, 256, 128, dtype=BF16, device=dev)
    b = torch.zeros(2, 256, 128, dtype=BF16, device=dev)
    with pytest.raises(ws.WsError):
        ws.gemm_tn(a.transpose(0, 1).contiguous().transpose(0, 1), b)  # batches interleaved, not stacked
    with pytest.raises(ws.WsError):
        ws.gemm_tn(a, b[:1])


def test_batched_fp8_scaled_bf16_out(ws, dev):
    """FP8 e4m3 batched launch with per-tensor scales and 16-bit output (256 x 512 pair tiles):
    each product equals the oracle rounded once to bf16 (power-of-two scales keep it exact)."""
    nb, M, N, K = 2, 512, 1024, 2048
    a = torch.stack([ref_tensor(f"a{i}", (M, K), E4M3, dev) for i in range(nb)])
    b = torch.stack([ref_tensor(f"b{i}", (N, K), E4M3, dev) for i in range(nb)])
    c = ws.gemm_tn(a, b, out_dtype=BF16, scale_a=0.5, scale_b=0.25, cta_pair=True, bn=512)
    torch.cuda.synchronize()
    for i in range(nb):
        want = oracle.gemm(oracle.generate_real(f"a{i}", (M, K)), oracle.generate_real(f"b{i}", (N, K)), scale=0.125)
        assert torch.equal(c[i], torch.from_numpy(want).to(dev).to(BF16)), i


@pytest.mark.parametrize("M,N,K,out_dt,kw", [
    (8192, 4096, 2048, F32, dict(cta_pair=True, bn=512)),     # 256 tiles over 74 pairs: a partial last wave
    (8192, 4096, 2048, BF16, dict(cta_pair=True, bn=512)),    # the early-release path, 16-bit out
    (4096, 4096, 1024, F32, dict(cta_pair=False, bn=256)),    # 512 single-CTA tiles over 148 CTAs
    (8192, 4096, 4096, F16, dict(cta_pair=True, bn=512)),
])
def test_partial_last_wave_exact(ws, dev, M, N, K, out_dt, kw):
    """The N-shard shapes of the strong-scaling projection (a partial last wave): exact against the
    oracle (fp32 out; 16-bit out = the oracle rounded once). Every row through the row-sum
    identity, sampled rows element by element, including the last M blocks in raster order."""
    a = ref_tensor("a", (M, K), BF16, dev)
    b = ref_tensor("b", (N, K), BF16, dev)
    c = ws.gemm_tn(a, b, out_dtype=out_dt, **kw)
    torch.cuda.synchronize()
    if out_dt == F32:
        assert torch.equal(c.double().sum(1), a.double() @ b.double().sum(0))
    rows = np.array([0, 255, 256, M // 2, M - 257, M - 256, M - 129, M - 1]
                    + list(np.random.default_rng(K).integers(0, M, 8)))
    want = _want(M, N, K, rows=rows)
    got = c[torch.from_numpy(rows).to(dev)]
    if out_dt == F32:
        assert np.array_equal(as_f64(got), want)
    else:
        assert torch.equal(got, torch.from_numpy(want).to(dev).to(out_dt))


def test_prepared_launch_and_cuda_graph(ws, dev):
    """Repeated calls go through a cached prepared launch (ws_gemm_plan_*) and capture into a CUDA
    graph: replaying the graph gives the bit-exact result again (C1 shape, fp32 out)."""
    a = ref_tensor("a", (1024, 1024), F16, dev)
    b = ref_tensor("b", (1024, 1024), F16, dev)
    c = torch.empty(1024, 1024, dtype=F32, device=dev)
    want = _want(1024, 1024, 1024)
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        ws.gemm_tn(a, b, c)
        with torch.cuda.graph(g, stream=side):
            for _ in range(3):
                ws.gemm_tn(a, b, c)
    torch.cuda.current_stream(dev).wait_stream(side)
    c.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert np.array_equal(as_f64(c), want)
    n0 = ws.launch_count()
    for _ in range(5):
        ws.gemm_tn(a, b, c)
    torch.cuda.synchronize()
    assert ws.launch_count() - n0 == 5
    assert np.array_equal(as_f64(c), want)


def test_plan_api_directly(ws, dev):
    """ws_gemm_plan_create / launch / destroy through ctypes, as a C caller would use them."""
    import ctypes

    lib = ws._lib.load()
    a = ref_tensor("a", (256, 512), BF16, dev)
    b = ref_tensor("b", (256, 512), BF16, dev)
    c = torch.empty(256, 256, dtype=F32, device=dev)
    d = ws._lib.GemmDesc(in_dtype=ws._lib.WS_BF16, out_dtype=ws._lib.WS_F32, M=256, N=256, K=512,
                         A=a.data_ptr(), lda=512, B=b.data_ptr(), ldb=512, C=c.data_ptr(), ldc=256,
                         scale_a=1.0, scale_b=1.0, persistent=1)
    plan = ctypes.c_void_p()
    assert lib.ws_gemm_plan_create(ctypes.byref(d), ctypes.byref(plan)) == 0
    s = torch.cuda.current_stream(dev).cuda_stream
    for _ in range(2):
        assert lib.ws_gemm_plan_launch(plan, s) == 0
    torch.cuda.synchronize()
    lib.ws_gemm_plan_destroy(plan)
    assert np.array_equal(as_f64(c), _want(256, 256, 512))


def test_repeat_call_fast_path_tracks_every_operand_property(ws, dev):
    """gemm_tn's repeat-call path reuses a prepared launch only for the same addresses, shapes,
    strides, dtypes and knobs: views over the same storage with a different shape or stride, a new
    scale, and an out of another dtype each get their own validated plan (results stay exact), and
    an invalid view at a cached address is still rejected."""
    a = ref_tensor("a", (512, 1024), BF16, dev)
    b = ref_tensor("b", (512, 1024), BF16, dev)
    c = torch.empty(512, 512, dtype=F32, device=dev)
    want = _want(512, 512, 1024)
    for _ in range(2):  # the second call takes the fast path
        ws.gemm_tn(a, b, c)
        torch.cuda.synchronize()
        assert np.array_equal(as_f64(c), want)
    # same storage, half the rows (same data_ptr, other shape)
    c2 = torch.empty(256, 512, dtype=F32, device=dev)
    ws.gemm_tn(a[:256], b, c2)
    torch.cuda.synchronize()
    assert np.array_equal(as_f64(c2), want[:256])
    # same pointers, other scale: the plan must not be reused
    ws.gemm_tn(a, b, c, scale_a=0.5)
    torch.cuda.synchronize()
    assert np.array_equal(as_f64(c), want * 0.5)
    ws.gemm_tn(a, b, c)
    torch.cuda.synchronize()
    assert np.array_equal(as_f64(c), want)
    # out at the same address reinterpreted as bf16 (other dtype): tolerance of the 16-bit output
    c16 = c.view(torch.bfloat16)[:, :512]
    ws.gemm_tn(a, b, c16)
    torch.cuda.synchronize()
    assert rel_err(as_f64(c16), want) <= 1e-2
    # same storage viewed with K-stride 2 (not row-major): still rejected after the cached calls
    bad = a.as_strided((512, 512), (1024, 2))
    with pytest.raises(ws.WsError):
        ws.gemm_tn(bad, b[:, :512], c)


def test_clock_probe_sums_every_probed_launch(ws, dev):
    """ws_debug_gemm_clock: CTA 0's %clock64 / %globaltimer spans are summed over every probed
    launch (clk[4], clk[5]) with a launch count (clk[6]); the mean clock they give is a plausible
    SM clock, and launches after the probe is turned off leave the buffer alone."""
    import ctypes

    lib = ws._lib.load()
    a = ref_tensor("a", (1024, 2048), BF16, dev)
    b = ref_tensor("b", (1024, 2048), BF16, dev)
    c = torch.empty(1024, 1024, dtype=F32, device=dev)
    clk = torch.zeros(8, dtype=torch.int64, device=dev)
    ws.gemm_tn(a, b, c)  # plan built before probing
    torch.cuda.synchronize()
    lib.ws_debug_gemm_clock(ctypes.c_void_p(clk.data_ptr()))
    try:
        for _ in range(3):
            ws.gemm_tn(a, b, c)
        torch.cuda.synchronize()
    finally:
        lib.ws_debug_gemm_clock(None)
    v = clk.cpu().tolist()
    assert v[6] == 3
    assert v[2] > v[0] and v[3] > v[1]
    ghz = v[4] / v[5]
    assert 0.3 < ghz < 2.5, ghz
    ws.gemm_tn(a, b, c)
    torch.cuda.synchronize()
    assert clk.cpu().tolist() == v
    assert np.array_equal(as_f64(c), _want(1024, 1024, 2048))
