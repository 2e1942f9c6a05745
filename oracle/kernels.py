"""`.k` kernel instances for the hot path, in the reference grammar (ref SPEC.md:120-134,
ref proj/include/warpspec/parse.hpp:412-686). TEST INFRASTRUCTURE: these are the checker's
inputs, the analogue of the reference fixtures (ref proj/tests/support/fixtures.hpp:14-145).

gemm_src      — real-valued gemm.k (ref proj/kernels/gemm.k:2-17): c = a . b^T, pid column-major
                over TM x TN output tiles (pm = pid mod TM, pn = pid div TM).
gemm_src(elem="int") — the shipped integer form (the reference fixture gemm_tiled_src shape).
flash_src     — FlashAttention forward of SURVEY.md Appendix A (batched over B*H slices, causal via
                the mask bank `mb`), emitting acc, row sum l and running max m.
"""
from __future__ import annotations

import math


def gemm_src(M: int, N: int, K: int, BM: int, BN: int, BK: int, elem: str = "real",
             scale: float | None = None) -> str:
    assert M % BM == 0 and N % BN == 0 and K % BK == 0
    tm = M // BM
    lines = [
        f"kernel gemm(a: buf<{M}x{K} {elem}>, b: buf<{N}x{K} {elem}>, c: buf<{M}x{N} {elem}>) {{",
        "  %p = pid",
        f"  %pm = mod %p, {tm}",
        f"  %pn = div %p, {tm}",
        f"  %r = mul %pm, {BM}",
        f"  %cn = mul %pn, {BN}",
        f"  %z = const zeros : {BM}x{BN} {elem}",
        "  %k0 = const 0",
    ]
    if scale is not None:
        lines.append(f"  %s = const [[{scale!r}]] : 1x1 {elem}")
    lines += [
        f"  loop %k in 0..{K // BK} iter (%acc = %z, %ok = %k0) {{",
        f"    %ta = tma_load a[%r, %ok] : {BM}x{BK} {elem}",
        f"    %tb = tma_load b[%cn, %ok] : {BN}x{BK} {elem}",
        "    %acc1 = dot %ta, %tb.T, acc=%acc",
        f"    %ok1 = add %ok, {BK}",
        "    yield %acc1, %ok1",
        "  }",
    ]
    if scale is not None:
        lines += ["  %o = ew mul %acc, %s", "  store c[%r, %cn] = %o"]
    else:
        lines.append("  store c[%r, %cn] = %acc")
    lines.append("}")
    return "\n".join(lines) + "\n"


def gemm_tiles(M: int, N: int, BM: int, BN: int) -> int:
    return (M // BM) * (N // BN)


def flash_src(BH: int, S: int, D: int, BR: int, causal: bool, scale: float | None = None) -> str:
    """Batched flash .k over (B*H*S) x D rows; pid = bh * (S/BR) + query block (BR == BC)."""
    BC = BR
    nqb = S // BR
    rows = BH * S
    sc = scale if scale is not None else 1.0 / math.sqrt(D)
    L = [
        f"kernel flash(q: buf<{rows}x{D} real>, k: buf<{rows}x{D} real>, v: buf<{rows}x{D} real>, "
        f"mb: buf<{BR}x{3 * BC} real>, o: buf<{rows}x{D} real>, lsum: buf<{rows}x1 real>, "
        f"mx: buf<{rows}x1 real>) {{",
        "  %p = pid",
        f"  %bh = div %p, {nqb}",
        f"  %qb = mod %p, {nqb}",
        f"  %r = mul %p, {BR}",
        f"  %kvb = mul %bh, {S}",
        f"  %zacc = const zeros : {BR}x{D} real",
        f"  %zc = const zeros : {BR}x1 real",
        "  %ninf = const [[-1000000.0]] : 1x1 real",
        "  %m0 = ew add %zc, %ninf",
        f"  %sc = const [[{sc!r}]] : 1x1 real",
        "  %k0 = const 0",
    ]
    if not causal:
        L.append(f"  %zs = const zeros : {BR}x{BC} real")
    L.append(f"  loop %j in 0..{S // BC} iter (%acc = %zacc, %m = %m0, %l = %zc, %ok = %kvb) {{")
    L.append(f"    %tq = tma_load q[%r, 0] : {BR}x{D} real")
    L.append(f"    %tk = tma_load k[%ok, 0] : {BC}x{D} real")
    if causal:
        # sel = x/NB + (x-1)/NB with x = j - qb + NB: 0 below, 1 on, 2 above the diagonal
        L += [
            "    %x0 = sub %j, %qb",
            f"    %x = add %x0, {nqb}",
            f"    %s0 = div %x, {nqb}",
            "    %xm = sub %x, 1",
            f"    %s1 = div %xm, {nqb}",
            "    %sel = add %s0, %s1",
            f"    %mc = mul %sel, {BC}",
            f"    %tm = tma_load mb[0, %mc] : {BR}x{BC} real",
            "    %s = dot %tq, %tk.T, acc=%tm",
        ]
    else:
        L.append("    %s = dot %tq, %tk.T, acc=%zs")
    L += [
        f"    %tv = tma_load v[%ok, 0] : {BC}x{D} real",
        "    %ss = ew mul %s, %sc",
        "    %rm = reduce max %ss axis=1",
        "    %mn = ew max %m, %rm",
        "    %d = ew sub %ss, %mn",
        "    %pp = ew exp %d",
        "    %dm = ew sub %m, %mn",
        "    %al = ew exp %dm",
        "    %rs = reduce add %pp axis=1",
        "    %la = ew mul %l, %al",
        "    %l1 = ew add %la, %rs",
        "    %as = ew mul %acc, %al",
        "    %acc1 = dot %pp, %tv, acc=%as",
        f"    %ok1 = add %ok, {BC}",
        "    yield %acc1, %mn, %l1, %ok1",
        "  }",
        "  store o[%r, 0] = %acc",
        "  store lsum[%r, 0] = %l",
        "  store mx[%r, 0] = %m",
        "}",
    ]
    return "\n".join(L) + "\n"


def flash_mask_bank(BR: int):
    """The causal mask bank [0 | lower-tri(0)/upper(-1e7) | -1e7]."""
    import numpy as np
    BC = BR
    mb = np.zeros((BR, 3 * BC))
    for r in range(BR):
        for c in range(BC):
            if c > r:
                mb[r, BC + c] = -1e7
    mb[:, 2 * BC:] = -1e7
    return mb


def flash_block_src(S: int, D: int, BR: int, scale: float | None = None, causal: bool = False, qb: int = 0) -> str:
    """Panel-local flash .k: ONE BR-row query block against S keys (q is only BR rows), the unit
    the CPU baseline times so per-pid whole-buffer copies (ref interp.hpp:140-154) do not
    dominate (CPU baseline plan). causal: the block sits at query-block position qb
    and takes its score accumulator from the mask bank `mb` exactly as the batched causal .k
    (SURVEY App. A selector sel = x/NB + (x-1)/NB, x = j - qb + NB); like the reference, it
    masks instead of skipping, so its cost does not depend on qb."""
    BC = BR
    sc = scale if scale is not None else 1.0 / math.sqrt(D)
    nb = S // BC
    mb_param = f", mb: buf<{BR}x{3 * BC} real>" if causal else ""
    if causal:
        qk = [f"    %x0 = sub %j, {qb}", f"    %x = add %x0, {nb}", f"    %s0 = div %x, {nb}",
              "    %xm = sub %x, 1", f"    %s1 = div %xm, {nb}", "    %sel = add %s0, %s1",
              f"    %mc = mul %sel, {BC}", f"    %tm = tma_load mb[0, %mc] : {BR}x{BC} real",
              "    %s = dot %tq, %tk.T, acc=%tm"]
    else:
        qk = ["    %s = dot %tq, %tk.T, acc=%zs"]
    return "\n".join([
        f"kernel flash_block(q: buf<{BR}x{D} real>, k: buf<{S}x{D} real>, v: buf<{S}x{D} real>{mb_param}, "
        f"o: buf<{BR}x{D} real>, lsum: buf<{BR}x1 real>, mx: buf<{BR}x1 real>) {{",
        f"  %zacc = const zeros : {BR}x{D} real",
        f"  %zc = const zeros : {BR}x1 real",
        "  %ninf = const [[-1000000.0]] : 1x1 real",
        "  %m0 = ew add %zc, %ninf",
        f"  %sc = const [[{sc!r}]] : 1x1 real",
        "  %k0 = const 0",
        f"  %zs = const zeros : {BR}x{BC} real",
        f"  loop %j in 0..{S // BC} iter (%acc = %zacc, %m = %m0, %l = %zc, %ok = %k0) {{",
        f"    %tq = tma_load q[0, 0] : {BR}x{D} real",
        f"    %tk = tma_load k[%ok, 0] : {BC}x{D} real",
        *qk,
        f"    %tv = tma_load v[%ok, 0] : {BC}x{D} real",
        "    %ss = ew mul %s, %sc",
        "    %rm = reduce max %ss axis=1",
        "    %mn = ew max %m, %rm",
        "    %d = ew sub %ss, %mn",
        "    %pp = ew exp %d",
        "    %dm = ew sub %m, %mn",
        "    %al = ew exp %dm",
        "    %rs = reduce add %pp axis=1",
        "    %la = ew mul %l, %al",
        "    %l1 = ew add %la, %rs",
        "    %as = ew mul %acc, %al",
        "    %acc1 = dot %pp, %tv, acc=%as",
        f"    %ok1 = add %ok, {BC}",
        "    yield %acc1, %mn, %l1, %ok1",
        "  }",
        "  store o[0, 0] = %acc",
        "  store lsum[0, 0] = %l",
        "  store mx[0, 0] = %m",
        "}",
    ]) + "\n"


def gemm_batched_src(batches: int, T: int, BT: int, K: int, BK: int, elem: str = "int") -> str:
    """gemm_batched.k shape (ref proj/kernels/gemm_batched.k:2-22): `batches` independent T x T x K
    products stacked along rows, BT x BT tiles, pid = batch * (T/BT)^2 + tile."""
    tpb = T // BT
    rows = batches * T
    return "\n".join([
        f"kernel gemm_batched(a: buf<{rows}x{K} {elem}>, b: buf<{rows}x{K} {elem}>, c: buf<{rows}x{T} {elem}>) {{",
        "  %p = pid",
        f"  %bi = div %p, {tpb * tpb}",
        f"  %t = mod %p, {tpb * tpb}",
        f"  %tm = mod %t, {tpb}",
        f"  %tn = div %t, {tpb}",
        f"  %rbase = mul %bi, {T}",
        f"  %tmr = mul %tm, {BT}",
        f"  %tnr = mul %tn, {BT}",
        "  %r = add %rbase, %tmr",
        "  %rb = add %rbase, %tnr",
        f"  %z = const zeros : {BT}x{BT} {elem}",
        "  %k0 = const 0",
        f"  loop %k in 0..{K // BK} iter (%acc = %z, %ok = %k0) {{",
        f"    %ta = tma_load a[%r, %ok] : {BT}x{BK} {elem}",
        f"    %tb = tma_load b[%rb, %ok] : {BT}x{BK} {elem}",
        "    %acc1 = dot %ta, %tb.T, acc=%acc",
        f"    %ok1 = add %ok, {BK}",
        "    yield %acc1, %ok1",
        "  }",
        "  store c[%r, %tnr] = %acc",
        "}",
    ]) + "\n"


def gemm_act_src(M: int, N: int, K: int, BM: int, BN: int, BK: int, elem: str = "int") -> str:
    """gemm_act.k shape (ref proj/kernels/gemm_act.k:2-18): the stored value is relu of the
    accumulator after the last iteration (yielded through %last)."""
    tm = M // BM
    return "\n".join([
        f"kernel gemm_act(a: buf<{M}x{K} {elem}>, b: buf<{N}x{K} {elem}>, c: buf<{M}x{N} {elem}>) {{",
        "  %p = pid",
        f"  %pm = mod %p, {tm}",
        f"  %pn = div %p, {tm}",
        f"  %r = mul %pm, {BM}",
        f"  %cn = mul %pn, {BN}",
        f"  %z = const zeros : {BM}x{BN} {elem}",
        "  %k0 = const 0",
        f"  loop %k in 0..{K // BK} iter (%acc = %z, %last = %z, %ok = %k0) {{",
        f"    %ta = tma_load a[%r, %ok] : {BM}x{BK} {elem}",
        f"    %tb = tma_load b[%cn, %ok] : {BN}x{BK} {elem}",
        "    %acc1 = dot %ta, %tb.T, acc=%acc",
        "    %rl = ew relu %acc1",
        f"    %ok1 = add %ok, {BK}",
        "    yield %acc1, %rl, %ok1",
        "  }",
        "  store c[%r, %cn] = %last",
        "}",
    ]) + "\n"


def shipped(name: str, root: str = "/root/reference/proj/kernels") -> str:
    """A `.k` file shipped with the reference, verbatim (golden generation only: /root/reference
    exists in the build container, not on the GPU box; the text is stored in the golden)."""
    with open(f"{root}/{name}") as f:
        return f.read()


def maxshift_src(R: int, D: int, S: int, BR: int, DV: int | None = None, elem: str = "int") -> str:
    """The shipped max-shift attention.k (ref proj/kernels/attention.k:1-21) at other sizes: q R x D,
    kt D x S, v S x DV, o R x DV; pid = query block of BR rows; iteration j takes the D x D key tile
    kt[0, j*D] and the D x DV value tile v[j*D, 0] (the shipped file is R=32, D=8, S=64, BR=8)."""
    DV = DV or D
    assert R % BR == 0 and S % D == 0
    return "\n".join([
        f"kernel attention(q: buf<{R}x{D} {elem}>, kt: buf<{D}x{S} {elem}>, v: buf<{S}x{DV} {elem}>, "
        f"o: buf<{R}x{DV} {elem}>) {{",
        "  %p = pid",
        f"  %r = mul %p, {BR}",
        f"  %zs = const zeros : {BR}x{D} {elem}",
        f"  %zacc = const zeros : {BR}x{DV} {elem}",
        "  %k0 = const 0",
        f"  loop %k in 0..{S // D} iter (%acc = %zacc, %ok = %k0) {{",
        f"    %tq = tma_load q[%r, 0] : {BR}x{D} {elem}",
        f"    %tk = tma_load kt[0, %ok] : {D}x{D} {elem}",
        f"    %tv = tma_load v[%ok, 0] : {D}x{DV} {elem}",
        "    %s = dot %tq, %tk.T, acc=%zs",
        "    %m = reduce max %s axis=1",
        "    %sub = ew sub %s, %m",
        "    %acc1 = dot %sub, %tv, acc=%acc",
        f"    %ok1 = add %ok, {D}",
        "    yield %acc1, %ok1",
        "  }",
        "  store o[%r, 0] = %acc",
        "}",
        "",
    ])
