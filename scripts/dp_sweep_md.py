"""Render profiles/r02_dp_sweep.md from the dp_sweep timing JSON and the ncu rows (runs here).

  python scripts/dp_sweep_md.py gpurun_out/r02f/dp_sweep.json gpurun_out/dp/rows.jsonl > profiles/r02_dp_sweep.md
"""
import json
import sys

timing = json.load(open(sys.argv[1]))
ncu = {}
for line in open(sys.argv[2]):
    line = line.strip()
    if line.startswith("{"):
        r = json.loads(line)
        ncu[r["id"].replace("dp_", "", 1)] = r


def fmt(x, nd=1):
    return "—" if x is None else f"{x:.{nd}f}"


print("# D x P x persistent sweep on B200 (round 2)\n")
print("The B200 counterpart of the reference's `cmd_sweep` (ref proj/include/warpspec/driver.hpp:304-335):")
print("one row per (D, P, persistent); cells the reference would refuse are marked with its ErrorCode")
print("(`P > D` -> pipeline-infeasible, ref pipeline.hpp:84-92; shared memory over the 227 KB sm_100a limit ->")
print("smem-overflow, ref sim.hpp:81-84 with the real limit). Paper claim to compare: \"persistent peaks at")
print("D=3, P=2; persistent +5-10%\" (ref PAPER.md:498-504, H100).\n")
print("* Timing (`scripts/dp_sweep.py`): CUDA events, per cell the median of 3 windows of 10 launches, and the")
print("  median over three passes (forward, reverse, forward). The GPU runs power-capped under sustained")
print("  tensor load, so absolute TFLOP/s are sustained-clock numbers; compare cells with each other.")
print("* Counters (`scripts/dp_sweep_ncu.sh` + `scripts/dp_sweep_report.py`, one ncu launch per cell after")
print("  2 warm-ups, `--clock-control none`): tensor pipe = `sm__pipe_tensor_cycles_active` % of elapsed;")
print("  DRAM = (`dram__bytes_read` + `dram__bytes_write`) / `gpu__time_duration`; mbarrier-wait = share of")
print("  warp-state samples on `SYNCS.PHASECHK` try-wait instructions and their retry branch (all warps).\n")
for title, prefix, algo in (("GEMM bf16 8192 x 8192 x 16384, 256x512 CTA-pair tiles", "gemm_bn512", 0.671e9),
                            ("GEMM bf16 8192 x 8192 x 16384, 256x256 CTA-pair tiles", "gemm_bn256", 0.671e9),
                            ("FlashAttention fwd bf16 hdim 128, H=16, S=16K, non-causal (D = K/V aref depth)", "attn_bn128", None),
                            ("FlashAttention fwd FP8 e4m3 hdim 128, H=16, S=16K, non-causal", "attn_fp8_bn128", None)):
    print(f"## {title}\n")
    print("| D | P | persistent | status | TFLOP/s | tensor pipe % | SM GHz (ncu) | DRAM GB/s | DRAM bytes / launch | mbarrier-wait share |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for k, v in timing.items():
        if not k.startswith(prefix + "_D"):
            continue
        parts = k[len(prefix) + 1:].split("_")
        D, P, pers = parts[0][1:], parts[1][1:], parts[2][4:]
        n = ncu.get(k, {})
        st = v["status"]
        print(f"| {D} | {P if prefix.startswith('gemm') else '—'} | {pers} | {st} | {fmt(v.get('tflops'))} | "
              f"{fmt(n.get('tensor_pipe_pct'))} | {fmt(n.get('sm_clock_ghz'), 3)} | {fmt(n.get('dram_gbs'))} | "
              f"{fmt(n.get('dram_bytes') / 1e9 if n.get('dram_bytes') else None, 3)} GB | "
              f"{fmt(100 * n['mbarrier_wait_sample_share'] if n.get('mbarrier_wait_sample_share') is not None else None)} % |")
    if algo:
        print(f"\nAlgorithmic bytes per launch (A + B + C once): {algo / 1e9:.3f} GB.")
    print()
