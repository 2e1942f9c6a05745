"""Reduce one dp_sweep ncu report to a JSON row (runs where the .ncu-rep is, e.g. on the GPU box):
tensor-pipe activity, DRAM bytes / achieved GB/s, duration, SM clock, and the share of warp-state
samples spent in mbarrier waits (SYNCS.PHASECHK try-wait instructions and the retry branch that
follows each), overall and for the softmax / epilogue warps vs the producer / MMA warps is not
separable from SASS alone, so it is reported for the whole kernel.

  python scripts/dp_sweep_report.py X.ncu-rep  -> prints {"id": ..., ...}
"""
import csv
import io
import json
import os
import re
import subprocess
import sys


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return {}
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


def num(d, k, scale=None):
    if k not in d:
        return None
    v, u = d[k]
    try:
        f = float(v.replace(",", ""))
    except ValueError:
        return None
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1,
            "Ghz": 1e9, "Mhz": 1e6, "hz": 1}.get(u, 1)
    return f * mult


def syncs_share(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    for i, r in enumerate(rows[:5]):
        if "Source" in r and "Warp Stall Sampling (All Samples)" in r:
            hdr, start = r, i + 1
            break
    if hdr is None:
        return None
    ix = {h: i for i, h in enumerate(hdr)}
    tot = wait = 0
    prev_syncs = False
    for r in rows[start:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]]
        n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        tot += n
        is_syncs = "SYNCS.PHASECHK" in src
        if is_syncs or (prev_syncs and re.search(r"\bBRA\b", src)):
            wait += n
        prev_syncs = is_syncs
    return wait / tot if tot else None


def main():
    path = sys.argv[1]
    d = raw(path)
    t = num(d, "gpu__time_duration.sum")
    rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
    row = {"id": os.path.basename(path).replace(".ncu-rep", ""),
           "duration_ms": round(t * 1e3, 4) if t else None,
           "sm_clock_ghz": round(num(d, "sm__cycles_elapsed.avg.per_second") / 1e9, 3)
           if num(d, "sm__cycles_elapsed.avg.per_second") else None,
           "tensor_pipe_pct": num(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
           "dram_bytes": (rd or 0) + (wr or 0),
           "dram_gbs": round(((rd or 0) + (wr or 0)) / t / 1e9, 1) if t else None,
           "mbarrier_wait_sample_share": syncs_share(path)}
    print(json.dumps(row))


if __name__ == "__main__":
    main()
