"""Summarise an ncu --set full report (read here, no GPU): key metrics per kernel launch.

  python scripts/ncu_summary.py gpurun_out/prof_gemm.ncu-rep [--json key] [--details]
"""
import csv, io, json, subprocess, sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "launch__registers_per_thread", "smsp__inst_executed_pipe_xu.sum", "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum", "launch__grid_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]

def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, vals):
            d[h] = (v, u)
        res.append(d)
    return res

def details(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    i_sec, i_name, i_unit, i_val = (hdr.index(x) for x in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    return [(r[i_sec], r[i_name], r[i_unit], r[i_val]) for r in rows[1:] if len(r) > i_val and r[i_name]]

def to_bytes(v, u):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)

if __name__ == "__main__":
    path = sys.argv[1]
    for i, d in enumerate(raw(path)):
        print(f"--- launch {i}: {d.get('Kernel Name', ('?',))[0][:100]}")
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k][0]} {d[k][1]}")
        rd = to_bytes(*d["dram__bytes_read.sum"]); wr = to_bytes(*d["dram__bytes_write.sum"])
        print(f"  dram bytes per launch = {rd + wr:.4e}")
        if "--json" in sys.argv:
            key = sys.argv[sys.argv.index("--json") + 1]
            print(json.dumps({key: {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                                    "duration_ms": float(d["gpu__time_duration.sum"][0]) if d["gpu__time_duration.sum"][1] == "ms" else None}}))
    if "--details" in sys.argv:
        for sec, name, unit, val in details(path):
            print(f"  [{sec}] {name} = {val} {unit}")
