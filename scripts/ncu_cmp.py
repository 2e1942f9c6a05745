"""Side-by-side raw metrics of two ncu reports (first launch of each), read here without a GPU.
  python scripts/ncu_cmp.py A.ncu-rep B.ncu-rep [regex ...]"""
import csv, io, re, subprocess, sys


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


a, b = raw(sys.argv[1]), raw(sys.argv[2])
pats = sys.argv[3:] or [r"^gpu__time_duration.sum$", r"^sm__cycles_elapsed.avg.per_second$", r"^sm__cycles_elapsed.max$",
                        r"^dram__bytes_(read|write).sum$", r"^lts__t_sectors_srcunit_(tex|ltcfabric).sum$",
                        r"^lts__t_sectors.sum$", r"^l1tex__m_xbar2l1tex_read_bytes.sum$", r"^smsp__inst_executed.sum$",
                        r"^sm__pipe_tensor.*realtime.avg.pct_of_peak_sustained_elapsed$", r"^launch__(grid|block|cluster).*",
                        r"^lts__t_sector_hit_rate.pct$", r"^sm__throughput.avg.pct", r"^lts__throughput.avg.pct",
                        r"^smsp__inst_executed_op_tma_ld.sum$", r"^l1tex__m_l1tex2xbar_write_bytes.sum$",
                        r"^lts__t_requests_srcunit_tex.sum$", r"smsp__sass_inst_executed_op_utcmma.sum"]
keys = [k for k in a if any(re.search(p, k) for p in pats)]
print(f"{'metric':75s} {'A':>18s} {'B':>18s}")
for k in keys:
    va, ua = a.get(k, ("-", ""))
    vb, ub = b.get(k, ("-", ""))
    print(f"{k[:75]:75s} {va:>14s} {ua:3s} {vb:>14s} {ub:3s}")
print("A:", a.get("Kernel Name", ("?",))[0][:90]); print("B:", b.get("Kernel Name", ("?",))[0][:90])
