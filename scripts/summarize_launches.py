"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel shares.

  python scripts/summarize_launches.py gpurun_out/launches.csv > profiles/launches_r01.md
"""
import csv, collections, re, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0] != "ID"]
tot = collections.defaultdict(float); cnt = collections.Counter(); grids = {}
for r in rows:
    name = r[4]
    short = re.sub(r"\(.*", "", name)
    short = short.replace("void ", "")
    if "ws_gemm" in name or "ws_attn" in name:
        m = re.search(r"(ws_\w+)<([^>]*)>", name)
        short = f"{m.group(1)}<{m.group(2)}>" if m else short
    else:
        short = short[:60]
    key = (short, r[8])
    tot[key] += float(r[14]); cnt[key] += 1
all_ns = sum(tot.values())
ours = sum(v for (k, g), v in tot.items() if k.startswith("ws_"))
print(f"# ncu launch list: {len(rows)} launches, {all_ns/1e6:.3f} ms total device time; "
      f"our kernels {100*ours/all_ns:.1f}% (cold-cache, serialised replay: compare shares, not absolutes)\n")
print("| kernel | grid | launches | total ms | avg us | share |")
print("|---|---|---|---|---|---|")
for (k, g), v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
    print(f"| `{k}` | {g} | {cnt[(k, g)]} | {v/1e6:.3f} | {v/cnt[(k, g)]/1e3:.1f} | {100*v/all_ns:.1f}% |")
