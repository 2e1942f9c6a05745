"""Per-region warp-stall breakdown from an ncu source page (SASS), read here without a GPU.

  ncu -i X.ncu-rep --page source --csv --print-source sass > src.csv
  python scripts/ncu_stalls.py src.csv [--top N]
Regions are split at instructions matching a marker (LDTM/STTM/MUFU/SYNCS...) so the softmax
phases, the MMA issue loop and the producer can be told apart; prints stall reasons per region
and the top instructions by samples."""
import csv, re, sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    samples = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ex = int(r[ix["Instructions Executed"]] or 0)
    st = {h: int(r[ix[h]] or 0) for h in stall_cols}
    data.append((r[ix["Address"]], src, samples, ex, st))
tot = sum(d[2] for d in data)
print(f"total samples {tot}, instructions {len(data)}")
agg = Counter()
for d in data:
    agg.update(d[4])
print("all:", ", ".join(f"{k[6:]}={v/tot:.1%}" for k, v in agg.most_common(10)))
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
print(f"--- top {top} instructions by samples")
for i, d in sorted(enumerate(data), key=lambda x: -x[1][2])[:top]:
    st = sorted(d[4].items(), key=lambda kv: -kv[1])[:3]
    print(f"{i:5d} {d[2]/tot:6.2%} ex={d[3]:9d} {d[1][:70]:70s} " + " ".join(f"{k[6:]}={v}" for k, v in st))
# opcode class totals
cls = defaultdict(lambda: [0, 0])
for d in data:
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]+)", d[1])
    op = m.group(2) if m else "?"
    cls[op][0] += d[2]
    cls[op][1] += d[3]
print("--- samples by opcode")
for op, (s, e) in sorted(cls.items(), key=lambda kv: -kv[1][0])[:25]:
    print(f"  {op:12s} {s/tot:6.2%} executed={e}")
