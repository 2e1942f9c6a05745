"""Per-tile timeline of the persistent GEMM (developer script, GPU): %clock64 stamps of CTA 0 (the
pair leader: producer, MMA issuer, epilogue warps 4 and 8) via ws_debug_gemm_trace.
  python scripts/gemm_trace.py K [json-kwargs]       e.g. 2048 '{"cta_pair":1,"bn":512}'
Events (csrc/gemm_sm100.cuh GT): 0 MMA waits TMEM half 0 / accumulator, 1 got it, 2 half 1 free,
3 half-0 commit, 4 tile's MMAs issued, 5 first K block staged; 6/7/8 epilogue half 0 full /
released / stores issued; 9/10/11 the same for half 1; 12/13 producer first put / last put."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_14719_b200 as ws
from paper_2510_14719_b200 import _lib

K = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
kw = json.loads(sys.argv[2]) if len(sys.argv) > 2 else {"cta_pair": 1, "bn": 512}
a = torch.randn(8192, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(8192, K, device="cuda", dtype=torch.bfloat16)
c = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
lib = _lib.load()
tr = torch.zeros(2 * 32 * 16, dtype=torch.int64, device="cuda")
for _ in range(3):
    ws.gemm_tn(a, b, c, **kw)
lib.ws_debug_gemm_trace(ctypes.c_void_p(tr.data_ptr()))
ws.gemm_tn(a, b, c, **kw)
torch.cuda.synchronize()
lib.ws_debug_gemm_trace(None)
t = tr.view(2, 32, 16).cpu()
base = int(t[0, 0, 12])
names = ["mma_wait0", "mma_got0", "h1_free", "commit0", "issued", "kb0_staged", "e0_full", "e0_rel", "e0_done",
         "e1_full", "e1_rel", "e1_done", "prod_first", "prod_last", "e0_rel_w7", "e0_rel_w11"]
print(f"K={K} {kw}  (cycles from CTA 0's first producer put)")
print("tile " + " ".join(f"{n:>10s}" for n in names) + "   tile_dt  mma_idle")
prev_issued = None
for ti in range(32):
    row = t[0, ti]
    if int(row[12]) == 0:
        break
    vals = [int(row[e]) - base if int(row[e]) else -1 for e in range(16)]
    dt = vals[4] - prev_issued if prev_issued is not None else 0
    idle = vals[1] - vals[0]  # MMA warp blocked on the accumulator hand-over
    print(f"{ti:4d} " + " ".join(f"{v:10d}" for v in vals) + f" {dt:9d} {idle:9d}")
    prev_issued = vals[4]
if os.environ.get("WS_GEMM_TRACE_GLOBAL"):
    # globaltimer (ns) is common to both SMs: the pair's releases on one time line
    off = int(t[0, 0, 12])
    for ti in range(1, 8):
        r0, r1_ = t[0, ti], t[1, ti]
        print(f"tile {ti}: CTA0 e0_full {int(r0[6]) - off} rel(w4,w7,w11) {int(r0[7]) - off} {int(r0[14]) - off} {int(r0[15]) - off}"
              f" | CTA1 e0_full {int(r1_[6]) - off} rel {int(r1_[7]) - off} {int(r1_[14]) - off} {int(r1_[15]) - off}"
              f" | MMA next got0 {int(t[0, ti + 1, 1]) - off} wait0 {int(t[0, ti + 1, 0]) - off}")
r1 = t[1]
print("CTA 1 (its own clock): half 0 full->release of warps 4/7/11, half 1 full->release, per tile:",
      [(int(r1[ti, 7] - r1[ti, 6]), int(r1[ti, 14] - r1[ti, 6]), int(r1[ti, 15] - r1[ti, 6]), int(r1[ti, 10] - r1[ti, 9]))
       for ti in range(8) if int(r1[ti, 12])])
