#!/bin/bash
# correctness + speed of the attention variants (developer script, run under gpurun)
echo "== P in shared memory (default)"; KVB=128 timeout 300 python scripts/gpu_quick_attn.py 2>&1 | grep -v "flash_attn"
echo "== P in TMEM"; WS_ATTN_PTMEM=1 KVB=128 timeout 300 python scripts/gpu_quick_attn.py 2>&1 | grep BENCH
for P in 1 3; do echo "== psmem POLY=$P"; WS_ATTN_POLY=$P python -c "
import sys; sys.path.insert(0,'scripts'); import gpu_quick_attn as g
for S in (1024,16384): g.bench(16384//S,16,S,128,False,kv_block=128)
g.bench(1,16,16384,128,True,kv_block=128); g.bench(1,16,16384,64,True,kv_block=128); g.bench(1,16,16384,64,False,kv_block=128)
"; done
