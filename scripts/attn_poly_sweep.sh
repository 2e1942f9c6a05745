#!/bin/bash
# exp-mix sweep of the 128-key attention kernel (developer script, run under gpurun)
for P in 1 2 3 4; do echo POLY=$P; WS_ATTN_POLY=$P python -c "
import sys; sys.path.insert(0,'scripts'); import gpu_quick_attn as g
for S in (1024,16384): g.bench(16384//S,16,S,128,False,kv_block=128)
g.bench(1,16,16384,128,True,kv_block=128); g.bench(1,16,16384,64,True,kv_block=128); g.bench(1,16,16384,64,False,kv_block=128)
"; done
