for P in 2 3 4 5; do WS_ATTN_POLY=$P timeout 200 python scripts/attn_trace.py 2>&1 | grep median | head -1 | sed "s/^/POLY=$P /"; done
for P in 2 3 4 5; do WS_ATTN_POLY=$P timeout 200 python -c "
import sys; sys.path.insert(0,'.'); sys.argv=['x']
exec(open('scripts/gpu_quick_attn.py').read().split('if __name__')[0])
bench(1,16,16384,128,False); bench(1,16,16384,128,True)" | sed "s/^/POLY=$P /"; done
