set -u
out=gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "pool or network" 2>&1 | tail -2
for v in 1; do XNC_POOL_K1=$v timeout 300 python tools/c4_kernels.py 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('POOL_K1=$v total', d['total_us'], [(t,n,k[:40]) for t,n,k in d['us_per_forward'] if 'pool' in k or 'pack_small' in k])"; done
