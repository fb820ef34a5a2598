set -u
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python tools/c4_launches.py 256 > gpurun_out/c4_launches_256_r3c.json 2>/dev/null; echo rc=$?
timeout 600 python bench.py --config C4 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('C4',d['ms_per_step'])"
timeout 900 python bench.py --config C5 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('C5',d['ms_per_step'])"
