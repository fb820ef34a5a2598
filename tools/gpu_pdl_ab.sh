# PDL on/off: C3 step (bench quick), C4 network
out=gpurun_out; tag=${1:-r4s}
for i in 1 2 3; do for p in 1 0; do
  XNC_PDL=$p timeout 600 python bench.py --no-cpu --no-ksweep 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('pdl=$p C3',round(d['ms_per_step'],4),d['kernel_ms'],d['clocks']['sm_mhz'])"
  XNC_PDL=$p timeout 600 python bench.py --config C4 --no-cpu 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('pdl=$p C4',round(d['ms_per_step'],4),d['clocks']['sm_mhz'])"
done; done > $out/pdl_ab_$tag.log 2>&1
cat $out/pdl_ab_$tag.log
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
