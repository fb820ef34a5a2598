set -u
out=gpurun_out
timeout 300 python tools/c4_kernels.py > $out/c4_kernels_r2m.json 2>/dev/null; echo "c4k rc=$?"; head -c 1600 $out/c4_kernels_r2m.json; echo
timeout 600 python bench.py --config C4 --no-cpu > $out/bench_C4_r2m.json 2>$out/bench_C4_r2m.err; echo "C4 rc=$?"; python -c "import json;d=json.loads(open('$out/bench_C4_r2m.json').read().strip().splitlines()[-1]);print('C4',d['ms_per_step'],d.get('images_per_s'))"
timeout 900 python bench.py --config C5 --no-cpu > $out/bench_C5_r2m.json 2>$out/bench_C5_r2m.err; echo "C5 rc=$?"; python -c "import json;d=json.loads(open('$out/bench_C5_r2m.json').read().strip().splitlines()[-1]);print('C5',d['ms_per_step'],d.get('images_per_s'))"
