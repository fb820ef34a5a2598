set -u
out=gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "conv1 or front_end or pool or network or long_channel" > $out/pytest_r2j.log 2>&1; echo "tests rc=$?"; tail -3 $out/pytest_r2j.log
timeout 300 python tools/c4_kernels.py > $out/c4_kernels_r2j.json 2>/dev/null; echo "c4k rc=$?"; head -c 1500 $out/c4_kernels_r2j.json; echo
timeout 600 python bench.py --config C4 --no-cpu > $out/bench_C4_r2j.json 2>$out/bench_C4_r2j.err; echo "C4 rc=$?"; head -c 400 $out/bench_C4_r2j.json; echo
