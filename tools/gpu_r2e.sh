set -u
out=gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "conv1 or front_end or network" > $out/pytest_conv1_r2e.log 2>&1; echo "conv1 tests rc=$?"; tail -15 $out/pytest_conv1_r2e.log
timeout 300 python tools/c4_kernels.py > $out/c4_kernels_r2e.json 2>&1; echo "c4k rc=$?"; head -c 1500 $out/c4_kernels_r2e.json; echo
timeout 600 python bench.py --config C4 --no-cpu > $out/bench_C4_r2e.json 2>$out/bench_C4_r2e.err; echo "C4 rc=$?"; head -c 600 $out/bench_C4_r2e.json; echo
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu_r2e.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu_r2e.log
SAN_TIMEOUT=600 bash tools/sanitize.sh r2e racecheck memcheck synccheck
