set -u
bash tools/gpu_round.sh r2r tests smoke bench ncu-launch ncu-conv
timeout 600 python bench.py --config C4 --no-cpu > gpurun_out/bench_C4_r2r.json 2>/dev/null; echo "C4 rc=$?"
timeout 900 python bench.py --config C5 --no-cpu > gpurun_out/bench_C5_r2r.json 2>/dev/null; echo "C5 rc=$?"
timeout 300 python tools/c4_kernels.py > gpurun_out/c4_kernels_r2r.json 2>/dev/null; echo "c4k rc=$?"
