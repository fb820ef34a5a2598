set -u
bash tools/gpu_round.sh r3h tests smoke bench ncu-launch ncu-conv ncu-pack
timeout 600 python bench.py --config C4 --no-cpu > gpurun_out/bench_C4_r3h.json 2>/dev/null; echo "C4 rc=$?"
timeout 900 python bench.py --config C5 --no-cpu > gpurun_out/bench_C5_r3h.json 2>/dev/null; echo "C5 rc=$?"
timeout 300 python tools/c4_kernels.py > gpurun_out/c4_kernels_r3h.json 2>/dev/null; echo "c4k rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r3h.json 2>/dev/null; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_ref_r3h.json
timeout 300 python -m paper_2007_14178_b200 verify --kernels 1,3,5,7 > gpurun_out/cli_verify_r3h.log 2>&1; echo "cli verify rc=$?"; tail -3 gpurun_out/cli_verify_r3h.log
timeout 300 python -m paper_2007_14178_b200 bench --sizes 256,512,1024 --channels 8 --repeats 20 --warmup 3 > gpurun_out/cli_bench_r3h.log 2>&1; echo "cli bench rc=$?"; cat gpurun_out/cli_bench_r3h.log
