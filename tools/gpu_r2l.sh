set -u
timeout 600 python -m pytest tests -x -q -m gpu -k "conv1 or front_end" 2>&1 | tail -2
for d in 0 1 4 0; do XNC_CONV1_DEBUG=$d timeout 120 python tools/conv1_probe2.py; done 2>&1 | tee gpurun_out/conv1_debug_r2l.log
