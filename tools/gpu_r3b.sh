for d in 0 1 2 4 3 6 7; do XNC_CONV1_DEBUG=$d timeout 120 python tools/conv1_probe2.py; done 2>&1 | tee gpurun_out/conv1_debug_r3b.log
