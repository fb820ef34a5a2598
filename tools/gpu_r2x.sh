timeout 300 python tools/c4_launches.py 256 > gpurun_out/c4_launches_256_r2x.json 2>/dev/null; echo rc=$?
timeout 300 python tools/c4_launches.py 2048 > gpurun_out/c4_launches_2048_r2x.json 2>/dev/null; echo rc=$?
