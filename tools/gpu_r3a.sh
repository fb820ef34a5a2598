set -u
timeout 900 python -m pytest tests -x -q -m gpu -k "random_shapes" 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv1_tf32 -s 2 -c 1 -o gpurun_out/conv1_r3a -f python tools/conv1_probe2.py > gpurun_out/ncu_conv1_r3a.log 2>&1; echo "ncu rc=$?"
