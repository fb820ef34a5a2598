set -u
out=gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "conv1 or front_end or long_channel or network" > $out/pytest_r2i.log 2>&1; echo "tests rc=$?"; tail -3 $out/pytest_r2i.log
timeout 300 python tools/c4_kernels.py > $out/c4_kernels_r2i.json 2>/dev/null; echo "c4k rc=$?"; head -c 1200 $out/c4_kernels_r2i.json; echo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv1_tf32 -s 2 -c 1 -o $out/conv1_r2i -f python tools/c4_kernels.py > $out/ncu_conv1_r2i.log 2>&1; echo "ncu conv1 rc=$?"
