set -u
out=gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "conv1 or front_end" > $out/pytest_conv1_r2f.log 2>&1; echo "conv1 tests rc=$?"; tail -2 $out/pytest_conv1_r2f.log
timeout 300 python tools/c4_kernels.py > $out/c4_kernels_r2f.json 2>/dev/null; echo "c4k rc=$?"; head -c 700 $out/c4_kernels_r2f.json; echo
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv1_tf32 -s 2 -c 1 -o $out/conv1_r2f -f python tools/c4_kernels.py > $out/ncu_conv1_r2f.log 2>&1; echo "ncu conv1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_absmean_wide -s 2 -c 1 -o $out/absw_r2f -f python tools/c4_kernels.py > $out/ncu_absw_r2f.log 2>&1; echo "ncu absw rc=$?"
