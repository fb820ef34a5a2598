set -u
out=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu_r2g.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu_r2g.log
for b in 1 0 1 0; do
  XNC_UMMA_V4=$b timeout 300 python tools/umma_sweep.py --cfgs C3,C2k3,C2k5,C2k7 --reps 30 | sed "s/^/v4=$b /"
done 2>&1 | tee $out/v4_ab_r2g.log
XNC_UMMA_V4=1 timeout 300 python tools/umma_sweep.py --cfgs C3,C2k3 --debug 128 --reps 10 2>&1 | tee -a $out/v4_ab_r2g.log
timeout 300 python tools/c4_kernels.py > $out/c4_kernels_r2g.json 2>/dev/null; echo "c4k rc=$?"; head -c 900 $out/c4_kernels_r2g.json; echo
