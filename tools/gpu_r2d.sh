set -u
out=gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > $out/pytest_gpu_r2d.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_gpu_r2d.log
for b in 1 0 1 0; do
  XNC_UMMA_BULK=$b timeout 300 python tools/umma_sweep.py --cfgs C3,C2k3,C2k5,C2k7 --reps 30 | sed "s/^/bulk=$b /"
done 2>&1 | tee $out/bulk_ab_r2d.log
XNC_UMMA_BULK=1 timeout 300 python tools/umma_sweep.py --cfgs C3,C2k3 --debug 128 --reps 10 2>&1 | tee -a $out/bulk_ab_r2d.log
timeout 300 python tools/sanitize_cases.py; echo "cases rc=$?"
bash tools/sanitize.sh r2d memcheck synccheck racecheck initcheck
