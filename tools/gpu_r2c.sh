set -u
out=gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -k "abs_mean or reference_backend" > $out/pytest_refbe_r2c.log 2>&1; echo "refbe rc=$?"; tail -3 $out/pytest_refbe_r2c.log
bash tools/sanitize.sh r2c
