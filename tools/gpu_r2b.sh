set -u
out=gpurun_out
for v in popc b1mma umma; do
  for c in C3 C2k3; do
    timeout 300 python bench.py --config $c --variant $v --no-cpu --no-ksweep --no-strong --steps 20 --warmup 5 > $out/bench_${c}_${v}_r2b.json 2>/dev/null; echo "$c $v rc=$?"
  done
done
timeout 900 python -m pytest tests -x -q -m gpu -k "abs_mean" > $out/pytest_absmean_r2b.log 2>&1; echo "absmean rc=$?"; tail -1 $out/pytest_absmean_r2b.log
bash tools/sanitize.sh r2b
