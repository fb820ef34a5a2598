# pooled-K1 kernels: parity, C4 per-kernel times, C4 bench, sanitizers on the pool cases
out=gpurun_out; tag=${1:-r4d}
timeout 600 python -m pytest tests -x -q -m gpu -k "pooled or network or in_pool" > $out/pytest_pool_$tag.log 2>&1; echo "pytest rc=$?"; tail -3 $out/pytest_pool_$tag.log
timeout 300 python tools/c4_launches.py 256 > $out/c4_launches_256_$tag.json 2>/dev/null; echo "c4 launches rc=$?"
python - <<PY
import json
d=json.load(open("$out/c4_launches_256_$tag.json"))
for t0,us,name in d["launches"]: print(f"{us:8.1f}  {name[:90]}")
print("total", d["total_us"])
PY
timeout 600 python bench.py --config C4 --no-cpu > $out/bench_C4_$tag.json 2> $out/bench_C4_$tag.err; echo "C4 rc=$?"; cut -c1-400 $out/bench_C4_$tag.json
for t in memcheck racecheck; do
  extra=""; [ "$t" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 600 /usr/local/cuda/bin/compute-sanitizer --tool $t $extra --kernel-name regex=xnc --target-processes application-only \
     python tools/sanitize_cases.py pool_k1 > $out/sanitize_${t}_pool_$tag.log 2>&1; echo "$t rc=$? $(grep -h SUMMARY $out/sanitize_${t}_pool_$tag.log | tail -1)"
done
