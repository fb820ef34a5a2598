#!/usr/bin/env bash
# One gpurun session: tests, smoke, bench, ncu launch list + full capture.
# Usage (under gpurun): bash tools/gpu_round.sh <tag> [what...]
#   what: tests smoke bench bench-quick c4 ncu-launch ncu-conv ncu-pack sanitize (default: the
#   first six of tests smoke bench ncu-launch ncu-conv ncu-pack)
set -u
tag=${1:-r1}; shift || true
what=${*:-"tests smoke bench ncu-launch ncu-conv ncu-pack"}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $out/gpu_$tag.txt 2>&1
for w in $what; do
  case $w in
    tests) timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" ;;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke_$tag.log 2>&1; echo "smoke rc=$?" ;;
    bench) timeout 900 python bench.py > $out/bench_$tag.json 2> $out/bench_$tag.err; echo "bench rc=$?"; cat $out/bench_$tag.json ;;
    bench-quick) timeout 600 python bench.py --no-cpu --no-ksweep > $out/benchq_$tag.json 2> $out/benchq_$tag.err; echo "benchq rc=$?"; cat $out/benchq_$tag.json ;;
    c4) timeout 600 python bench.py --config C4 --no-cpu > $out/bench_C4_$tag.json 2> $out/bench_C4_$tag.err; echo "C4 rc=$?"
        timeout 900 python bench.py --config C5 --no-cpu > $out/bench_C5_$tag.json 2> $out/bench_C5_$tag.err; echo "C5 rc=$?"
        timeout 300 python tools/c4_launches.py 256 > $out/c4_launches_256_$tag.json 2>/dev/null; echo "c4 launches rc=$?" ;;
    sanitize) SAN_TIMEOUT=900 bash tools/sanitize.sh $tag memcheck synccheck racecheck ;;
    ncu-launch) timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
        --log-file $out/launches_$tag.csv python bench.py --steps 3 --warmup 3 --no-cpu --no-ksweep > /dev/null 2>&1; echo "ncu-launch rc=$?" ;;
    ncu-conv) timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_conv -s 3 -c 1 \
        -o $out/conv_$tag -f python bench.py --steps 2 --warmup 3 --no-cpu --no-ksweep > $out/ncu_conv_$tag.log 2>&1; echo "ncu-conv rc=$?" ;;
    ncu-pack) timeout 600 ncu --set full --clock-control none -k regex:k_pack_input -s 3 -c 1 \
        -o $out/pack_$tag -f python bench.py --steps 2 --warmup 3 --no-cpu --no-ksweep > $out/ncu_pack_$tag.log 2>&1; echo "ncu-pack rc=$?" ;;
  esac
done
