#!/usr/bin/env bash
# compute-sanitizer over every kernel family of libxnorb200.so (under gpurun).
# Runs the small-shape GPU parity tests (drop-in seams, K1/K2, popc/b1mma/tcgen05
# convs incl. the sign-emitting, split-K and fc forms, network data movement) with
# each tool, instrumenting only this library's kernels (mangled names carry the
# `xnc` namespace).  Logs: gpurun_out/sanitize_<tool>_<tag>.log
# Usage: bash tools/sanitize.sh <tag> [tools...]
set -u
tag=${1:-r2}; shift || true
tools=${*:-"memcheck initcheck synccheck racecheck"}
out=gpurun_out
mkdir -p $out
sel="not full_size and not tcgen05_at_c3 and not 256 and not large and not two_devices and not host_threads and not c1_full"
for t in $tools; do
  extra=""
  [ "$t" = "memcheck" ] && extra="--leak-check no --padding 32"
  [ "$t" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $t $extra --kernel-name regex=xnc \
      --print-limit 50 --target-processes application-only \
      python -m pytest tests/test_gpu_dropin.py tests/test_gpu_parity.py tests/test_gpu_network.py \
      -m gpu -q -x -p no:cacheprovider -k "$sel" > $out/sanitize_${t}_${tag}.log 2>&1
  echo "$t rc=$? $(grep -h 'ERROR SUMMARY' $out/sanitize_${t}_${tag}.log | tail -1) $(tail -1 $out/sanitize_${t}_${tag}.log)"
done
