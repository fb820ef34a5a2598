#!/usr/bin/env bash
# compute-sanitizer over every kernel family of libxnorb200.so (run under gpurun).
# tools/sanitize_cases.py launches each family once at small shapes and checks the
# results; only this library's kernels are instrumented (mangled names carry the
# `xnc` namespace).  racecheck prints every hazard (--print-limit 0) and
# tools/race_summary.py folds them per kernel and per shared-memory object.
# Logs: gpurun_out/sanitize_<tool>_<tag>.log (+ racecheck summary .txt)
# Usage: bash tools/sanitize.sh <tag> [tools...]
set -u
tag=${1:-r2}; shift || true
tools=${*:-"memcheck initcheck synccheck racecheck"}
out=gpurun_out
mkdir -p $out
for t in $tools; do
  extra="--print-limit 100"
  [ "$t" = "memcheck" ] && extra="--print-limit 100 --padding 32"
  [ "$t" = "racecheck" ] && extra="--print-limit 0 --racecheck-report hazard"
  timeout ${SAN_TIMEOUT:-1200} /usr/local/cuda/bin/compute-sanitizer --tool $t $extra --kernel-name regex=xnc \
      --target-processes application-only python tools/sanitize_cases.py > $out/sanitize_${t}_${tag}.log 2>&1
  rc=$?
  echo "$t rc=$rc $(grep -h 'SUMMARY' $out/sanitize_${t}_${tag}.log | tail -1) cases_ok=$(grep -c ': ok' $out/sanitize_${t}_${tag}.log)"
  if [ "$t" = "racecheck" ]; then
    python tools/race_summary.py $out/sanitize_${t}_${tag}.log > $out/sanitize_racecheck_${tag}_summary.txt
    head -c 200000 $out/sanitize_${t}_${tag}.log > $out/sanitize_${t}_${tag}.head.log
    rm -f $out/sanitize_${t}_${tag}.log
    cat $out/sanitize_racecheck_${tag}_summary.txt | head -40
  fi
done
