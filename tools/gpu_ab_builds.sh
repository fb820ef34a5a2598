# A/B of library builds on the conv sweep: cur = the in-tree .so, others = build/<name>.so
# usage: bash tools/gpu_ab_builds.sh <tag> <cfgs> <name>...
out=gpurun_out; tag=$1; cfgs=$2; shift 2
for i in 1 2 3; do
  for v in cur "$@"; do
    if [ "$v" = cur ]; then timeout 300 python tools/umma_sweep.py --cfgs $cfgs 2>&1
    else XNC_LIB=build/$v.so timeout 300 python tools/umma_sweep.py --cfgs $cfgs 2>&1; fi | cut -c1-62 | sed "s/^/$v /"
  done
done > $out/ab_$tag.log
cat $out/ab_$tag.log
