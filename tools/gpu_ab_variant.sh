# A/B a build variant against the default library on the conv sweep: bash tools/gpu_ab_variant.sh <variant.so> [cfgs]
v=$1; cfgs=${2:-C3,C2k3,C2k5,C2k7}
for i in 1 2; do
  timeout 300 python tools/umma_sweep.py --cfgs $cfgs --reps 30 | sed "s/^/default /"
  XNC_LIB=$v timeout 300 python tools/umma_sweep.py --cfgs $cfgs --reps 30 | sed "s/^/variant /"
done
