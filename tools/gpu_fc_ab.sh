timeout 600 python -m pytest tests -x -q -m gpu -k "fc or network" 2>&1 | tail -1
for v in 1 0 1 0; do XNC_WIDE_A_1X1=$v timeout 120 python tools/fc_probe.py | sed "s/^/wide1x1=$v /"; done
