for m in 1 2 4 8; do XNC_UMMA_SPLIT_MAX=$m timeout 120 python tools/fc_probe.py | sed "s/^/split_max=$m /"; done
