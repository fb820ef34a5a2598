for d in 0 1024 2048; do XNC_FUSED_DEBUG=$d timeout 120 python tools/fused_probe.py C3 | sed "s/^/dbg=$d /"; done
XNC_FUSED=0 timeout 120 python tools/fused_probe.py C3
