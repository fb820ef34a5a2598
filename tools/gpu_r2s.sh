set -u
timeout 600 python -m pytest tests -x -q -m gpu -k "fused" 2>&1 | tail -15
for f in 1 0 1 0; do XNC_FUSED=$f timeout 120 python tools/fused_probe.py C3; done 2>&1 | tee gpurun_out/fused_ab_r2s.log
