set -u
timeout 900 python -m pytest tests -x -q -m gpu  2>&1 | tail -1
for i in 1 2 3; do timeout 300 python tools/umma_sweep.py --cfgs C3,C2k3,C2k5,C2k7 --reps 30; done 2>&1 | tee gpurun_out/fmul2_r3l.log
