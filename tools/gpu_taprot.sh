out=gpurun_out; tag=${1:-r4i}
for r in 0 1 0 1; do XNC_TAP_ROT=$r timeout 300 python tools/umma_sweep.py --cfgs C3,C2k3,C2k5,C2k7,conv2,conv3,conv5 | sed "s/^/rot=$r /"; done > $out/taprot_$tag.log 2>&1; cat $out/taprot_$tag.log | cut -c1-90
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
