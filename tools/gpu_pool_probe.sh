# pooled-K1 passes at batch 256 (tools/pool_probe.py) and an ncu capture of their kernels
out=gpurun_out; tag=${1:-r4g}
timeout 300 python tools/pool_probe.py 256 > $out/pool_probe_$tag.jsonl 2>&1; cat $out/pool_probe_$tag.jsonl
timeout 900 ncu --set full --clock-control none -k regex:"pool|pack_input_nhwc" -s 6 -c 8 -o $out/pool_$tag -f \
    python tools/pool_probe.py 256 > $out/ncu_pool_$tag.log 2>&1; echo "ncu rc=$?"
