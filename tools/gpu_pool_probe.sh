out=gpurun_out; tag=${1:-r4g}
for b in 0 1; do XNC_POOL_BAND=$b timeout 300 python tools/pool_probe.py 256; done > $out/pool_probe_$tag.jsonl 2>&1; cat $out/pool_probe_$tag.jsonl
XNC_POOL_BAND=0 timeout 900 ncu --set full --clock-control none -k regex:"pool|pack_input_nhwc" -s 6 -c 8 -o $out/poolold_$tag -f python tools/pool_probe.py 256 > $out/ncu_poolold_$tag.log 2>&1; echo "ncu rc=$?"
