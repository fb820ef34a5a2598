out=gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pool_pack -c 3 -o $out/pool_r4f -f python tools/c4_launches.py 8 > $out/ncu_pool_r4f.log 2>&1; echo "ncu rc=$?"
tail -5 $out/ncu_pool_r4f.log
