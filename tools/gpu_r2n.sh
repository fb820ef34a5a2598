set -u
out=gpurun_out
timeout 300 python tools/c4_stages.py 256 > $out/c4_stages_256_r2n.json 2>&1; tail -1 $out/c4_stages_256_r2n.json
timeout 300 python tools/c4_stages.py 2048 > $out/c4_stages_2048_r2n.json 2>&1; tail -1 $out/c4_stages_2048_r2n.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pack_small_pool -s 2 -c 1 -o $out/poolk1_r2n -f python tools/c4_kernels.py > $out/ncu_poolk1_r2n.log 2>&1; echo "ncu rc=$?"
