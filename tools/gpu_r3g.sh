timeout 300 python tools/umma_sweep.py --cfgs conv2,conv3,conv5,C3 --debug 0,128,1 --reps 20 2>&1 | tee gpurun_out/umma_net_layers_r3g.log
