#!/usr/bin/env bash
# ncu metrics of the tcgen05 pair conv kernel at C3 for a list of XNC_UMMA_DEBUG values
out=gpurun_out; mkdir -p $out
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__average_warp_latency_issue_stalled_long_scoreboard
for d in "$@"; do
  XNC_UMMA_DEBUG=$d timeout 300 ncu --metrics $M --clock-control none -k regex:k_conv_umma -s 2 -c 1 --csv \
    python tools/umma_sweep.py --child C3 --reps 3 > $out/ncu_pair_d$d.csv 2>&1
  echo "debug=$d rc=$?"
done
