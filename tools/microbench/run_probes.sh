set -x
cd tools/microbench
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/mxf4_probe mxf4_probe.cu && timeout 120 /tmp/mxf4_probe > ../../gpurun_out/mxf4_probe.jsonl 2>&1; echo mxf4 rc=$?
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/store_probe store_probe.cu && timeout 120 /tmp/store_probe > ../../gpurun_out/store_probe.jsonl 2>&1; echo store rc=$?
cat ../../gpurun_out/mxf4_probe.jsonl ../../gpurun_out/store_probe.jsonl
