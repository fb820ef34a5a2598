out=gpurun_out
timeout 300 python tools/umma_sweep.py --cfgs C3,C2k3,C2k5,C2k7,conv2,conv3,conv5 > $out/fp4_sweep_r4a.jsonl 2>&1; echo "fp4 sweep rc=$?"
XNC_LIB=build/i8.so timeout 300 python tools/umma_sweep.py --cfgs C3,C2k3,C2k5,C2k7,conv2,conv3,conv5 > $out/i8_sweep_r4a.jsonl 2>&1; echo "i8 sweep rc=$?"
paste -d' ' <(cut -c1-80 $out/fp4_sweep_r4a.jsonl) <(cut -c1-80 $out/i8_sweep_r4a.jsonl)
timeout 900 python -m pytest tests -x -q -m gpu > $out/pytest_gpu_r4a.log 2>&1; echo "pytest rc=$?"; tail -15 $out/pytest_gpu_r4a.log
