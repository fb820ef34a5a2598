out=gpurun_out
timeout 600 python tools/umma_sweep.py --cfgs C3,C2k3,conv3 --debug 0,1,4,32,37,128 > $out/fp4_dbg_r4b.jsonl 2>&1; echo "fp4 dbg rc=$?"
XNC_LIB=build/i8.so timeout 600 python tools/umma_sweep.py --cfgs C3,C2k3 --debug 0,1,4,32,37,128 > $out/i8_dbg_r4b.jsonl 2>&1; echo "i8 dbg rc=$?"
cat $out/fp4_dbg_r4b.jsonl; echo; cat $out/i8_dbg_r4b.jsonl
