out=gpurun_out
timeout 600 python tools/umma_sweep.py --cfgs C3,conv3 --debug 2,6,7,134 > $out/fp4_dbg_r4c.jsonl 2>&1; echo "fp4 dbg rc=$?"
XNC_LIB=build/i8.so timeout 600 python tools/umma_sweep.py --cfgs C3 --debug 2,6,7,134 > $out/i8_dbg_r4c.jsonl 2>&1; echo "i8 dbg rc=$?"
cat $out/fp4_dbg_r4c.jsonl; echo; cat $out/i8_dbg_r4c.jsonl
