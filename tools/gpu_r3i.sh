set -u
timeout 900 python -m pytest tests -x -q -m gpu -k "fc or channels_last or network or umma" 2>&1 | tail -1
bash tools/gpu_round.sh r3i ncu-conv bench-quick
python tools/ncu_summary.py gpurun_out/conv_r3i.ncu-rep | head -8
