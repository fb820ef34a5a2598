#!/usr/bin/env bash
# Build an alternative libxnorb200.so with extra -D flags into build/<name>.so
# (tuning experiments; load with XNC_LIB=build/<name>.so).
# Usage: tools/build_variant.sh <name> [-DXNC_...=...]...
set -e
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
mkdir -p "$root/build"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
  -Xcompiler -fPIC -I "$root/include" "$@" -o "$root/build/$name.so" "$root"/paper_2007_14178_b200/csrc/*.cu
echo "built build/$name.so"
