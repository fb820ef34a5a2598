#!/usr/bin/env bash
# Compile the reference's own CPU kernels (xnorconv._kernels_cy, the Cython/OpenMP
# extension behind ConvWorkspace.run) into oracle/_ref/ -- the CPU baseline and a
# second checker.  Reads the .pyx where it lies under /root/reference (read-only;
# nothing is copied into the repo).  Two steps:
#   1. cython -> oracle/_ref/_kernels_cy.c       (only where /root/reference exists)
#   2. gcc    -> oracle/_ref/_kernels_cy<EXT>.so (the reference's setup.py flags:
#      -O3 -fopenmp -march=native; /usr/bin/gcc because sysconfig's wrapper
#      lacks libgomp.spec -- SURVEY.md section 0 item 7)
# Step 2 alone re-runs on the GPU box (`build_ref.sh --cc-only`) so -march=native
# matches that host.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
out="$here/_ref"
pyx=/root/reference/pkg/src/xnorconv/_kernels_cy.pyx
mkdir -p "$out"
if [[ "${1:-}" != "--cc-only" ]]; then
  if [[ ! -f "$pyx" ]]; then echo "reference sources absent: $pyx" >&2; exit 3; fi
  cython -3 --module-name xnorconv._kernels_cy "$pyx" -o "$out/_kernels_cy.c"
fi
[[ -f "$out/_kernels_cy.c" ]] || { echo "no generated C in $out" >&2; exit 3; }
py=${PYTHON:-python3}
inc=$($py -c 'import sysconfig; print(sysconfig.get_paths()["include"])')
npinc=$($py -c 'import numpy; print(numpy.get_include())')
suffix=$($py -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')
march=${REF_MARCH:-native}
/usr/bin/gcc -O3 -fopenmp -march="$march" -fPIC -shared -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
  -I"$inc" -I"$npinc" "$out/_kernels_cy.c" -o "$out/_kernels_cy$suffix" -lgomp
echo "built $out/_kernels_cy$suffix (march=$march)"
