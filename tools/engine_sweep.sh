#!/bin/bash
# Build engine variants (-D flags) into /tmp and time each with
# tools/engine_bench.py.  Usage: bash tools/engine_sweep.sh "-DA=1" "-DA=2" ...
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
SRC="${SWEEP_SRC:-paper_2506_14851_b200/csrc}"
[ -n "${SWEEP_APPEND:-}" ] || : > gpurun_out/sweep.txt
i=0
for flags in "$@"; do
  out=/tmp/pdg_var_${SWEEP_TAG:-}$i.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -shared -cudart static -I include $flags -o $out \
    $SRC/*.cu > /tmp/nvcc_$i.log 2>&1 || { echo "build failed: $flags" >> gpurun_out/sweep.txt; cat /tmp/nvcc_$i.log >> gpurun_out/sweep.txt; i=$((i+1)); continue; }
  echo "== $flags" >> gpurun_out/sweep.txt
  PDG_LIB_PATH=$out timeout 300 python tools/engine_bench.py >> gpurun_out/sweep.txt 2>&1
  i=$((i+1))
done
echo done >> gpurun_out/sweep.txt
