#!/bin/bash
# Build variants (-D flags) and evaluate one Python expression (printed as
# JSON) with each.  Usage: bash tools/fn_sweep.sh 'bench.bench_refresh_latency()' "-DX=0" ...
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
SRC="paper_2506_14851_b200/csrc"
expr="$1"; shift
: > gpurun_out/fn_sweep.txt
i=0
for flags in "$@"; do
  out=/tmp/pdg_fn_$i.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -shared -cudart static -I include $flags -o $out \
    $SRC/*.cu \
    > /tmp/nvcc_fn_$i.log 2>&1 || { echo "build failed: $flags" >> gpurun_out/fn_sweep.txt; i=$((i+1)); continue; }
  echo "== $flags" >> gpurun_out/fn_sweep.txt
  PDG_LIB_PATH=$out timeout 600 python -c "
import json, torch, bench
print(json.dumps($expr))
" >> gpurun_out/fn_sweep.txt 2>&1
  i=$((i+1))
done
echo done >> gpurun_out/fn_sweep.txt
