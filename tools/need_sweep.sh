#!/bin/bash
# Build variants (-D flags) and time config 5 (bench.bench_need) with each.
# Usage: bash tools/need_sweep.sh "-DPDG_NEED_BATCH=2" ...
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
SRC="paper_2506_14851_b200/csrc"
: > gpurun_out/need_sweep.txt
i=0
for flags in "$@"; do
  out=/tmp/pdg_need_$i.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -shared -cudart static -I include $flags -o $out \
    $SRC/*.cu \
    > /tmp/nvcc_need_$i.log 2>&1 || { echo "build failed: $flags" >> gpurun_out/need_sweep.txt; i=$((i+1)); continue; }
  echo "== $flags" >> gpurun_out/need_sweep.txt
  PDG_LIB_PATH=$out timeout 300 python -c "
import json, torch, bench
r = bench.bench_need(torch.device('cuda', 0), cpu=False)
print(json.dumps({'ms': r['ms_per_launch'], 'frac': r['roofline']['frac']}))
" >> gpurun_out/need_sweep.txt 2>&1
  i=$((i+1))
done
echo done >> gpurun_out/need_sweep.txt
