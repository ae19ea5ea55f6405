#!/bin/bash
# Build variants (-D flags) and time K1b (bench.bench_k1_large) at 1M and
# 100k rows.  Usage: bash tools/k1_sweep.sh "-DPDG_ROWS_STAGES=2" ...
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
SRC="paper_2506_14851_b200/csrc"
: > gpurun_out/k1_sweep.txt
i=0
for flags in "$@"; do
  out=/tmp/pdg_k1_$i.so
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -shared -cudart static -I include $flags -o $out \
    $SRC/*.cu \
    > /tmp/nvcc_k1_$i.log 2>&1 || { echo "build failed: $flags" >> gpurun_out/k1_sweep.txt; i=$((i+1)); continue; }
  echo "== $flags" >> gpurun_out/k1_sweep.txt
  PDG_LIB_PATH=$out timeout 300 python -c "
import json, torch, bench
d = torch.device('cuda', 0)
a = bench.bench_k1_large(d)
b = bench.bench_k1_large(d, n=100_000)
print(json.dumps({'1m_ms': a['ms_per_launch'], '1m_frac': a['roofline']['frac'], '100k_ms': b['ms_per_launch'], '100k_frac': b['roofline']['frac']}))
" >> gpurun_out/k1_sweep.txt 2>&1
  i=$((i+1))
done
echo done >> gpurun_out/k1_sweep.txt
