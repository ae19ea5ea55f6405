#!/bin/bash
# Engine A/B: ab_base/csrc (A) vs the working tree (B), each built once,
# timed alternately (tools/engine_bench.py) ${AB_ROUNDS:-3} times.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
: > gpurun_out/ab.txt
build() {
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC -shared -cudart static -I include ${3:-} -o $2 $1/*.cu > $2.log 2>&1 \
    || { echo "build failed: $1" >> gpurun_out/ab.txt; cat $2.log >> gpurun_out/ab.txt; }
}
build ab_base/csrc /tmp/pdg_a.so &
build paper_2506_14851_b200/csrc /tmp/pdg_b.so "${1:-}" &
wait
for r in $(seq 1 ${AB_ROUNDS:-3}); do
  for v in a b; do
    echo "== $v$r" >> gpurun_out/ab.txt
    PDG_LIB_PATH=/tmp/pdg_$v.so timeout 300 python tools/engine_bench.py ${AB_ARGS:-} >> gpurun_out/ab.txt 2>&1
  done
done
echo done >> gpurun_out/ab.txt
