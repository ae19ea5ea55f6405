#!/bin/bash
# ncu --set full capture of one mc_walk launch of an engine variant built with
# the given -D flags.  Usage: bash tools/ncu_variant.sh NAME "-DFLAG=1 ..."
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
SRC="paper_2506_14851_b200/csrc"
out=/tmp/pdg_ncu_$1.so
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -shared -cudart static -I include $2 -o $out \
  $SRC/*.cu \
  > gpurun_out/ncu_$1_build.log 2>&1 || exit 1
PDG_LIB_PATH=$out timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:mc_walk -s 2 -c 1 -o gpurun_out/$1 -f python tools/engine_bench.py --reps 3 \
  > gpurun_out/ncu_$1.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_$1.log
