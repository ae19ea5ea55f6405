#!/bin/bash
# Careful second pass (in-visit Lemire redraw): parity, LLM/duration engine A/B,
# K1b pair variants, bench.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_e.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_e.txt
AB_ROUNDS=1 bash tools/ab2.sh
: > gpurun_out/llm_time.txt
for lib in /tmp/pdg_a.so /tmp/pdg_b.so; do PDG_LIB_PATH=$lib timeout 300 python tools/llm_time.py >> gpurun_out/llm_time.txt 2>&1; done
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
  -Xcompiler -fPIC -shared -cudart static -I include -DPDG_WALK_MINB=4 -o /tmp/pdg_m4.so \
  paper_2506_14851_b200/csrc/*.cu > /tmp/m4.log 2>&1 && \
  PDG_LIB_PATH=/tmp/pdg_m4.so timeout 300 python tools/llm_time.py >> gpurun_out/llm_time.txt 2>&1
bash tools/k1_sweep.sh "-DPDG_PAIR_WARPS=4 -DPDG_PAIR_STAGES=2 -DPDG_PAIR_MINB=3" \
  "-DPDG_PAIR_WARPS=2 -DPDG_PAIR_STAGES=2 -DPDG_PAIR_MINB=6" \
  "-DPDG_PAIR_WARPS=4 -DPDG_PAIR_STAGES=1 -DPDG_PAIR_MINB=5"
timeout 900 python bench.py > gpurun_out/bench_e.json 2> gpurun_out/bench_e.err
echo all-done
