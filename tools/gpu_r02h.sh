#!/bin/bash
# Min-tracking Lemire check: full GPU suite, engine A/B vs the round-start
# sources, ncu captures of the first-pass kernels, LLM timing.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_h.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_h.txt
AB_ROUNDS=2 bash tools/ab2.sh
timeout 300 python tools/llm_time.py > gpurun_out/llm_time_h.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"mc_walk_kernel<.int.0, unsigned int, .bool.0>" -s 3 -c 1 -o gpurun_out/engine -f \
  python bench.py --steps 1 --warmup 3 --ncu --no-extra > gpurun_out/ncu_engine.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"mc_walk_kernel<.int.7, unsigned int, .bool.0>" -s 2 -c 1 -o gpurun_out/engine_llm -f \
  python tools/llm_engine_run.py 100000 3 > gpurun_out/ncu_engine_llm.log 2>&1
echo all-done
