#!/bin/bash
# New-kernel GPU tests, K1b variant sweep, engine ncu source-line captures
# (duration variant <0> from the bench, LLM variant <7>), bench line.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gittins_gpu.py tests/test_attained_gpu.py \
  tests/test_prewarm_gpu.py tests/test_prewarm_wide_gpu.py tests/test_workload_gpu.py \
  tests/test_stream_gpu.py -q -x > gpurun_out/pytest_new.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_new.txt
bash tools/k1_sweep.sh "-DPDG_ROWS_WARPS=6 -DPDG_ROWS_STAGES=2" "-DPDG_ROWS_WARPS=4 -DPDG_ROWS_STAGES=3" \
  "-DPDG_ROWS_WARPS=12 -DPDG_ROWS_STAGES=1" "-DPDG_ROWS_WARPS=3 -DPDG_ROWS_STAGES=4" \
  "-DPDG_ROWS_WARPS=8 -DPDG_ROWS_STAGES=1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mc_walk" \
  -s 3 -c 1 -o gpurun_out/engine -f python bench.py --steps 1 --warmup 2 --ncu --no-extra \
  > gpurun_out/ncu_engine.log 2>&1
python tools/ncu_lines.py gpurun_out/engine.ncu-rep 0.003 > gpurun_out/engine_lines.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mc_walk" \
  -s 2 -c 1 -o gpurun_out/engine_llm -f python tools/llm_engine_run.py 100000 3 \
  > gpurun_out/ncu_engine_llm.log 2>&1
python tools/ncu_lines.py gpurun_out/engine_llm.ncu-rep 0.003 > gpurun_out/engine_llm_lines.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gittins_rows" \
  -s 3 -c 1 -o gpurun_out/k1 -f python bench.py --steps 1 --warmup 2 --ncu --no-extra \
  > gpurun_out/ncu_k1.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
