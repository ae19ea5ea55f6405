#!/bin/bash
# Own-input careful redraw: parity on the LLM queue's rejections, timings,
# engine ncu capture of the first-pass kernel, bench (both arms).
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_workload_gpu.py tests/test_engine_gpu.py tests/test_gittins_gpu.py -q > gpurun_out/pytest_g.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_g.txt
timeout 300 python tools/llm_time.py > gpurun_out/llm_time_g.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"mc_walk_kernel<0, unsigned int, 0>" -s 3 -c 1 -o gpurun_out/engine -f \
  python bench.py --steps 1 --warmup 3 --ncu --no-extra > gpurun_out/ncu_engine.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"mc_walk_kernel<7, unsigned int, 0>" -s 2 -c 1 -o gpurun_out/engine_llm -f \
  python tools/llm_engine_run.py 100000 3 > gpurun_out/ncu_engine_llm.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_g.json 2> gpurun_out/bench_ref_g.err
echo all-done
