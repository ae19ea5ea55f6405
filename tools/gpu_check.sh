#!/bin/bash
# One GPU round trip: tests, smoke, bench, ncu launch list + full captures.
# Usage (from the build container):
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/gpu_check.sh'
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.txt
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 2 --ncu \
  > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mc_walk|mc_engine" \
  -s 3 -c 1 -o gpurun_out/engine -f python bench.py --steps 1 --warmup 2 --ncu \
  > gpurun_out/ncu_engine.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gittins \
  -s 3 -c 1 -o gpurun_out/k1 -f python bench.py --steps 1 --warmup 2 --ncu \
  > gpurun_out/ncu_k1.log 2>&1

timeout 600 ncu --set full --clock-control none --import-source on -k regex:prewarm_need \
  -s 2 -c 1 -o gpurun_out/need -f python bench.py --steps 1 --warmup 1 --no-cpu-baseline \
  > gpurun_out/ncu_need.log 2>&1
echo done
