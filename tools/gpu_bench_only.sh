#!/bin/bash
# Bench + engine ncu only (fast perf iteration).
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python bench.py --no-extra --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mc_walk|mc_engine" \
  -s 3 -c 1 -o gpurun_out/engine -f python bench.py --steps 1 --warmup 2 --ncu --no-extra \
  > gpurun_out/ncu_engine.log 2>&1
echo done
