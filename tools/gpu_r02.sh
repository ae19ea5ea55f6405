#!/bin/bash
# Round-2 measurement pass on one B200: GPU tests, smoke, bench (both arms),
# ncu launch list of the bench, full ncu captures of the engine and K1b.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
bash tools/gpu_round.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mc_walk" \
  -s 3 -c 1 -o gpurun_out/engine -f python bench.py --steps 1 --warmup 3 --ncu --no-extra \
  > gpurun_out/ncu_engine.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gittins_rows" \
  -s 3 -c 1 -o gpurun_out/k1 -f python bench.py --steps 1 --warmup 3 --ncu --no-extra \
  > gpurun_out/ncu_k1.log 2>&1
echo all-done
