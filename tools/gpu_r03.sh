#!/bin/bash
# Final pass (r03): GPU suite, smoke, bench (both arms), engine + K1b ncu,
# launch list.
set -u
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_q.txt 2>&1
echo "exit $?" >> gpurun_out/pytest_q.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_q.txt 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_q.txt
timeout 300 python tools/llm_time.py > gpurun_out/llm_time_q.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_q.json 2> gpurun_out/bench_ref_q.err
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"mc_walk_kernel<.int.0, unsigned int, .bool.0>" -s 3 -c 1 -o gpurun_out/engine -f \
  python bench.py --steps 1 --warmup 3 --ncu --no-extra > gpurun_out/ncu_engine.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gittins_pair" \
  -s 3 -c 1 -o gpurun_out/k1 -f python -c "
import torch, bench
bench.bench_k1_large(torch.device('cuda', 0), reps=2)" > gpurun_out/ncu_k1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline \
  > gpurun_out/launches_bench.log 2>&1
echo all-done
